"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the builder container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src (and
its test helpers/oracle from /root/reference/pkg/tests), evaluates it on
seeded inputs, and writes small .npz fixtures next to this script.  The GPU
tests, smoke() and bench.py never read /root/reference; they read these files.

Fixtures
  dimer.npz        carbon dimer at 1.4 A (ScalarOpt) + the reference suite's
                   frozen 50-digit goldens (test_kernels.py:21-22)
  clusters.npz     random free clusters, carbon and the synthetic two-species
                   table (test helpers), n = 4..8 and 12/25/40: ScalarOpt
                   double + single, longdouble brute-force energy
                   (tests/oracle.py), zeta_visits
  si512.npz        BASELINE config 1 (512 Si): neighbour list, ScalarOpt
                   double/single E/F/e_i, virial diagonal from central finite
                   differences of the reference energy under affine strain,
                   100-step NVE energies (run_nve, ScalarOpt)
  sic216.npz       3C-SiC 3^3 cells on the SiC fixture table (ScalarOpt)
  disordered.npz   1000-atom min-separation random Si packing (ScalarOpt)
  nl_frames.npz    neighbour-list edge cases (random 200-atom frames with
                   ppp / fff / ffp periodicity; test_neighbor.py:16-82)
  harness.npz      gen_nanotube / gen_diamond positions, write_xyz text, a
                   40-step run_stretch record, the bench CSV header
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = os.environ.get("TERSOFF_REF", "/root/reference/pkg/src")
REF_TESTS = os.path.join(os.path.dirname(REF_SRC), "tests")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)
sys.path.insert(0, REPO)

import tersoffmd as R  # noqa: E402  (the reference)
from tersoffmd.kernels import compute as ref_compute, make_variant  # noqa: E402
from tersoffmd.neighbor import build_neighbor_list as ref_build  # noqa: E402
from tersoffmd.paramfile import parse_params as ref_parse, serialize_params  # noqa: E402

import helpers  # noqa: E402  (reference test helpers)
import oracle as ld_oracle  # noqa: E402  (reference longdouble oracle)

from paper_1710_00882_b200 import structures  # noqa: E402  (input generators)
from paper_1710_00882_b200.paramfile import DATA_DIR  # noqa: E402

SCALAR = make_variant("ScalarOpt")
SINGLE = make_variant("ScalarOpt", precision="single")


class Frame:
    def __init__(self, pos, lengths, periodic, species):
        self.positions = np.asarray(pos, dtype=np.float64)
        self.box = helpers.Box(lengths, periodic)
        self.species = np.asarray(species, dtype=np.int64)


def table_text(name):
    with open(os.path.join(DATA_DIR, f"{name}.tersoff")) as fh:
        return fh.read()


def run(fr, table, skin=0.3, single=True):
    nl = ref_build(fr, table.r_cut, skin)
    d = ref_compute(fr, nl, table, SCALAR)
    out = dict(offsets=nl.offsets, neighbors=nl.neighbors, energy=d.potential_energy,
               forces=d.forces, per_atom=d.per_atom_energy,
               zeta_visits=d.stats["zeta_visits"])
    if single:
        s = ref_compute(fr, nl, table, SINGLE)
        out.update(energy_single=s.potential_energy, forces_single=s.forces)
    return out


def state_frame(st):
    return Frame(st.positions, st.box.lengths, st.box.periodic, st.species)


def dimer():
    t = helpers.carbon_table()
    fr = helpers.free_frame(np.array([[0.0, 0.0, 0.0], [1.4, 0.0, 0.0]]))
    fr.species = np.zeros(2, dtype=np.int64)
    r = run(Frame(fr.positions, fr.box.lengths, fr.box.periodic, fr.species), t)
    np.savez(os.path.join(HERE, "dimer.npz"), positions=fr.positions,
             lengths=fr.box.lengths, periodic=np.array(fr.box.periodic),
             species=fr.species, table=serialize_params(t),
             frozen_energy=-10.235536457692383, frozen_f0x=-4.295997777189043, **r)


def clusters():
    rows = []
    specs = [(seed, 4 + seed % 5, mixed) for mixed in (False, True) for seed in range(6)]
    specs += [(0, 12, False), (1, 25, True), (2, 40, False), (7, 8, True), (6, 16, True)]
    for seed, n, mixed in specs:
        rng = np.random.default_rng(seed)
        t = helpers.two_species_table() if mixed else helpers.carbon_table()
        fr = helpers.free_frame(helpers.random_cluster_positions(rng, n))
        sp = rng.integers(0, 2, n) if mixed else np.zeros(n, dtype=np.int64)
        f = Frame(fr.positions, fr.box.lengths, fr.box.periodic, sp)
        r = run(f, t)
        e_ld = float(ld_oracle.oracle_energy(f.positions, f.species, t)) if n <= 12 else np.nan
        rows.append(dict(seed=seed, n=n, mixed=mixed, positions=f.positions,
                         lengths=f.box.lengths, species=f.species, energy_ld=e_ld, **r))
    out = {}
    for k, row in enumerate(rows):
        for key, v in row.items():
            out[f"c{k}_{key}"] = v
    out["count"] = len(rows)
    out["table_carbon"] = serialize_params(helpers.carbon_table())
    out["table_mixed"] = serialize_params(helpers.two_species_table())
    np.savez(os.path.join(HERE, "clusters.npz"), **out)


def strain_energy(fr, table, ax, eps):
    g = Frame(fr.positions.copy(), fr.box.lengths.copy(), fr.box.periodic, fr.species)
    g.positions[:, ax] *= 1.0 + eps
    g.box.lengths[ax] *= 1.0 + eps
    nl = ref_build(g, table.r_cut, 0.3)
    return ref_compute(g, nl, table, SCALAR).potential_energy


def si512():
    st, name = structures.config(1)
    t = ref_parse(table_text(name))
    fr = state_frame(st)
    r = run(fr, t)
    # virial diagonal W_aa = -L_a dE/dL_a by a 4th-order central difference in
    # the strain eps (dE/deps = L dE/dL)
    h = 1e-5
    wdiag = []
    for ax in range(3):
        e = [strain_energy(fr, t, ax, s * h) for s in (-2, -1, 1, 2)]
        dedeps = (e[0] - 8 * e[1] + 8 * e[2] - e[3]) / (12 * h)
        wdiag.append(-dedeps)
    # NVE: 100 steps, dt 1 fs (BASELINE config 1), reference ScalarOpt
    s2 = R.SimulationState(st.positions.copy(), R.SimulationBox(st.box.lengths, st.box.periodic),
                           species=st.species.copy(), masses=st.masses.copy(),
                           symbols=st.symbols, velocities=st.velocities.copy())
    nve = R.run_nve(s2, t, R.RunConfig(dt=1.0, steps=100, variant=SCALAR, skin=0.3))
    np.savez(os.path.join(HERE, "si512.npz"), positions=st.positions, lengths=st.box.lengths,
             periodic=np.array(st.box.periodic), species=st.species,
             velocities=st.velocities, masses=st.masses, table=table_text(name),
             virial_fd_diag=np.array(wdiag), nve_total=nve["total"],
             nve_potential=nve["potential"], nve_rebuilds=nve["rebuilds"],
             nve_final_positions=s2.positions, **r)


def small(name_out, st, tname):
    t = ref_parse(table_text(tname))
    r = run(state_frame(st), t)
    np.savez(os.path.join(HERE, name_out), positions=st.positions, lengths=st.box.lengths,
             periodic=np.array(st.box.periodic), species=st.species, table=table_text(tname),
             **r)


def nl_frames():
    out = {}
    for k, per in enumerate([(True, True, True), (False, False, False), (False, False, True)]):
        rng = np.random.default_rng(42)
        pos = rng.uniform(0, 9.0, (200, 3))
        fr = Frame(pos, (9.0, 9.0, 9.0), per, np.zeros(200, np.int64))
        nl = ref_build(fr, 2.1, 0.3)
        out[f"f{k}_positions"] = pos
        out[f"f{k}_periodic"] = np.array(per)
        out[f"f{k}_offsets"] = nl.offsets
        out[f"f{k}_neighbors"] = nl.neighbors
    out["count"] = 3
    np.savez(os.path.join(HERE, "nl_frames.npz"), **out)


def harness():
    """Structure generators, XYZ text, the stretch driver and the bench CSV
    schema of the reference (system.py:164-307, 478-550; bench.py:23-25)."""
    import tempfile

    from tersoffmd import bench as ref_bench
    from tersoffmd import system as ref_system
    out = {}
    for n, cells in [(3, 1), (5, 10), (8, 4)]:
        st = ref_system.gen_nanotube(n, cells)
        out[f"tube_{n}_{cells}_positions"] = st.positions
        out[f"tube_{n}_{cells}_lengths"] = st.box.lengths
    dia = ref_system.gen_diamond(3)
    out["diamond3_positions"] = dia.positions
    out["diamond3_lengths"] = dia.box.lengths
    st = ref_system.gen_nanotube(5, 2)
    st.time = 12.5
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "t.xyz")
        ref_system.write_xyz(path, st)
        ref_system.write_xyz(path, ref_system.gen_diamond(1), append=True)
        out["xyz_text"] = np.array(open(path).read())
    # stretch run on a (5,5) tube, carbon table (cli run --pull-speed)
    table = R.builtin_params("C")
    st = ref_system.gen_nanotube(5, 4)
    ref_system.seed_velocities(st, 300.0, 7)
    out["stretch_positions0"] = st.positions.copy()
    out["stretch_velocities0"] = st.velocities.copy()
    cfg = ref_system.RunConfig(dt=0.5, steps=40, variant=SCALAR, skin=0.3,
                               stretch=ref_system.StretchSpec(axis=2, speed=0.02))
    rec = ref_system.run_stretch(st, table, cfg)
    for k in ("potential", "kinetic", "total", "strain", "force_sum_max"):
        out[f"stretch_{k}"] = np.asarray(rec[k])
    out["stretch_grip_atoms"] = np.array(rec["grip_atoms"])
    out["stretch_rebuilds"] = rec["rebuilds"]
    out["stretch_final_positions"] = st.positions
    out["csv_fields"] = np.array(",".join(ref_bench.CSV_FIELDS))
    np.savez(os.path.join(HERE, "harness.npz"), **out)


def main():
    harness()
    dimer()
    clusters()
    si512()
    sic = structures.displace(structures.gen_zincblende(3, 4.359), 0.08, 1003)
    small("sic216.npz", sic, "SiC")
    dis = structures.gen_disordered(1000, 0.05, 2.0, 1004)
    small("disordered.npz", dis, "Si")
    nl_frames()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
