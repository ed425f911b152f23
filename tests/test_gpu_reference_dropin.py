"""Boundary acceptance: the reference's OWN code on the B200 ABI.

The reference package (installed read-only into baseline/_ref from the
reference sources; it travels to the GPU box with the repo) is imported and
the B200 kernel plugged in with integration.install() -- the binding
INTEGRATION.md describes.  Then:

* the assertions of pkg/tests/test_kernels.py:74-100 (frozen dimer goldens,
  random clusters against the reference's ScalarOpt) and :218-249 (visit
  counters, lane utilisation, gathers) hold for the B200 kernel, with the
  reference's KernelVariant / NeighborList objects passed straight to
  paper_1710_00882_b200.compute;
* the reference's ForceField / run_nve (system.py:314-348, :427-460) with
  the "B200" variant reproduce its ScalarOpt NVE trajectory;
* run_verification (verify.py:256-276), run_benchmark (bench.py:106-164) and
  the CLI (`--variant b200`) run on it.

Skipped when baseline/_ref is absent (it is never read from /root/reference).
"""

import json
import os
import sys

import numpy as np
import pytest

import paper_1710_00882_b200 as B
from conftest import ROOT, golden_clusters, load_golden
from paper_1710_00882_b200 import integration

pytestmark = pytest.mark.gpu

DIMER_E = -10.235536457692383   # test_kernels.py:21-22 (frozen from a 50-digit evaluation)
DIMER_F0X = -4.295997777189043


@pytest.fixture(scope="module")
def ref():
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "tersoffmd")):
        pytest.skip("reference package not installed in baseline/_ref")
    if path not in sys.path:
        sys.path.insert(0, path)
    import tersoffmd
    import tersoffmd.bench
    import tersoffmd.cli
    import tersoffmd.kernels
    import tersoffmd.neighbor
    import tersoffmd.paramfile
    import tersoffmd.system
    import tersoffmd.verify
    integration.install(tersoffmd)
    yield tersoffmd
    integration.uninstall(tersoffmd)


def _free_frame(ref, pos, species):
    pos = np.asarray(pos, dtype=np.float64)
    span = pos.max(axis=0) - pos.min(axis=0) + 8.0
    st = ref.system.SimulationState(pos, ref.system.SimulationBox(span), species=species,
                                    masses=np.full(int(np.max(species)) + 1, 12.011))
    return st


@pytest.mark.parametrize("precision", ["double"])
def test_dimer_frozen_goldens_through_reference_dispatch(ref, precision):
    K = ref.kernels
    table = ref.paramfile.builtin_params("C")
    st = _free_frame(ref, [[0.0, 0.0, 0.0], [1.4, 0.0, 0.0]], np.zeros(2, np.int64))
    nl = ref.neighbor.build_neighbor_list(st, table.r_cut, skin=0.3)
    res = K.compute(st, nl, table, K.make_variant("B200", precision=precision))
    assert type(res) is K.ForceEnergyResult
    assert res.potential_energy == pytest.approx(DIMER_E, rel=5e-14)
    assert res.forces[0, 0] == pytest.approx(DIMER_F0X, rel=5e-13)
    assert res.forces[0, 0] == -res.forces[1, 0]  # exact pair antisymmetry
    assert np.all(res.forces[:, 1:] == 0.0)
    assert res.per_atom_energy.sum() == pytest.approx(DIMER_E, rel=5e-14)


def test_clusters_match_reference_scalar_opt(ref):
    # the reference's ScalarOpt plays the oracle of test_kernels.py:88-100
    # (energy rel 1e-12, forces abs 1e-10) on the reference-generated clusters,
    # both species tables (m=1 and lam3 != 0 in the mixed one)
    K = ref.kernels
    for fr, table, _ in golden_clusters():
        st = _free_frame(ref, fr.positions, fr.species)
        rtab = ref.paramfile.parse_params(B.serialize_params(table))
        nl = ref.neighbor.build_neighbor_list(st, rtab.r_cut, skin=0.3)
        want = K.compute(st, nl, rtab, K.make_variant("ScalarOpt"))
        got = K.compute(st, nl, rtab, K.make_variant("B200"))
        assert got.potential_energy == pytest.approx(want.potential_energy, rel=1e-12)
        assert np.max(np.abs(got.forces - want.forces)) < 1e-10
        assert got.per_atom_energy.sum() == pytest.approx(want.potential_energy, rel=1e-12)
        # the reference's own objects straight into this package's compute()
        mine = B.compute(st, nl, rtab, K.make_variant("VecI", "native"))
        assert np.max(np.abs(mine.forces - want.forces)) < 1e-10


def _packed_row_lengths(st, r_cut):
    d = st.positions[:, None, :] - st.positions[None, :, :]
    for ax in range(3):
        if st.box.periodic[ax]:
            L = st.box.lengths[ax]
            d[..., ax] -= L * np.round(d[..., ax] / L)
    r = np.sqrt((d ** 2).sum(-1))
    np.fill_diagonal(r, np.inf)
    return (r < r_cut).sum(1)


def test_visit_counters_and_lanes_follow_reference_contract(ref):
    # test_kernels.py:218-249 with the reference's variants on the B200 kernel
    K = ref.kernels
    table = ref.paramfile.builtin_params("C")
    fr, _, _ = golden_clusters()[3]
    st = _free_frame(ref, fr.positions, np.zeros(len(fr.positions), np.int64))
    nl = ref.neighbor.build_neighbor_list(st, table.r_cut, skin=0.3)
    nsq = int((_packed_row_lengths(st, table.r_cut).astype(np.int64) ** 2).sum())
    r_ref = B.compute(st, nl, table, K.make_variant("Reference"))
    r_opt = B.compute(st, nl, table, K.make_variant("ScalarOpt"))
    assert r_ref.stats["zeta_visits"] == 2 * nsq
    assert r_opt.stats["zeta_visits"] == nsq
    for v in (K.make_variant("VecJ", "native"), K.make_variant("VecI", "emulated", 4),
              K.make_variant("B200")):
        res = B.compute(st, nl, table, v)
        assert res.stats["zeta_visits"] == nsq
        assert res.stats["gathers"] > 0
        assert 0.0 < res.lane_utilization <= 1.0
    assert r_opt.lane_utilization is None and r_opt.stats["gathers"] == 0
    assert r_ref.lane_utilization is None
    rec = B.count_flops_and_visits(st, nl, table, K.make_variant("Reference"))
    assert rec["zeta_visits"] == 2 * nsq and rec["gathers"] == 0
    assert rec["lane_utilization"] is None


def _si512(ref):
    g = load_golden("si512")
    st = ref.system.SimulationState(
        g["positions"].copy(), ref.system.SimulationBox(g["lengths"], tuple(g["periodic"])),
        species=g["species"], masses=g["masses"], symbols=("Si",),
        velocities=g["velocities"].copy())
    return g, st, ref.paramfile.parse_params(str(g["table"]))


@pytest.mark.parametrize("precision", ["double", "single"])
def test_reference_run_nve_on_b200(ref, precision):
    # the reference's ForceField + velocity_verlet_step + run_nve, forces from
    # the B200 ABI: the golden ScalarOpt trajectory (100 steps, 1 fs)
    g, st, table = _si512(ref)
    v = ref.kernels.make_variant("B200", precision=precision)
    rec = ref.system.run_nve(st, table, ref.system.RunConfig(dt=1.0, steps=100, variant=v,
                                                             skin=0.3))
    assert rec["rebuilds"] == int(g["nve_rebuilds"])
    tol = 1e-9 if precision == "double" else 2e-5
    scale = abs(g["nve_total"][0])
    assert np.max(np.abs(rec["total"] - g["nve_total"])) <= tol * scale
    assert np.max(np.abs(rec["potential"] - g["nve_potential"])) <= tol * scale
    # sum_i F_i = 0: exact up to fp64 round-off; the mixed mode's fp32 pieces leave ~1e-6
    assert np.max(rec["force_sum_max"]) < (1e-9 if precision == "double" else 1e-4)


def test_reference_verification_suite_on_b200(ref):
    g, st, table = _si512(ref)
    rep = ref.verify.run_verification(st, table, variant=ref.kernels.make_variant("B200"),
                                      conservation_steps=50, dt=0.5)
    names = {c["name"]: c["passed"] for c in rep["checks"]}
    assert rep["passed"], rep
    assert any(n.startswith("gradient") for n in names)
    assert any(n.startswith("nve") for n in names)


def test_reference_benchmark_and_cli_on_b200(ref, tmp_path, capsys):
    g, st, table = _si512(ref)
    K = ref.kernels
    rep = ref.bench.run_benchmark(st, table, [K.make_variant("ScalarOpt"),
                                              K.make_variant("B200")],
                                  steps=2, warmup=1, repeats=2)
    csv = rep.render("csv").splitlines()
    assert len(csv) == 3 and csv[2].split(",")[0] == "B200"
    b200 = rep.rows[1].as_dict() if hasattr(rep.rows[1], "as_dict") else vars(rep.rows[1])
    assert json.dumps(b200, default=str)
    assert ref.cli.main(["run", "--structure", "diamond:cells=2", "--steps", "10",
                         "--temperature", "300", "--variant", "b200"]) == 0
    out = capsys.readouterr().out
    assert "B200" in out
    assert ref.cli.main(["bench", "--structure", "diamond:cells=2", "--steps", "2",
                         "--repeats", "1", "--variant", "scalar,b200",
                         "--format", "csv"]) == 0
