"""Device-resident NVE (md.run_nve: tb_md_run graph loop / tb_md_step) and
md.ForceField as a drop-in force provider, against the reference's own NVE
run (golden) and the oracle's.  North-star bar: energy drift over 1000 NVE steps comparable to
the reference (fp64 and mixed)."""

import numpy as np
import pytest

import paper_1710_00882_b200 as B
from conftest import load_golden
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.paramfile import builtin_params, parse_params
from paper_1710_00882_b200.md import ForceField, RunConfig, run_nve
from paper_1710_00882_b200.state import ACCEL, SimulationBox, SimulationState


def run_nve_device(state, params, cfg, precision="double", scatter="atomic", record_every=1,
                   loop="auto"):
    cfg.variant = B.make_variant("B200", precision=precision, scatter=scatter)
    cfg.record_every = record_every
    return run_nve(state, params, cfg, loop=loop)

pytestmark = pytest.mark.gpu


def drift(total):
    # cli.py:145-157: max |E_tot - E_tot(0)| / |E_tot(0)|
    return float(np.max(np.abs(total - total[0])) / abs(total[0]))


def si512_state():
    g = load_golden("si512")
    st = SimulationState(g["positions"], SimulationBox(g["lengths"], tuple(g["periodic"])),
                         species=g["species"], masses=g["masses"], symbols=("Si",),
                         velocities=g["velocities"])
    return g, st, parse_params(str(g["table"]))


@pytest.mark.parametrize("loop", ["graph", "step"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_device_nve_matches_reference_run(precision, loop):
    g, st, t = si512_state()
    rec = run_nve_device(st, t, RunConfig(dt=1.0, steps=100, skin=0.3), precision=precision,
                         loop=loop)
    assert rec["loop"] == loop
    ref_total = g["nve_total"]
    assert rec["rebuilds"] == int(g["nve_rebuilds"])
    scale = abs(ref_total[0])
    tol = 1e-9 if precision == "double" else 2e-5
    assert np.max(np.abs(rec["total"] - ref_total)) <= tol * scale
    assert np.max(np.abs(rec["potential"] - g["nve_potential"])) <= tol * scale
    ptol = 1e-7 if precision == "double" else 1e-3
    assert np.abs(rec["positions"] - g["nve_final_positions"]).max() <= ptol
    assert drift(rec["total"]) < 5 * max(drift(ref_total), 1e-6)


def test_force_field_drives_host_verlet_like_reference():
    # ForceField as the forces_fn of a host velocity-Verlet loop (the
    # reference's velocity_verlet_step shape, system.py:355-380): the golden
    # trajectory of the reference's run_nve over 30 steps
    g, st, t = si512_state()
    ff = ForceField(t, B.make_variant("ScalarOpt"), skin=0.3)
    m = st.atom_masses[:, None]
    half = 0.5 * 1.0 * ACCEL
    res = ff(st)
    total = [res.potential_energy + B.kinetic_energy(st)]
    for _ in range(30):
        st.velocities += half * res.forces / m
        st.positions += 1.0 * st.velocities
        st.box.wrap(st.positions)
        res = ff(st)
        st.velocities += half * res.forces / m
        total.append(res.potential_energy + B.kinetic_energy(st))
    ref = g["nve_total"][:31]
    assert np.max(np.abs(np.array(total) - ref)) <= 1e-9 * abs(ref[0])
    assert ff.evaluations == 31 and ff.rebuilds >= 2
    assert isinstance(res.forces, np.ndarray)


def test_force_field_device_state_and_nonfinite():
    import torch
    g, st, t = si512_state()
    ff = ForceField(t, skin=0.3)
    dev = SimulationState(st.positions, st.box, species=st.species, masses=st.masses)
    dev.positions = torch.from_numpy(st.positions).cuda()
    dev.species = torch.from_numpy(st.species.astype(np.int32)).cuda()
    r_dev = ff(dev)
    r_host = ForceField(t, skin=0.3)(st)
    assert r_dev.forces.is_cuda
    assert np.abs(r_dev.forces.cpu().numpy() - r_host.forces).max() < 1e-12
    bad = st.copy()
    bad.positions[3, 0] = np.nan
    with pytest.raises(B.InputError):
        ForceField(t)(bad)


def test_run_nve_dumps_xyz_frames(tmp_path):
    g, st, t = si512_state()
    path = tmp_path / "traj.xyz"
    cfg = RunConfig(dt=1.0, steps=20, skin=0.3, dump_every=10, dump_path=str(path))
    rec = run_nve(st, t, cfg)
    frames = B.read_xyz(path)
    assert len(frames) == 3 and rec["loop"] == "graph"
    assert np.abs(frames[-1][1] - st.positions).max() < 1e-9
    ref = g["nve_total"][:21]
    assert np.max(np.abs(rec["total"] - ref)) <= 1e-9 * abs(ref[0])


@pytest.mark.parametrize("loop", ["graph", "step"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_1000_step_drift_comparable_to_reference(oracle_mod, precision, loop):
    # BASELINE config 2 protocol (skin 0.3, rebuild every 10 steps + trigger,
    # dt 1 fs, 1000 K) on 8^3 cells (4096 atoms); reference = the oracle's run
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=1.0, steps=1000, skin=0.3, rebuild_every=10)
    rec = run_nve_device(st.copy(), t, cfg, precision=precision, record_every=1, loop=loop)
    assert rec["loop"] == loop
    ref = oracle_mod.run_nve(st.positions, st.velocities, st.species, st.masses,
                             st.box.lengths, st.box.periodic, t, dt=1.0, steps=1000, skin=0.3,
                             threads=8, rebuild_every=10)
    d_gpu, d_ref = drift(rec["total"]), drift(ref["total"])
    assert np.isfinite(rec["total"]).all()
    # comparable: same order of magnitude (the trajectories decorrelate)
    assert d_gpu <= 3 * d_ref + 2e-6, (d_gpu, d_ref)
    if precision == "double":
        # early steps agree closely before chaos amplifies round-off
        assert np.max(np.abs(rec["total"][:50] - ref["total"][:50])) <= 1e-8 * abs(ref["total"][0])


def _run_both(st, t, cfg, **kw):
    a = run_nve_device(st.copy(), t, cfg, loop="graph", **kw)
    b = run_nve_device(st.copy(), t, cfg, loop="step", **kw)
    assert a["loop"] == "graph" and b["loop"] == "step"
    return a, b


@pytest.mark.parametrize("scatter", ["atomic", "gather"])
def test_graph_loop_matches_step_loop_si(scatter):
    # device-side rebuild decision + rebuild inside the graph == host-driven loop
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=1.0, steps=300, skin=0.3, rebuild_every=0)
    a, b = _run_both(st, t, cfg, scatter=scatter, record_every=1)
    assert a["rebuilds"] == b["rebuilds"] and a["rebuilds"] > 5
    scale = abs(b["total"][0])
    assert np.max(np.abs(a["total"] - b["total"])) <= 1e-9 * scale
    assert np.abs(a["positions"] - b["positions"]).max() <= 1e-7
    if scatter == "gather":
        # deterministic forces and a deterministic (radix-sorted) chunk plan
        c = run_nve_device(st.copy(), t, cfg, loop="graph", scatter=scatter, record_every=1)
        assert np.array_equal(c["positions"], a["positions"])


@pytest.mark.parametrize("precision", ["double", "single"])
def test_graph_loop_matches_step_loop_sic(precision):
    # two species: the species-pair compute filter is rebuilt on the device
    st, tname = structures.config(3, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=0.5, steps=200, skin=0.3, rebuild_every=10)
    a, b = _run_both(st, t, cfg, precision=precision, record_every=5)
    assert a["rebuilds"] == b["rebuilds"] >= 20
    scale = abs(b["total"][0])
    tol = 1e-9 if precision == "double" else 1e-5
    assert np.max(np.abs(a["total"] - b["total"])) <= tol * scale


def test_graph_loop_overflow_replay():
    # zero spare capacity: the first rebuild that grows the list overflows,
    # the run restarts from its entry state with regrown buffers
    from paper_1710_00882_b200 import _native
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=1.0, steps=200, skin=0.3)
    ctx = _native.default_context(0)
    ctx.set_option(_native.OPT_LIST_MARGIN, 0)
    try:
        a = run_nve_device(st.copy(), t, cfg, loop="graph", record_every=1)
    finally:
        ctx.set_option(_native.OPT_LIST_MARGIN, 25)
    b = run_nve_device(st.copy(), t, cfg, loop="step", record_every=1)
    assert a["rebuilds"] >= b["rebuilds"]
    assert np.max(np.abs(a["total"] - b["total"])) <= 1e-9 * abs(b["total"][0])


def test_graph_loop_free_axis_falls_back():
    g, st, t = si512_state()
    st.box = SimulationBox(st.box.lengths, (True, True, False))
    rec = run_nve_device(st, t, RunConfig(dt=1.0, steps=5, skin=0.3), loop="auto")
    assert rec["loop"] == "step"
    with pytest.raises(RuntimeError):
        run_nve_device(st, t, RunConfig(dt=1.0, steps=5, skin=0.3), loop="graph")


@pytest.mark.parametrize("precision", ["double", "single"])
def test_loose_list_matches_exact_list(precision):
    """tb_md_run with the loose list (skin + 0.3 A, rebuilt only for validity)
    and with the exact list rebuilt at every reference rebuild: same rebuild
    count and the same trajectory to round-off."""
    from paper_1710_00882_b200 import _native
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=1.0, steps=200, skin=0.3, rebuild_every=10)
    ctx = _native.default_context(0)
    ctx.set_option(_native.OPT_MD_LOOSE_SKIN, 0)
    try:
        exact = run_nve_device(st.copy(), t, cfg, precision=precision, loop="graph",
                               record_every=1)
    finally:
        ctx.set_option(_native.OPT_MD_LOOSE_SKIN, 30)
    loose = run_nve_device(st.copy(), t, cfg, precision=precision, loop="graph", record_every=1)
    assert loose["loop"] == exact["loop"] == "graph"
    assert loose["rebuilds"] == exact["rebuilds"] > 20
    scale = abs(exact["total"][0])
    tol = 1e-9 if precision == "double" else 1e-6
    assert np.max(np.abs(loose["total"] - exact["total"])) <= tol * scale
    assert np.abs(loose["positions"] - exact["positions"]).max() <= (1e-7 if precision == "double" else 1e-4)


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("loop", ["graph", "step"])
def test_row_kernel_md_matches_warp_kernel(loop, precision):
    """The atom-per-lane kernel (rows of <= 4 entries) inside the NVE loops --
    in the graph its bounds come from the device plan of the in-graph rebuild --
    against the same run on the warp-chunk kernel."""
    from paper_1710_00882_b200 import _native
    ctx = _native.default_context(0)
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    cfg = RunConfig(dt=1.0, steps=200, skin=0.3, rebuild_every=10)
    ctx.set_option(_native.OPT_ROW_KERNEL, 0)
    try:
        a = run_nve_device(st.copy(), t, cfg, precision=precision, loop=loop)
        ctx.set_option(_native.OPT_ROW_KERNEL, 2)
        b = run_nve_device(st.copy(), t, cfg, precision=precision, loop=loop)
    finally:
        ctx.set_option(_native.OPT_ROW_KERNEL, 1)
    assert a["loop"] == loop and b["loop"] == loop
    assert a["rebuilds"] == b["rebuilds"] and a["rebuilds"] >= 20
    scale = abs(a["total"][0])
    tol = 1e-9 if precision == "double" else 2e-5
    assert np.max(np.abs(a["total"] - b["total"])) <= tol * scale
    assert np.abs(a["positions"] - b["positions"]).max() <= (1e-7 if precision == "double" else 1e-3)
