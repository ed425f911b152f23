"""GPU parity: the sm_100a path against the reference (golden vectors) and the
CPU oracle on the same seeded inputs.

Bars (BASELINE north_star): neighbour lists bit-exact; fp64 energy/forces
within 1e-10 relative (energy: |dE|/|E|; forces: max|dF| / max|F|); mixed
precision max|dF| <= 1e-5 max|F|.
"""

import numpy as np
import pytest

import paper_1710_00882_b200 as B
from conftest import Frame, golden_clusters, golden_frame, load_golden
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.paramfile import builtin_params, parse_params

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-10
MIXED_TOL = 1e-5
MIXED_E_TOL = 1e-5
SCATTERS = ["atomic", "gather"]
PATHS = ["warp", "tile", "row"]


@pytest.fixture(params=PATHS)
def kernel_path(request):
    """Run the test on the warp-chunk kernel, on the general tile kernel and on
    the atom-per-lane row kernel (rows of <= 4 entries of one-species tables;
    the remaining rows -- and every row of a multi-species table -- stay on the
    warp-chunk kernel)."""
    from paper_1710_00882_b200 import _native
    ctx = _native.default_context(0)
    ctx.set_option(_native.OPT_TILE_KERNEL, request.param == "tile")
    ctx.set_option(_native.OPT_ROW_KERNEL, 2 if request.param == "row" else 0)
    yield request.param
    ctx.set_option(_native.OPT_TILE_KERNEL, 0)
    ctx.set_option(_native.OPT_ROW_KERNEL, 1)


def rel_f(a, b):
    return np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300)


def gpu_eval(fr, table, precision="double", scatter="atomic", skin=0.3):
    nl = B.build_neighbor_list(fr, table.r_cut, skin)
    return nl, B.compute(fr, nl, table, B.make_variant("B200", precision=precision,
                                                       scatter=scatter))


@pytest.mark.parametrize("name", ["dimer", "si512", "sic216", "disordered"])
def test_neighbor_list_bit_exact_vs_reference(name):
    g = load_golden(name)
    t = parse_params(str(g["table"]))
    nl = B.build_neighbor_list(golden_frame(g), t.r_cut, 0.3)
    assert np.array_equal(nl.offsets, g["offsets"])
    assert np.array_equal(nl.neighbors, g["neighbors"])


@pytest.mark.parametrize("frame", [0, 1, 2])
def test_neighbor_list_edge_frames(frame):
    g = load_golden("nl_frames")
    p = f"f{frame}_"
    fr = Frame(g[p + "positions"], (9.0, 9.0, 9.0), g[p + "periodic"])
    nl = B.build_neighbor_list(fr, 2.1, 0.3)
    assert np.array_equal(nl.offsets, g[p + "offsets"])
    assert np.array_equal(nl.neighbors, g[p + "neighbors"])


@pytest.mark.parametrize("scatter", SCATTERS)
@pytest.mark.parametrize("name", ["dimer", "si512", "sic216", "disordered"])
def test_fp64_matches_reference(name, scatter, kernel_path):
    g = load_golden(name)
    t = parse_params(str(g["table"]))
    _, r = gpu_eval(golden_frame(g), t, "double", scatter)
    e = float(g["energy"])
    assert abs(r.potential_energy - e) <= FP64_TOL * abs(e)
    assert rel_f(r.forces, g["forces"]) <= FP64_TOL
    assert np.abs(r.per_atom_energy - g["per_atom"]).max() <= FP64_TOL * np.abs(g["per_atom"]).max()
    assert r.stats["zeta_visits"] == int(g["zeta_visits"])


@pytest.mark.parametrize("live", [0, 1])
@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("name", ["si512", "sic216", "disordered"])
def test_live_repack_matches_reference(name, precision, live):
    """TB_OPT_LIVE_PACK forced off / on (rows cut to r < r_cut and re-chunked on
    the device before each evaluation): same results and counters."""
    from paper_1710_00882_b200 import _native
    g = load_golden(name)
    t = parse_params(str(g["table"]))
    ctx = _native.default_context(0)
    ctx.set_option(_native.OPT_LIVE_PACK, live)
    try:
        fr = golden_frame(g)
        nl, r = gpu_eval(fr, t, precision, "atomic")
        r2 = B.compute(fr, nl, t, B.make_variant("B200", precision=precision))  # second pass
    finally:
        ctx.set_option(_native.OPT_LIVE_PACK, 2)
    e = float(g["energy"])
    tol = FP64_TOL if precision == "double" else MIXED_TOL
    for res in (r, r2):
        assert abs(res.potential_energy - e) <= tol * abs(e)
        assert rel_f(res.forces, g["forces"]) <= tol
        assert res.stats["zeta_visits"] == int(g["zeta_visits"])


@pytest.mark.parametrize("name", ["si512", "sic216", "disordered"])
def test_mixed_matches_reference_fp64(name, kernel_path):
    g = load_golden(name)
    t = parse_params(str(g["table"]))
    _, r = gpu_eval(golden_frame(g), t, "single")
    assert rel_f(r.forces, g["forces"]) <= MIXED_TOL
    e = float(g["energy"])
    # the reference's own single mode is 1e-6..2e-6 off in energy
    assert abs(r.potential_energy - e) <= MIXED_E_TOL * abs(e)


def test_dimer_frozen_goldens():
    g = load_golden("dimer")
    t = parse_params(str(g["table"]))
    _, r = gpu_eval(golden_frame(g), t)
    assert r.potential_energy == pytest.approx(float(g["frozen_energy"]), rel=5e-14)
    assert r.forces[0, 0] == pytest.approx(float(g["frozen_f0x"]), rel=5e-13)
    assert np.all(r.forces[:, 1:] == 0.0)


def test_clusters_carbon_and_two_species(kernel_path):
    # free clusters incl. the synthetic table with m=1 and lam3 != 0
    for fr, table, row in golden_clusters():
        for scatter in SCATTERS:
            nl, r = gpu_eval(fr, table, "double", scatter)
            assert np.array_equal(nl.neighbors, row["neighbors"])
            e = float(row["energy"])
            assert abs(r.potential_energy - e) <= FP64_TOL * abs(e)
            assert rel_f(r.forces, row["forces"]) <= FP64_TOL
            assert r.stats["zeta_visits"] == int(row["zeta_visits"])
        _, rs = gpu_eval(fr, table, "single")
        assert rel_f(rs.forces, row["forces"]) <= MIXED_TOL


def test_virial_matches_oracle_and_strain_fd(oracle_mod, kernel_path):
    g = load_golden("si512")
    t = parse_params(str(g["table"]))
    fr = golden_frame(g)
    _, r = gpu_eval(fr, t)
    o = oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic,
                           g["offsets"], g["neighbors"], t)
    assert np.abs(r.virial - o["virial"]).max() <= 1e-10 * np.abs(o["virial"]).max()
    assert np.allclose(r.virial[:3], g["virial_fd_diag"], rtol=1e-7, atol=1e-6)


def _config(idx, small=True):
    st, tname = structures.config(idx, small=small)
    return st, builtin_params(tname)


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_configs_vs_oracle(oracle_mod, idx, precision, kernel_path):
    st, t = _config(idx)
    nl, r = gpu_eval(st, t, precision)
    off, nb = oracle_mod.build_neighbor_list(st.positions, st.box.lengths, st.box.periodic,
                                             t.r_cut, 0.3, threads=8)
    assert np.array_equal(nl.offsets, off) and np.array_equal(nl.neighbors, nb)
    o = oracle_mod.compute(st.positions, st.species, st.box.lengths, st.box.periodic, off, nb, t,
                           threads=8)
    tol = FP64_TOL if precision == "double" else MIXED_TOL
    assert rel_f(r.forces, o["forces"]) <= tol
    etol = FP64_TOL if precision == "double" else MIXED_E_TOL
    assert abs(r.potential_energy - o["energy"]) <= etol * abs(o["energy"])
    assert r.stats["zeta_visits"] == o["zeta_visits"]
    if precision == "double":
        assert np.abs(r.virial - o["virial"]).max() <= 1e-9 * np.abs(o["virial"]).max()


@pytest.mark.parametrize("shift", ["wrapped", "unwrapped"])
def test_list_with_unwrapped_coordinates(oracle_mod, shift):
    # the list scan takes each candidate's minimum image from its stencil cell
    # only for coordinates inside [0, L]; images of unwrapped input (atoms
    # several box lengths away) must still follow d - L*rint(d/L)
    st, t = _config(2)
    pos = st.positions.copy()
    if shift == "unwrapped":
        rng = np.random.default_rng(9)
        pos += rng.integers(-2, 3, size=pos.shape) * st.box.lengths
    fr = Frame(pos, st.box.lengths, st.box.periodic, st.species)
    nl = B.build_neighbor_list(fr, t.r_cut, 0.3)
    off, nb = oracle_mod.build_neighbor_list(pos, st.box.lengths, st.box.periodic, t.r_cut, 0.3,
                                             threads=8)
    assert np.array_equal(nl.offsets, off) and np.array_equal(nl.neighbors, nb)


def test_total_force_vanishes_and_gather_deterministic(kernel_path):
    st, t = _config(4)
    nl = B.build_neighbor_list(st, t.r_cut, 0.3)
    v = B.make_variant("B200", scatter="gather")
    a = B.compute(st, nl, t, v)
    b = B.compute(st, nl, t, v)
    assert a.forces.tobytes() == b.forces.tobytes()
    assert a.potential_energy == b.potential_energy
    assert np.abs(a.forces.sum(axis=0)).max() < 1e-12 * st.natoms * max(1, np.abs(a.forces).max())


def test_errors_map_to_reference_exceptions(kernel_path):
    t = builtin_params("C")
    fr = Frame([[0.0, 0, 0], [1.5, 0, 0]], (10, 10, 10), (False,) * 3)
    nl = B.build_neighbor_list(fr, t.r_cut, 0.3)
    fr.positions[1, 0] = np.nan
    with pytest.raises(B.InputError, match="non-finite"):
        B.compute(fr, nl, t)
    fr.positions[1, 0] = 1.5
    fr.species = np.array([0, 1])
    with pytest.raises(B.ConfigurationError, match="species index"):
        B.compute(fr, nl, t)
    fr2 = Frame([[0.0, 0, 0], [1e-9, 0, 0]], (10, 10, 10), (False,) * 3)
    nl2 = B.build_neighbor_list(fr2, t.r_cut, 0.3)
    with pytest.raises(B.InputError, match="coincident"):
        B.compute(fr2, nl2, t)
    with pytest.raises(B.ConfigurationError, match="skin"):
        B.build_neighbor_list(fr2, t.r_cut, -0.1)
    box = Frame([[0.5, 1.0, 1.0], [2.0, 1.0, 1.0]], (4.0, 9.0, 9.0), (True, True, True))
    with pytest.raises(B.ConfigurationError, match="twice the build cutoff"):
        B.build_neighbor_list(box, 2.1, 0.3)


def test_lone_and_distant_atoms(kernel_path):
    t = builtin_params("C")
    for pos in ([[0.0, 0, 0]], [[0.0, 0, 0], [5.0, 0, 0]]):
        fr = Frame(pos, (20, 20, 20), (False,) * 3)
        _, r = gpu_eval(fr, t)
        assert r.potential_energy == 0.0
        assert np.all(r.forces == 0.0)


def test_needs_rebuild_threshold():
    t = builtin_params("C")
    fr = Frame([[0, 0, 0], [1.5, 0, 0], [3.0, 0, 0]], (20, 20, 20), (False,) * 3)
    nl = B.build_neighbor_list(fr, 2.1, 0.3)
    assert not B.needs_rebuild(fr, nl)
    fr.positions[1, 1] += 0.5 * 0.3 - 1e-9
    assert not B.needs_rebuild(fr, nl)
    fr.positions[1, 1] += 2e-9
    assert B.needs_rebuild(fr, nl)
    p = Frame([[0.2, 5, 5]], (10, 10, 10), (True, False, False))
    nlp = B.build_neighbor_list(p, 2.1, 0.3)
    p.positions[0, 0] = 9.95
    assert B.needs_rebuild(p, nlp)


@pytest.mark.parametrize("precision", ["double", "single"])
def test_pinned_host_buffers_match_pageable(precision):
    """compute() with pinned host arrays (finalize writes forces / results
    through their device aliases, per-atom energies on the side stream) gives
    the same result as pageable arrays, repeatedly, including after an error."""
    import torch
    g = load_golden("si512")
    t = parse_params(str(g["table"]))
    fr = golden_frame(g)
    nl = B.build_neighbor_list(fr, t.r_cut, 0.3)
    var = B.make_variant("B200", precision=precision)
    ref = B.compute(fr, nl, t, var)
    n = len(fr.positions)
    pos = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    pos[:] = fr.positions
    sp = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
    sp[:] = np.asarray(fr.species)
    pf = Frame(pos, fr.box.lengths, fr.box.periodic)
    pf.species = sp
    out = B.ForceEnergyResult(torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy(), 0.0,
                              torch.empty(n, dtype=torch.float64).pin_memory().numpy(), {})
    for _ in range(3):
        r = B.compute(pf, nl, t, var, out=out)
        assert np.array_equal(r.forces, ref.forces) or rel_f(r.forces, ref.forces) < 1e-12
        assert abs(r.potential_energy - ref.potential_energy) <= 1e-12 * abs(ref.potential_energy)
        assert np.allclose(r.per_atom_energy, ref.per_atom_energy, rtol=0, atol=1e-12)
        assert np.allclose(r.virial, ref.virial, rtol=1e-12, atol=1e-12)
        assert r.stats["zeta_visits"] == ref.stats["zeta_visits"]
    pos[3, 1] = np.nan  # an error reported through the pinned result block
    with pytest.raises(B.InputError, match="non-finite"):
        B.compute(pf, nl, t, var, out=out)
    pos[3, 1] = fr.positions[3, 1]
    r = B.compute(pf, nl, t, var, out=out)  # flags were reset: clean again
    assert abs(r.potential_energy - ref.potential_energy) <= 1e-12 * abs(ref.potential_energy)


def _si_table(eta=None, beta=None):
    """Si(C) (BASELINE) with eta / beta replaced (17-token line: m gamma lam3 c d
    h eta beta lam2 B R D lam1 A)."""
    tok = "Si Si Si 3 1.0 0.0 100390 16.217 -0.59825 0.78734 1.1e-6 1.7322 471.18 2.85 0.15 2.4799 1830.8".split()
    if eta is not None:
        tok[9] = repr(eta)
    if beta is not None:
        tok[10] = repr(beta)
    return parse_params(" ".join(tok) + "\n")


def _oracle_free(oracle_mod, pos, table):
    fr = Frame(pos, np.ptp(pos, axis=0) + 8.0, (False, False, False))
    fr.positions = fr.positions - fr.positions.min(axis=0) + 4.0
    off, nb = oracle_mod.build_neighbor_list(fr.positions, fr.box.lengths, fr.box.periodic,
                                             table.r_cut, 0.3)
    return fr, oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic,
                                  off, nb, table)


@pytest.mark.parametrize("case", ["tiny_zeta", "huge_u", "moderate"])
def test_bond_order_extreme_regimes(oracle_mod, case, kernel_path):
    # eta log(beta zeta) below -708 (u underflows: b = 1) and above the
    # log1p(u) = x switch (u beyond 1e15): the kernel's branch-free bond order
    # against the oracle's libm pow (potential.py:202-215), fp64 1e-10
    if case == "tiny_zeta":
        # Si(B)-like eta = 22.956, beta = 0.33675; the third atom sits 1e-7 A
        # inside the cutoff: f_C ~ 3e-14, zeta ~ 1e-13, x ~ -760
        table = _si_table(22.956, 0.33675)
        d = 3.0 - 1e-7
        pos = np.array([[0.0, 0, 0], [2.35, 0, 0], [d * np.cos(1.9), d * np.sin(1.9), 0]])
    elif case == "huge_u":
        # beta = 3, eta = 22.956 on a compact cluster: x = eta log(3 zeta) >> 36
        table = _si_table(22.956, 3.0)
        rng = np.random.default_rng(11)
        pos = np.array([[0.0, 0, 0], [2.3, 0.1, 0], [0.2, 2.35, 0.1], [-0.1, 0.3, 2.3],
                        [1.6, 1.7, 1.5], [-1.6, 1.2, -1.0]]) + rng.normal(0, 0.02, (6, 3))
    else:
        table = _si_table(3.0, 0.05)
        pos = structures.gen_diamond(1).positions[:8] * 1.0
    fr, ref = _oracle_free(oracle_mod, pos, table)
    nl, res = gpu_eval(fr, table)
    assert np.isfinite(res.forces).all() and np.isfinite(res.potential_energy)
    assert abs(res.potential_energy - ref["energy"]) <= FP64_TOL * abs(ref["energy"])
    assert rel_f(res.forces, ref["forces"]) <= FP64_TOL


@pytest.mark.parametrize("precision", ["double", "single"])
def test_collinear_bonds_cos_pm1(oracle_mod, precision, kernel_path):
    # cos(theta) = -1 (a straight chain) and +1 (j and k on the same ray): the
    # warp kernel does not clamp cos to [-1, 1] (|e_a . e_b| exceeds 1 by a few
    # ulp at most, g is smooth there); parity with the clamping oracle
    # (potential.py:256)
    table = builtin_params("Si")
    chain = np.array([[2.35 * q, 0.0, 0.0] for q in range(6)])
    ray = np.array([[0.0, 0, 0], [2.2, 0, 0], [2.9, 0, 0], [0.0, 2.3, 0.0], [0.0, 2.9, 0.0]])
    # (mixed: these near-equilibrium chains have net forces ~30x smaller than
    # the pair terms that cancel into them, so the fp32 terms' relative error
    # shows up ~30x amplified against max|F|)
    tol = FP64_TOL if precision == "double" else 30 * MIXED_TOL
    for pos in (chain, ray):
        fr, ref = _oracle_free(oracle_mod, pos, table)
        nl, res = gpu_eval(fr, table, precision=precision)
        assert abs(res.potential_energy - ref["energy"]) <= tol * abs(ref["energy"])
        assert rel_f(res.forces, ref["forces"]) <= tol


def test_out_of_range_tables_are_refused():
    # the fp64 kernel's exp / log domains: refused loudly, never rounded away
    with pytest.raises(B.ConfigurationError, match="exp range"):
        t = _si_table()
        t2 = parse_params(B.serialize_params(t).replace("2.4799", "400.0"))
        B.compute(*_tiny_frame(), t2)
    # a refused table leaves the previous one in place
    fr, nl = _tiny_frame()
    good = _si_table()
    want = B.compute(fr, nl, good).potential_energy
    with pytest.raises(B.ConfigurationError, match="beta"):
        B.compute(*_tiny_frame(), _si_table(beta=1e-300))
    from paper_1710_00882_b200 import _native
    ctx = _native.default_context(0)
    ctx._table_key = id(good)  # as if `good` were still the uploaded table
    assert B.compute(fr, nl, good).potential_energy == want


def _tiny_frame():
    fr = Frame([[0.0, 0, 0], [2.35, 0, 0]], [10.0, 10.0, 10.0], (False, False, False))
    nl = B.build_neighbor_list(fr, 3.0, 0.3)
    return fr, nl


@pytest.mark.parametrize("margin", [1, 50])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_margin_repack_tracks_moving_atoms(oracle_mod, precision, margin):
    """TB_OPT_REPACK_MARGIN (rows cut at r_cut + delta, re-cut only after a
    delta/2 drift, decided on the device): a sequence of evaluations at moving
    positions -- small moves that keep the repack, larger ones that force it --
    equals the oracle at every step, and equals the exact (margin 0) repack."""
    from paper_1710_00882_b200 import _native
    st, tname = structures.config(3, small=True)
    t = builtin_params(tname)
    ctx = _native.default_context(0)
    rng = np.random.default_rng(5)
    fr = Frame(st.positions.copy(), st.box.lengths, st.box.periodic, st.species)
    nl = B.build_neighbor_list(fr, t.r_cut, 0.3)
    nl0 = B.build_neighbor_list(fr, t.r_cut, 0.3)  # the exact-repack twin
    var = B.make_variant("B200", precision=precision)
    tol = FP64_TOL if precision == "double" else MIXED_TOL
    ctx.set_option(_native.OPT_REPACK_MARGIN, margin)
    moves = [0.0, 0.0, 0.0002, 0.004, 0.004, 0.03, 0.002, 0.05, 0.001]  # A per component (sigma)
    base = st.positions.copy()
    for k, s in enumerate(moves):
        base = base + rng.normal(0.0, s, base.shape)
        fr.positions = np.remainder(base, st.box.lengths)
        res = B.compute(fr, nl, t, var)
        ctx.set_option(_native.OPT_REPACK_MARGIN, 0)
        try:
            exact = B.compute(fr, nl0, t, var)
        finally:
            ctx.set_option(_native.OPT_REPACK_MARGIN, margin)
        ref = oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic,
                                 nl.offsets, nl.neighbors, t)
        assert abs(res.potential_energy - ref["energy"]) <= tol * abs(ref["energy"]), k
        assert rel_f(res.forces, ref["forces"]) <= tol, k
        # fp64: the same terms in the same order (dead lanes add exact zeros);
        # mixed: the chunk shapes differ, so the fp32 partial sums round apart
        same = 1e-12 if precision == "double" else MIXED_TOL
        assert abs(res.potential_energy - exact.potential_energy) <= same * abs(ref["energy"])
        assert res.stats["zeta_visits"] == exact.stats["zeta_visits"]
    ctx.set_option(_native.OPT_REPACK_MARGIN, 1)


def _many_species_table(S):
    """A synthetic S-species table (not a published set): carbon-like values
    varied by the species of each slot, m = 1 with lam3 != 0 on some triples."""
    from paper_1710_00882_b200.potential import ParamTable, TersoffParams
    ent = {}
    for i in range(S):
        for j in range(S):
            for k in range(S):
                m = 1 if (i + k) % 3 == 0 else 3
                ent[(i, j, k)] = TersoffParams(
                    m=m, gamma=1.0 + 0.05 * k, lam3=0.6 if m == 1 else 0.0,
                    c=38049.0 * (1.0 - 0.08 * i), d=4.3484 + 0.3 * j, h=-0.57058 + 0.04 * k,
                    eta=0.72751 + 0.05 * i, beta=1.5724e-7 * (1.0 + 0.5 * (i + j)),
                    lam2=2.2119 - 0.05 * j, B=346.74 * (1.0 + 0.05 * i),
                    R=1.95 + 0.06 * (i + k), D=0.15 + 0.01 * j,
                    lam1=3.4879 - 0.05 * i, A=1393.6 * (1.0 + 0.03 * j))
    return ParamTable(tuple(f"X{q}" for q in range(S)), ent)


@pytest.mark.parametrize("S", [5, 7])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_more_than_four_species(oracle_mod, S, precision):
    # the reference's ParamTable takes any species count (potential.py:94-110):
    # S > 4 runs the tile kernel with a runtime species count (tables in HBM)
    table = _many_species_table(S)
    rng = np.random.default_rng(40 + S)
    # periodic random packing (min separation 1.3 A) with all species present
    n, L = 300, 14.0
    pos = rng.uniform(0, L, (1, 3))
    while len(pos) < n:
        c = rng.uniform(0, L, 3)
        d = pos - c
        d -= L * np.round(d / L)
        if (d * d).sum(1).min() > 1.3 ** 2:
            pos = np.vstack([pos, c])
    species = rng.integers(0, S, n)
    fr = Frame(pos, [L, L, L], (True, True, True), species)
    nl, res = gpu_eval(fr, table, precision=precision)
    off, nb = oracle_mod.build_neighbor_list(fr.positions, fr.box.lengths, fr.box.periodic,
                                             table.r_cut, 0.3)
    assert np.array_equal(nl.offsets, off) and np.array_equal(nl.neighbors, nb)
    ref = oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic, off, nb,
                             table)
    tol = FP64_TOL if precision == "double" else MIXED_TOL
    assert abs(res.potential_energy - ref["energy"]) <= tol * abs(ref["energy"])
    assert rel_f(res.forces, ref["forces"]) <= tol
    assert np.abs(res.virial - ref["virial"]).max() <= 1e3 * tol * np.abs(ref["virial"]).max()
    assert res.stats["zeta_visits"] == int(ref["zeta_visits"])
    with pytest.raises(B.ConfigurationError, match="species"):
        bad = fr.species.copy()
        bad[0] = S
        B.compute(Frame(pos, [L, L, L], (True, True, True), bad), nl, table)


def test_neighbor_list_pairs_at_the_cutoff(oracle_mod):
    """The list scan decides candidates in fp32 unless their r^2 is within a
    band of the build cutoff, where the exact fp64 test runs (k_nl_atoms,
    TB_NL_F32).  1000 isolated dimers at bc + delta, delta from 0 and +-1 ulp up
    to +-1e-2 A on both sides of the band, random orientations, all-periodic
    box of 24 cells per axis: the pair set must equal the oracle's."""
    rng = np.random.default_rng(12345)
    r_cut, skin = 3.0, 0.3
    bc = r_cut + skin
    L = 80.0
    sites = np.stack(np.meshgrid(*[np.arange(10) * 8.0 + 2.0] * 3, indexing="ij"), -1).reshape(-1, 3)
    deltas = np.array([0.0] + [s * m for m in (np.spacing(bc), 4 * np.spacing(bc), 1e-14, 1e-12,
                                               1e-10, 1e-8, 1e-6, 1e-5, 1e-4, 2e-4, 3e-4, 5e-4,
                                               1e-3, 1e-2) for s in (1.0, -1.0)])
    u = rng.normal(size=(len(sites), 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    d = bc + deltas[np.arange(len(sites)) % len(deltas)]
    a = sites + rng.uniform(0.0, 1.0, size=sites.shape)
    pos = np.concatenate([a, a + u * d[:, None]])
    pos %= L  # dimers across the periodic faces too
    fr = Frame(pos, (L, L, L), (True, True, True))
    nl = B.build_neighbor_list(fr, r_cut, skin)
    off, nb = oracle_mod.build_neighbor_list(fr.positions, fr.box.lengths, fr.box.periodic,
                                             r_cut, skin)
    assert np.array_equal(nl.offsets, off) and np.array_equal(nl.neighbors, nb)
    n_in = int(np.diff(off).sum()) // 2
    assert 300 < n_in < 700  # both sides of the cutoff are populated
