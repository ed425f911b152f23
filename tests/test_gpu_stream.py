"""Streamed tb_compute (pinned host buffers, TB_OPT_STREAM_RANGE; csrc/tb_stream.cuh):
ranges of positions in, stages of warp chunks, ranges of forces out.  The
chunks and their arithmetic are those of the unstreamed call, so per-atom
energies are bit-identical and forces / energy differ only by the order of the
fp64 atomic adds; both are checked against the CPU oracle too."""

import numpy as np
import pytest

import paper_1710_00882_b200 as B
from conftest import Frame
from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.paramfile import builtin_params

pytestmark = pytest.mark.gpu


def pinned(shape):
    import torch
    return torch.empty(shape, dtype=torch.float64).pin_memory().numpy()


@pytest.fixture
def stream_range():
    ctx = _native.default_context(0)

    def set_range(r):
        ctx.set_option(_native.OPT_STREAM_RANGE, r)
    # the streamed stages run the warp-chunk kernel: compare like with like
    ctx.set_option(_native.OPT_ROW_KERNEL, 0)
    yield set_range
    ctx.set_option(_native.OPT_STREAM_RANGE, 131072)
    ctx.set_option(_native.OPT_ROW_KERNEL, 1)


class HostState:
    def __init__(self, positions, species, box):
        self.positions, self.species, self.box = positions, species, box


def evaluate(st, nl, table, precision, pin=True):
    n = st.positions.shape[0]
    pos = pinned((n, 3)) if pin else np.empty((n, 3))
    pos[:] = st.positions
    hs = HostState(pos, st.species, st.box)
    out = B.ForceEnergyResult(pinned((n, 3)), 0.0, pinned(n), {})
    out.forces[:] = np.nan
    out.per_atom_energy[:] = np.nan
    res = B.compute(hs, nl, table, B.make_variant("B200", precision=precision), out=out)
    return (res.forces.copy(), res.potential_energy, res.per_atom_energy.copy(),
            dict(res.stats), res.virial.copy())


def make_state(cells, sigma, seed, shuffle=False, hole=False):
    st = structures.displace(structures.gen_diamond(cells), sigma, seed)
    pos, L, per = st.positions, st.box.lengths, st.box.periodic
    if hole:
        # carve out the surroundings of atom 100: it keeps an empty row and the
        # atoms around the hole get rows of other lengths
        d = pos - pos[100]
        d -= L * np.rint(d / L)
        keep = np.linalg.norm(d, axis=1) > 3.9
        keep[100] = True
        pos = pos[keep]
    if shuffle:
        pos = pos[np.random.default_rng(seed).permutation(pos.shape[0])]
    return Frame(pos, L, per)


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("case", ["lattice", "shuffled", "hole"])
def test_streamed_equals_unstreamed(case, precision, stream_range, oracle_mod):
    st = make_state((8, 8, 8), 0.1, 7, shuffle=case == "shuffled", hole=case == "hole")
    table = builtin_params("Si")
    n = st.positions.shape[0]
    nl = B.build_neighbor_list(st, table.r_cut, 0.3)
    stream_range(0)
    f0, e0, pa0, st0, w0 = evaluate(st, nl, table, precision)
    stream_range(96)  # n >= 8 * 96: K = ceil(n / max(96, n / 32)) ranges
    f1, e1, pa1, st1, w1 = evaluate(st, nl, table, precision)
    f2, e2, pa2, st2, w2 = evaluate(st, nl, table, precision)  # cached plan
    fmax = np.abs(f0).max()
    for f, e, pa, s_, w in ((f1, e1, pa1, st1, w1), (f2, e2, pa2, st2, w2)):
        assert np.isfinite(f).all() and np.isfinite(pa).all()
        assert np.array_equal(pa, pa0)          # one writer per atom: same bits
        assert np.abs(f - f0).max() <= 1e-12 * fmax
        assert abs(e - e0) <= 1e-12 * abs(e0)
        assert np.abs(w - w0).max() <= 1e-11 * np.abs(w0).max()
        assert s_ == st0
    if case == "hole":
        assert (np.diff(nl.offsets) == 0).any()
    # and against the oracle (fp64 1e-10, mixed 1e-5)
    O = oracle_mod
    ref = O.compute(st.positions, st.species, st.box.lengths, st.box.periodic, nl.offsets,
                    nl.neighbors, table)
    tol = 1e-10 if precision == "double" else 1e-5
    assert np.abs(f1 - ref["forces"]).max() <= tol * np.abs(ref["forces"]).max()
    assert abs(e1 - ref["energy"]) <= tol * abs(ref["energy"])


def test_streamed_after_list_rebuild(stream_range):
    """The stage plan follows the list: a rebuilt list gets a new plan."""
    table = builtin_params("Si")
    st = make_state((8, 8, 8), 0.1, 11)
    nl = B.build_neighbor_list(st, table.r_cut, 0.3)
    stream_range(128)
    evaluate(st, nl, table, "double")
    st2 = make_state((8, 8, 8), 0.12, 12)
    nl2 = B.build_neighbor_list(st2, table.r_cut, 0.3)
    f1, e1, pa1, _, _ = evaluate(st2, nl2, table, "double")
    stream_range(0)
    f0, e0, pa0, _, _ = evaluate(st2, nl2, table, "double")
    assert np.array_equal(pa1, pa0)
    assert np.abs(f1 - f0).max() <= 1e-12 * np.abs(f0).max()


def test_pageable_buffers_take_the_plain_path(stream_range):
    table = builtin_params("Si")
    st = make_state((6, 6, 6), 0.1, 3)
    nl = B.build_neighbor_list(st, table.r_cut, 0.3)
    stream_range(64)
    res = B.compute(st, nl, table, B.make_variant("B200"))
    f1, e1, pa1, _, _ = evaluate(st, nl, table, "double")
    assert np.array_equal(res.per_atom_energy, pa1)
    assert np.abs(res.forces - f1).max() <= 1e-12 * np.abs(f1).max()
