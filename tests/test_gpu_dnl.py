"""Device-side neighbour-list rebuild (the builder inside the graph MD loop,
tb_nlist_rebuild_device) against the host-synchronised build: identical pair
sets and row order (neighbor.py:157-212), identical forces."""

import numpy as np
import pytest
import torch

from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.kernels import compute, make_variant
from paper_1710_00882_b200.neighbor import build_neighbor_list
from paper_1710_00882_b200.paramfile import builtin_params
from paper_1710_00882_b200.state import SimulationBox, SimulationState

pytestmark = pytest.mark.gpu


def _dev_state(st):
    class _S:
        pass
    s = _S()
    s.positions = torch.from_numpy(np.ascontiguousarray(st.positions)).cuda()
    s.species = torch.from_numpy(st.species.astype(np.int32)).cuda()
    s.box = st.box
    return s


def _moved(st, sigma, seed):
    st2 = st.copy()
    rng = np.random.default_rng(seed)
    st2.positions += rng.normal(scale=sigma, size=st2.positions.shape)
    st2.box.wrap(st2.positions)
    return st2


CASES = [(2, 0.08), (3, 0.05), (4, 0.1)]


@pytest.mark.parametrize("scatter", ["atomic", "gather"])
@pytest.mark.parametrize("cfg,sigma", CASES)
def test_device_rebuild_matches_host_build(cfg, sigma, scatter):
    st, tname = structures.config(cfg, small=True)
    t = builtin_params(tname)
    ctx = _native.default_context(0)
    ctx.set_table(t)
    d0 = _dev_state(st)
    nl = build_neighbor_list(d0, t.r_cut, 0.3)
    v = make_variant("B200", scatter=scatter)
    compute(d0, nl, t, v)  # species-pair filter for SiC built at first use
    st1 = _moved(st, sigma, 77)
    d1 = _dev_state(st1)
    nl.rebuild_on_device(d1.positions, d1.species, scatter)
    ref = build_neighbor_list(d1, t.r_cut, 0.3)
    assert np.array_equal(nl.offsets, ref.offsets)
    assert np.array_equal(nl.neighbors, ref.neighbors)
    assert nl.max_row == ref.max_row
    a = compute(d1, nl, t, v)
    fa = a.forces.cpu().numpy()
    b = compute(d1, ref, t, v)
    fb = b.forces.cpu().numpy()
    if scatter == "gather":
        assert np.array_equal(fa, fb)
    assert np.abs(fa - fb).max() <= 1e-12 * np.abs(fb).max()
    assert abs(a.potential_energy - b.potential_energy) <= 1e-12 * abs(b.potential_energy)


def test_device_rebuild_overflow_falls_back():
    # zero spare capacity, then a denser configuration: the device builder
    # overflows and the list is regrown by the host build
    st, tname = structures.config(2, small=True)
    t = builtin_params(tname)
    ctx = _native.default_context(0)
    ctx.set_table(t)
    ctx.set_option(_native.OPT_LIST_MARGIN, 0)
    try:
        d0 = _dev_state(st)
        nl = build_neighbor_list(d0, t.r_cut, 0.3)
        m0 = nl.n_entries
        st1 = _moved(st, 0.25, 5)
        d1 = _dev_state(st1)
        ref = build_neighbor_list(d1, t.r_cut, 0.3)
        assert ref.n_entries > m0
        nl.rebuild_on_device(d1.positions, d1.species)
    finally:
        ctx.set_option(_native.OPT_LIST_MARGIN, 25)
    assert np.array_equal(nl.offsets, ref.offsets)
    assert np.array_equal(nl.neighbors, ref.neighbors)


def test_device_rebuild_unsupported_free_axis():
    st, tname = structures.config(1)
    t = builtin_params(tname)
    st.box = SimulationBox(st.box.lengths, (True, False, True))
    d0 = _dev_state(st)
    nl = build_neighbor_list(d0, t.r_cut, 0.3)
    with pytest.raises(RuntimeError):
        nl.rebuild_on_device(d0.positions, d0.species)
