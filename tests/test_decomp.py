"""Slab decomposition (decomp.py) on CPU with the gloo backend, world sizes 2
and 3, the per-rank engine being the oracle: the decomposed forces, energy
and virial must equal the single-domain result, including after atoms
migrate between slabs."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleEngine:
    """Test double of B200Engine: the CPU oracle on the rank's local atoms,
    rows only for owned atoms (as tb_build_neighbors_owned)."""

    def __init__(self, table, skin=0.3):
        from oracle import oracle as O
        self.O, self.table, self.skin = O, table, skin

    def rebuild(self, pos_l, sp_l, n_owned, box):
        p = pos_l.numpy()
        off, nb = self.O.build_neighbor_list(p, box.lengths, box.periodic, self.table.r_cut,
                                             self.skin)
        cnt = np.diff(off)
        cnt[n_owned:] = 0
        keep = np.repeat(np.arange(len(p)) < n_owned, np.diff(off))
        self.off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        self.nb = nb[keep]
        self.box = box

    def compute(self, pos_l, sp_l):
        r = self.O.compute(pos_l.numpy(), sp_l.numpy().astype(np.int64), self.box.lengths,
                           self.box.periodic, self.off, self.nb, self.table)
        res = torch.tensor([r["energy"]] + list(r["virial"]), dtype=torch.float64)
        return torch.from_numpy(r["forces"]), res


def _worker(rank, world, port, cfg, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_00882_b200 import decomp, structures
        from paper_1710_00882_b200.paramfile import builtin_params
        st, tname = structures.config(cfg, small=True)
        table = builtin_params(tname)
        d = decomp.SlabDecomposition(st.box.lengths, st.box.periodic, table.r_cut + 0.3, world)
        dom = decomp.scatter_state(d, st, rank, "cpu")
        ff = decomp.DecomposedForceField(d, st.box, OracleEngine(table), rank, world, "cpu")
        out = {}
        for phase in range(2):
            if phase == 1:
                # move every atom by 0.2-0.6 A along x (beyond the skin, across
                # slab boundaries): migration + rebuild
                rng = np.random.default_rng(7)
                shift = rng.uniform(0.2, 0.6, size=st.natoms)
                st.positions[:, 0] = np.remainder(st.positions[:, 0] + shift, st.box.lengths[0])
                dom.pos = torch.from_numpy(st.positions[dom.ids].copy())
            dom = ff.rebuild(dom)
            f, res = ff(dom)
            fg = decomp.gather_global(dom, f, st.natoms, "cpu")
            nown = torch.tensor([dom.n_owned], dtype=torch.int64)
            dist.all_reduce(nown)
            out[phase] = (fg.numpy(), res.numpy(), int(nown.item()), st.positions.copy())
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def _run(world, cfg, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,cfg,port", [(2, 1, 29611), (3, 1, 29623), (2, 4, 29637)])
def test_slab_decomposition_matches_single_domain(oracle_mod, world, cfg, port):
    from paper_1710_00882_b200 import structures
    from paper_1710_00882_b200.paramfile import builtin_params
    out = _run(world, cfg, port)
    st, tname = structures.config(cfg, small=True)
    table = builtin_params(tname)
    for phase in (0, 1):
        fg, res, nown, pos = out[phase]
        assert nown == st.natoms  # every atom owned exactly once
        off, nb = oracle_mod.build_neighbor_list(pos, st.box.lengths, st.box.periodic,
                                                 table.r_cut, 0.3)
        ref = oracle_mod.compute(pos, st.species, st.box.lengths, st.box.periodic, off, nb, table)
        fmax = np.abs(ref["forces"]).max()
        assert np.abs(fg - ref["forces"]).max() <= 1e-12 * fmax
        assert abs(res[0] - ref["energy"]) <= 1e-12 * abs(ref["energy"])
        assert np.abs(res[1:7] - ref["virial"]).max() <= 1e-10 * np.abs(ref["virial"]).max()


def test_slab_geometry():
    from paper_1710_00882_b200 import decomp
    d = decomp.SlabDecomposition([43.448, 43.448, 43.448], (True, True, True), 3.3, 4)
    assert d.ncx == 13 and d.bounds == [0, 3, 6, 9, 13]
    x = np.array([0.0, 3.3422, 43.447999, -1e-12, 43.448])  # width 3.34215
    assert list(d.columns(x)) == [0, 1, 12, 12, 0]
    with pytest.raises(Exception):
        decomp.SlabDecomposition([10.0, 10, 10], (True, True, True), 3.3, 2)
