"""The decomposed path on the GPU kernels: two processes share cuda:0 (their
kernels are independent; only the host-level gloo exchange connects them) and
each drives B200Engine (tb_build_neighbors_owned + tb_compute_device) on its
slab.  Gathered forces / energy / virial must equal the single-domain GPU
evaluation (same kernels) to round-off, and the oracle within 1e-10."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, cfg, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_00882_b200 import decomp, structures
        from paper_1710_00882_b200.paramfile import builtin_params
        torch.cuda.set_device(0)
        st, tname = structures.config(cfg, small=True)
        table = builtin_params(tname)
        decomp.set_comm_device("cpu")
        d = decomp.SlabDecomposition(st.box.lengths, st.box.periodic, table.r_cut + 0.3, world)
        dom = decomp.scatter_state(d, st, rank, "cuda:0")
        eng = decomp.B200Engine(table, 0.3, device=0)
        ff = decomp.DecomposedForceField(d, st.box, eng, rank, world, "cuda:0")
        dom = ff.rebuild(dom)
        f, res = ff(dom)
        fg = decomp.gather_global(dom, f, st.natoms, "cuda:0")
        if rank == 0:
            q.put((fg.cpu().numpy(), res.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg,port", [(2, 2, 29711), (3, 3, 29733)])
def test_decomposed_gpu_matches_single_domain(oracle_mod, world, cfg, port):
    import paper_1710_00882_b200 as B
    from paper_1710_00882_b200 import structures
    from paper_1710_00882_b200.paramfile import builtin_params
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    fg, res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    st, tname = structures.config(cfg, small=True)
    table = builtin_params(tname)
    nl = B.build_neighbor_list(st, table.r_cut, 0.3)
    single = B.compute(st, nl, table)
    fmax = np.abs(single.forces).max()
    assert np.abs(fg - single.forces).max() <= 1e-12 * fmax
    assert abs(res[0] - single.potential_energy) <= 1e-12 * abs(single.potential_energy)
    assert np.abs(res[1:7] - single.virial).max() <= 1e-10 * np.abs(single.virial).max()
