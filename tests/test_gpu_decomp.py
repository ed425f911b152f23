"""The decomposed path on the GPU kernels (B200Domain, C ABI tb_dd_*): two or
three processes share cuda:0 -- their kernels are independent, only the
host-level gloo exchange (Comm route "cpu") connects them -- and each drives
its slab through DomainMD.  Checks against the single-domain GPU path and the
oracle:
  * t = 0 evaluation: gathered forces / energy / virial;
  * union of the ranks' owned rows == the single-domain pair set;
  * 100 decomposed NVE steps (migrations, cross-rank rebuild trigger) ==
    the single-domain device NVE run (md.run_nve) and the oracle's."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _worker(rank, world, port, cfg, steps, precision, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_00882_b200 import decomp, structures
        from paper_1710_00882_b200.paramfile import builtin_params
        torch.cuda.set_device(0)
        st, tname = structures.config(cfg, small=True)
        table = builtin_params(tname)
        comm = decomp.Comm(rank, world, route="cpu")
        md = decomp.decompose(st, table, rank, world, comm, precision=precision, dt=1.0,
                              rebuild_every=10)
        r0 = md.setup().clone().cpu().numpy()
        ids, _, _, f = md.eng.export()
        f0 = decomp.gather_global(comm, ids, f, st.natoms).numpy()
        pairs0 = md.eng.pairs()
        mig = 0
        rec = [r0]
        for _ in range(steps):
            rec.append(md.step().clone().cpu().numpy())
            c = md.eng.counts()
            mig += int(c[5] + c[6])
        md.eng.check_errors()
        ids, pos, _, _ = md.eng.export()
        parts = [None] * world
        dist.all_gather_object(parts, (pairs0, ids, pos, mig))
        if rank == 0:
            q.put(dict(r0=r0, f0=f0, rec=np.array(rec), rebuilds=md.rebuilds, parts=parts))
    finally:
        dist.destroy_process_group()


def _run(world, cfg, steps, precision, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, steps, precision, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("world,cfg,precision,port",
                         [(2, 2, "double", 29711), (3, 3, "double", 29733),
                          (2, 2, "single", 29751)])
def test_decomposed_gpu_matches_single_domain(oracle_mod, world, cfg, precision, port):
    import paper_1710_00882_b200 as B
    from paper_1710_00882_b200 import structures
    from paper_1710_00882_b200.md import RunConfig, run_nve
    from paper_1710_00882_b200.paramfile import builtin_params
    steps = 100
    out = _run(world, cfg, steps, precision, port)
    st, tname = structures.config(cfg, small=True)
    table = builtin_params(tname)
    L, per = st.box.lengths, st.box.periodic
    tol = 1e-12 if precision == "double" else 1e-5
    # t = 0 evaluation vs the single-domain GPU path
    nl = B.build_neighbor_list(st, table.r_cut, 0.3)
    single = B.compute(st, nl, table, B.make_variant("B200", precision=precision))
    fmax = np.abs(single.forces).max()
    assert np.abs(out["f0"] - single.forces).max() <= tol * fmax
    assert abs(out["r0"][0] - single.potential_energy) <= tol * abs(single.potential_energy)
    assert np.abs(out["r0"][1:7] - single.virial).max() <= 1e3 * tol * np.abs(single.virial).max()
    # pair sets: union of owned rows == single-domain rows, none twice
    off, nb = nl.offsets, nl.neighbors
    i = np.repeat(np.arange(st.natoms), np.diff(off))
    want = set(zip(i.tolist(), nb.tolist()))
    got = [p[0] for p in out["parts"]]
    assert sum(len(g) for g in got) == len(want)
    assert set(map(tuple, np.concatenate(got).tolist())) == want
    # NVE vs the single-domain device run and the oracle's
    cfg_run = RunConfig(dt=1.0, steps=steps, skin=0.3, rebuild_every=10,
                        variant=B.make_variant("B200", precision=precision))
    one = run_nve(st.copy(), table, cfg_run)
    rec = out["rec"]
    total = rec[:, 0] + rec[:, 7]
    scale = abs(one["total"][0])
    ttol = 1e-9 if precision == "double" else 2e-6
    assert np.max(np.abs(total - one["total"])) <= ttol * scale
    assert out["rebuilds"] == one["rebuilds"]
    ids = np.concatenate([p[1] for p in out["parts"]])
    pos = np.concatenate([p[2] for p in out["parts"]])
    assert np.array_equal(np.sort(ids), np.arange(st.natoms))
    assert np.abs(pos[np.argsort(ids)] - one["positions"]).max() <= (
        1e-8 if precision == "double" else 1e-4)
    assert sum(p[3] for p in out["parts"]) > 0  # migrations happened
    if precision == "double":
        nve = oracle_mod.run_nve(st.positions, st.velocities, st.species, st.masses, L, per,
                                 table, dt=1.0, steps=steps, skin=0.3, rebuild_every=10)
        assert np.max(np.abs(total - nve["total"])) <= 1e-9 * scale
        assert out["rebuilds"] == nve["rebuilds"]
