"""Slab decomposition (decomp.DomainMD + Comm) on CPU with the gloo backend,
world sizes 2, 3 and 4.

The per-rank engine here is a test double of B200Domain built on the CPU
oracle (its list build, evaluation, half-kick and drift -- the same arithmetic
as the oracle's own single-domain NVE run); DomainMD, Comm and the message
layout are the product code.  Checks:
  * an evaluation equals the single-domain oracle (forces, energy, virial);
  * 100 decomposed NVE steps with migrations reproduce the single-domain
    oracle run_nve (energies, rebuild count, final positions);
  * the union of the ranks' owned rows is the single-domain pair set, at the
    start and after the run (per-rank rows are never duplicated)."""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleDomain:
    """B200Domain's interface on numpy + the oracle (test infrastructure)."""

    def __init__(self, table, box, rank, nranks, skin=0.3):
        from oracle import oracle as O
        from paper_1710_00882_b200 import decomp
        self.O, self.table, self.box, self.skin = O, table, box, skin
        self.d = decomp.SlabDecomposition(box.lengths, box.periodic, table.r_cut + skin, nranks)
        self.rank, self.nranks = rank, nranks
        self.left, self.right = (rank - 1) % nranks, (rank + 1) % nranks
        self.device = torch.device("cpu")
        self.drift2 = torch.zeros(1, dtype=torch.float64)
        self.migrated = 0
        self.ngl = self.ngr = 0
        self.send = np.zeros(0, np.int64)

    # ---- state ----
    def load(self, ids, pos, vel, mass, species):
        self.ids = np.array(ids, np.int64)
        self.pos = np.array(pos, np.float64)
        self.vel = np.array(vel, np.float64)
        self.mass = np.array(mass, np.float64)
        self.sp = np.array(species, np.int64)
        self._local()

    def _local(self):
        n = len(self.ids)
        self.n_owned = n
        self.lpos = np.zeros((n + self.ngl + self.ngr, 3))
        self.lpos[:n] = self.pos
        self.frc = np.zeros_like(self.lpos)
        t = torch.from_numpy(self.lpos)
        f = torch.from_numpy(self.frc)
        self.pos_ghosts = (t[n:n + self.ngl], t[n + self.ngl:])
        self.force_ghosts = (f[n:n + self.ngl], f[n + self.ngl:])
        ns = len(self.send)
        self._back = torch.zeros((ns, 3), dtype=torch.float64)
        self.force_recv = (self._back[:self.nsl], self._back[self.nsl:]) if ns else (
            self._back[:0], self._back[:0])
        self._psend = torch.zeros((ns, 3), dtype=torch.float64)
        self.pos_send = (self._psend[:self.nsl], self._psend[self.nsl:])

    nsl = 0

    def export(self):
        return self.ids, self.pos, self.vel, self.frc[:self.n_owned]

    # ---- rebuild ----
    def migrate_pack(self):
        own = self.d.owner(self.pos[:, 0])
        to_l = own == self.left
        to_r = (own == self.right) & ~to_l
        if np.any((own != self.rank) & ~to_l & ~to_r):
            raise RuntimeError("an atom moved more than one slab")
        self._keep = np.nonzero(own == self.rank)[0]
        rows = np.column_stack([self.pos, self.vel, self.mass, self.sp, self.ids]).astype(float)
        self.migrated += int(to_l.sum() + to_r.sum())
        return torch.from_numpy(rows[to_l].copy()), torch.from_numpy(rows[to_r].copy())

    def migrate_recv(self, nl, nr):
        self._rows = torch.zeros((nl + nr, 9), dtype=torch.float64)
        return self._rows[:nl], self._rows[nl:]

    def migrate_unpack(self, nl, nr):
        k, r = self._keep, self._rows.numpy()
        self.ids = np.concatenate([self.ids[k], r[:, 8].astype(np.int64)])
        self.pos = np.concatenate([self.pos[k], r[:, 0:3]])
        self.vel = np.concatenate([self.vel[k], r[:, 3:6]])
        self.mass = np.concatenate([self.mass[k], r[:, 6]])
        self.sp = np.concatenate([self.sp[k], r[:, 7].astype(np.int64)])
        self.ngl = self.ngr = 0

    def halo_pack(self):
        col = self.d.columns(self.pos[:, 0])
        sl = np.nonzero(col == self.d.first_col(self.rank))[0]
        sr = np.nonzero(col == self.d.last_col(self.rank))[0]
        self.send, self.nsl = np.concatenate([sl, sr]), len(sl)
        meta = np.column_stack([self.ids, self.sp]).astype(float)
        return torch.from_numpy(meta[sl].copy()), torch.from_numpy(meta[sr].copy())

    def halo_recv(self, nl, nr):
        self._meta = torch.zeros((nl + nr, 2), dtype=torch.float64)
        return self._meta[:nl], self._meta[nl:]

    def halo_unpack(self, nl, nr):
        m = self._meta.numpy()
        self.gids, self.gsp = m[:, 0].astype(np.int64), m[:, 1].astype(np.int64)
        self.ngl, self.ngr = nl, nr
        self._local()

    def build(self):
        n = self.n_owned
        self.lpos[:n] = self.pos
        off, nb = self.O.build_neighbor_list(self.lpos, self.box.lengths, self.box.periodic,
                                             self.table.r_cut, self.skin)
        cnt = np.diff(off)
        cnt[n:] = 0  # rows only for owned atoms
        keep = np.repeat(np.arange(len(self.lpos)) < n, np.diff(off))
        self.off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        self.nb = nb[keep]
        self.ref = self.pos.copy()

    def local_ids(self):
        return np.concatenate([self.ids, self.gids]) if self.nranks > 1 else self.ids

    def pairs(self):
        ids = self.local_ids()
        i = np.repeat(np.arange(len(self.off) - 1), np.diff(self.off))
        return np.stack([ids[i], ids[self.nb]], axis=1)

    # ---- every evaluation ----
    def pack_positions(self):
        self._psend.copy_(torch.from_numpy(self.pos[self.send]))

    def compute(self, result, stats=None):
        n = self.n_owned
        self.lpos[:n] = self.pos
        sp = np.concatenate([self.sp, self.gsp]) if self.nranks > 1 else self.sp
        r = self.O.compute(self.lpos, sp, self.box.lengths, self.box.periodic, self.off, self.nb,
                           self.table)
        self.frc[:] = r["forces"]
        result[0] = r["energy"]
        result[1:7] = torch.from_numpy(np.asarray(r["virial"]))

    def reverse_add(self):
        np.add.at(self.frc, self.send, self._back.numpy())

    # ---- integration (the oracle's own half-kick / drift arithmetic) ----
    def kick_drift(self, dt, accel):
        O, n = self.O, self.n_owned
        L, per = O._box(self.box.lengths, self.box.periodic)
        f = np.ascontiguousarray(self.frc[:n])
        O.lib().or_half_kick(n, O._p(self.vel), O._p(f), O._p(self.mass), 0.5 * dt * accel)
        O.lib().or_drift_wrap(n, O._p(self.pos), O._p(self.vel), float(dt), O._p(L), O._p(per))
        d = self.pos - self.ref
        for ax in range(3):
            if self.box.periodic[ax]:
                d[:, ax] -= L[ax] * np.round(d[:, ax] / L[ax])
        self.drift2[0] = float(((d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1]) + d[:, 2] * d[:, 2])
                               .max(initial=0.0))
        return self.drift2

    def kick(self, dt, accel, result):
        O, n = self.O, self.n_owned
        f = np.ascontiguousarray(self.frc[:n])
        O.lib().or_half_kick(n, O._p(self.vel), O._p(f), O._p(self.mass), 0.5 * dt * accel)
        result[7] = 0.5 * float((self.mass * (self.vel ** 2).sum(axis=1)).sum()) / accel


def _worker(rank, world, port, cfg, steps, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1710_00882_b200 import decomp, structures
        from paper_1710_00882_b200.paramfile import builtin_params
        st, tname = structures.config(cfg, small=True)
        table = builtin_params(tname)
        eng = OracleDomain(table, st.box, rank, world)
        d = eng.d
        ids = decomp.owned_atoms(d, st, rank)
        eng.load(ids, st.positions[ids], st.velocities[ids], st.atom_masses[ids],
                 st.species[ids])
        md = decomp.DomainMD(eng, decomp.Comm(rank, world), skin=0.3, dt=1.0, rebuild_every=10)
        out = {}
        r0 = md.setup().clone().numpy()
        f0 = decomp.gather_global(md.comm, eng.ids, eng.frc[:eng.n_owned], st.natoms)
        pairs0 = eng.pairs()
        rec = [r0]
        for _ in range(steps):
            rec.append(md.step().clone().numpy())
        md.rebuild()  # final list at the final positions: pair set check
        ids_f, pos_f, vel_f, _ = eng.export()
        allp = [None] * world
        dist.all_gather_object(allp, (pairs0, eng.pairs(), ids_f, pos_f, eng.migrated))
        if rank == 0:
            out = dict(r0=r0, f0=f0.numpy(), rec=np.array(rec), rebuilds=md.rebuilds - 1,
                       parts=allp)
            q.put(out)
    finally:
        dist.destroy_process_group()


def _run(world, cfg, steps, port):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


def _pair_set(pairs):
    return set(map(tuple, np.concatenate(pairs).tolist()))


@pytest.mark.parametrize("world,port", [(2, 29611), (3, 29623), (4, 29637)])
def test_decomposed_nve_matches_single_domain(oracle_mod, world, port):
    from paper_1710_00882_b200 import structures
    from paper_1710_00882_b200.paramfile import builtin_params
    steps = 100
    out = _run(world, 2, steps, port)
    st, tname = structures.config(2, small=True)
    table = builtin_params(tname)
    L, per = st.box.lengths, st.box.periodic
    # evaluation at t = 0 against the single-domain oracle
    off, nb = oracle_mod.build_neighbor_list(st.positions, L, per, table.r_cut, 0.3)
    ref = oracle_mod.compute(st.positions, st.species, L, per, off, nb, table)
    fmax = np.abs(ref["forces"]).max()
    assert np.abs(out["f0"] - ref["forces"]).max() <= 1e-12 * fmax
    assert abs(out["r0"][0] - ref["energy"]) <= 1e-12 * abs(ref["energy"])
    assert np.abs(out["r0"][1:7] - ref["virial"]).max() <= 1e-10 * np.abs(ref["virial"]).max()
    # pair sets: union of owned rows == single-domain list, no row twice
    i = np.repeat(np.arange(st.natoms), np.diff(off))
    want0 = set(zip(i.tolist(), nb.tolist()))
    parts = out["parts"]
    got0 = [p[0] for p in parts]
    assert sum(len(p) for p in got0) == len(want0) and _pair_set(got0) == want0
    # 100 NVE steps (dt 1 fs, skin 0.3, rebuild every 10 + trigger) vs the oracle
    nve = oracle_mod.run_nve(st.positions, st.velocities, st.species, st.masses, L, per, table,
                             dt=1.0, steps=steps, skin=0.3, rebuild_every=10)
    rec = out["rec"]
    total = rec[:, 0] + rec[:, 7]
    scale = abs(nve["total"][0])
    assert np.max(np.abs(total - nve["total"])) <= 1e-9 * scale
    assert np.max(np.abs(rec[:, 0] - nve["potential"])) <= 1e-9 * scale
    assert out["rebuilds"] == nve["rebuilds"]
    ids = np.concatenate([p[2] for p in parts])
    pos = np.concatenate([p[3] for p in parts])
    assert np.array_equal(np.sort(ids), np.arange(st.natoms))  # each atom owned exactly once
    assert np.abs(pos[np.argsort(ids)] - nve["positions"]).max() <= 1e-8
    assert sum(p[4] for p in parts) > 0  # atoms did migrate between slabs
    # final pair set at the final positions
    offf, nbf = oracle_mod.build_neighbor_list(nve["positions"], L, per, table.r_cut, 0.3)
    i = np.repeat(np.arange(st.natoms), np.diff(offf))
    assert _pair_set([p[1] for p in parts]) == set(zip(i.tolist(), nbf.tolist()))


def test_slab_geometry():
    from paper_1710_00882_b200 import decomp
    d = decomp.SlabDecomposition([43.448, 43.448, 43.448], (True, True, True), 3.3, 4)
    assert d.ncx == 13 and d.bounds == [0, 3, 6, 9, 13]
    x = np.array([0.0, 3.3422, 43.447999, -1e-12, 43.448])  # width 3.34215
    assert list(d.columns(x)) == [0, 1, 12, 12, 0]
    with pytest.raises(Exception):
        decomp.SlabDecomposition([10.0, 10, 10], (True, True, True), 3.3, 2)
