"""Spatial (slab) domain decomposition of the Tersoff evaluation and of the NVE
run across ranks -- BASELINE north_star (4), SURVEY.md 8(e).

One process per GPU.  Each rank owns a slab of whole x cell columns of the
neighbour grid (>= 2 columns per rank: ncx = max(int(Lx / bc), 1), width =
Lx / ncx, column = floor(remainder(x, Lx) / width) clipped -- neighbor.py:54-88
arithmetic, so an atom's owner is the same on every rank and in the
single-domain build).  Ghosts are the atoms of the one column beyond each face
(width >= r_cut + skin) at unshifted coordinates: every displacement is the
global-box minimum image, so each owned row, its displacement bits and its
energy terms equal the single-domain ones; only owned atoms get rows, so each
term is evaluated exactly once; forces landing on ghosts go back to their
owners (reverse halo).  The reference has no decomposition: the
parity target is the single-domain evaluation and NVE run.

Per evaluation: forward halo (positions of the send lists to the +-1 ranks),
evaluation over [owned | ghosts], reverse halo, sum of [E, W6] over ranks.
Per NVE step (system.py:355-380, :427-460): half-kick + drift + wrap of the
owned atoms; the skin/2 trigger (neighbor.py:220-229) on the max drift over
ranks (all-reduce MAX), plus the fixed cadence; at a rebuild migration of the
atoms whose column changed owner, new send lists and ghost ids / species, a
positions halo and the owned-rows list; evaluation; second half-kick;
[E, W6, E_kin] summed over ranks.

Two layers:
  * the rank's data and kernels -- B200Domain, the C ABI tb_dd_* (csrc/tb_dd.cuh:
    classification, stable compaction by hand-written scans, packing, ghost
    unpacking, reverse adds, velocity Verlet; all in HBM, no host copies);
  * the transport and the step logic -- Comm (torch.distributed P2P: NCCL over
    NVLink on GPUs, gloo in the CPU tests) and DomainMD, engine-agnostic (the
    CPU tests drive the same DomainMD with a numpy/oracle engine).
"""

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigurationError

# ---------------------------------------------------------------------------
# slab geometry (host mirror of tb_dd.cuh Slab; scatter and tests)
# ---------------------------------------------------------------------------


class SlabDecomposition:
    """Which cell columns each rank owns."""

    def __init__(self, lengths, periodic, bc, nranks):
        if not periodic[0]:
            raise ConfigurationError("slab decomposition needs a periodic x axis")
        self.Lx = float(lengths[0])
        self.ncx = max(int(self.Lx / bc), 1)
        self.width = self.Lx / self.ncx
        self.nranks = int(nranks)
        if self.nranks > 1 and self.ncx < 2 * self.nranks:
            raise ConfigurationError(
                f"{self.ncx} cell columns cannot give {self.nranks} ranks two columns each")
        self.bounds = [r * self.ncx // self.nranks for r in range(self.nranks + 1)]
        self._owner = np.zeros(self.ncx, dtype=np.int64)
        for r in range(self.nranks):
            self._owner[self.bounds[r]:self.bounds[r + 1]] = r

    def columns(self, x):
        c = np.floor(np.remainder(np.asarray(x, dtype=np.float64), self.Lx)
                     / self.width).astype(np.int64)
        return np.clip(c, 0, self.ncx - 1)

    def owner(self, x):
        return self._owner[self.columns(x)]

    def first_col(self, r):
        return self.bounds[r]

    def last_col(self, r):
        return self.bounds[r + 1] - 1


def owned_atoms(decomp, state, rank):
    """Global ids of the atoms rank `rank` owns initially (every rank sees the
    same seeded global state)."""
    return np.nonzero(decomp.owner(state.positions[:, 0]) == rank)[0].astype(np.int64)


# ---------------------------------------------------------------------------
# transport
# ---------------------------------------------------------------------------


class Comm:
    """Neighbour P2P and all-reduces over torch.distributed.

    `route` (e.g. "cpu"): move tensors there for the transport (a gloo group
    with CUDA-resident domains); None = use the tensors where they live
    (NCCL).  Zero-row messages are padded to one row on both ends (the
    counts are exchanged first, so both ends agree)."""

    def __init__(self, rank, nranks, route=None):
        self.rank, self.nranks, self.route = rank, nranks, route
        self.left = (rank - 1) % nranks
        self.right = (rank + 1) % nranks

    def _p2p(self, sends, recvs):
        # fixed message order per peer (to-left before to-right) also pairs the
        # two messages of the two-rank ring, where left == right
        ops = [dist.P2POp(dist.isend, sends[0], self.left),
               dist.P2POp(dist.irecv, recvs[1], self.right),
               dist.P2POp(dist.isend, sends[1], self.right),
               dist.P2POp(dist.irecv, recvs[0], self.left)]
        for req in dist.batch_isend_irecv(ops):
            req.wait()

    def exchange(self, sends, recvs):
        """sends = (to_left, to_right), recvs = (from_left, from_right): row
        blocks of equal width and dtype; received in place."""
        if self.nranks == 1:
            return
        dev = recvs[0].device
        route = self.route if self.route is not None and str(self.route) != str(dev) else None
        pad = any(t.shape[0] == 0 for t in (*sends, *recvs))
        if route is None and not pad:
            self._p2p([t.contiguous() for t in sends], recvs)
            return
        where = route or dev

        def staged(t):
            t = t.to(where).contiguous()
            return t if t.shape[0] else torch.zeros((1,) + tuple(t.shape[1:]), dtype=t.dtype,
                                                    device=where)
        s = [staged(t) for t in sends]
        r = [torch.empty((max(t.shape[0], 1),) + tuple(t.shape[1:]), dtype=t.dtype, device=where)
             for t in recvs]
        self._p2p(s, r)
        for dst, src in zip(recvs, r):
            if dst.shape[0]:
                dst.copy_(src[:dst.shape[0]])

    def exchange_counts(self, to_left, to_right, device):
        s = (torch.tensor([[to_left]], dtype=torch.int64, device=device),
             torch.tensor([[to_right]], dtype=torch.int64, device=device))
        r = (torch.empty((1, 1), dtype=torch.int64, device=device),
             torch.empty((1, 1), dtype=torch.int64, device=device))
        self.exchange(s, r)
        return int(r[0].item()), int(r[1].item())

    def allreduce(self, t, op="sum"):
        if self.nranks == 1:
            return t
        o = dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX
        if self.route is not None and str(self.route) != str(t.device):
            x = t.to(self.route)
            dist.all_reduce(x, op=o)
            t.copy_(x)
        else:
            dist.all_reduce(t, op=o)
        return t


# ---------------------------------------------------------------------------
# the rank's atoms on the B200 (C ABI tb_dd_*)
# ---------------------------------------------------------------------------

_POS, _VEL, _FORCES, _MASS, _SPECIES, _IDS, _SEND, _RECV = range(8)
_DT = {"f8": torch.float64, "i4": torch.int32, "i8": torch.int64}


class _Dev:
    """A CUDA array interface over a domain buffer (zero-copy torch view)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<" + typestr,
                                         "data": (int(ptr or 0), False), "version": 3,
                                         "strides": None}


class B200Domain:
    """One rank's atoms in HBM and the tb_dd_* kernels (engine of DomainMD)."""

    def __init__(self, params, box, rank, nranks, skin=0.3, device=0, precision="double",
                 scatter="atomic"):
        from . import _native
        self.native = _native
        self.ctx = _native.default_context(device)
        self.ctx.set_table(params)
        self.params, self.box, self.skin = params, box, skin
        self.device = torch.device("cuda", device)
        self.prec = _native.PRECISION[precision]
        self.scat = _native.SCATTER[scatter]
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        L = np.ascontiguousarray(np.asarray(box.lengths, dtype=np.float64))
        per = np.ascontiguousarray(np.asarray(box.periodic, dtype=np.int32))
        h = ctypes.c_void_p()
        self._check(self.ctx.lib.tb_dd_create(self.ctx.handle, rank, nranks, _native.ptr(L),
                                              _native.ptr(per), float(params.r_cut),
                                              float(skin), ctypes.byref(h)), "tb_dd_create")
        self.h = h
        self.nl = _native.NList(self.ctx)
        self._i64 = (ctypes.c_int64(), ctypes.c_int64())
        self.drift2 = torch.zeros(1, dtype=torch.float64, device=self.device)

    def __del__(self):
        try:
            if self.h:
                self.ctx.lib.tb_dd_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def _check(self, rc, what):
        self.ctx.check(rc, what)

    def counts(self):
        out = np.zeros(10, dtype=np.int64)
        self._check(self.ctx.lib.tb_dd_counts(self.h, self.native.ptr(out)), "tb_dd_counts")
        return out

    def _view(self, which, row0, rows, width, typestr="f8"):
        p = ctypes.c_void_p()
        self._check(self.ctx.lib.tb_dd_buffer(self.h, which, ctypes.byref(p)), "tb_dd_buffer")
        item = int(typestr[1])
        if rows == 0:
            return torch.empty((0, width) if width else (0,), dtype=_DT[typestr],
                               device=self.device)
        shape = (rows, width) if width else (rows,)
        return torch.as_tensor(_Dev((p.value or 0) + row0 * max(width, 1) * item, shape, typestr),
                               device=self.device)

    def _recv(self, rows, width):
        p = ctypes.c_void_p()
        self._check(self.ctx.lib.tb_dd_recv_buffer(self.h, rows, width, ctypes.byref(p)),
                    "tb_dd_recv_buffer")
        return p.value

    def _split(self, which, nl, nr, width):
        return (self._view(which, 0, nl, width), self._view(which, nl, nr, width))

    # ---- state ----
    def load(self, ids, pos, vel, mass, species):
        P, n = self.native.ptr, len(ids)
        arr = [np.ascontiguousarray(pos, dtype=np.float64),
               np.ascontiguousarray(vel, dtype=np.float64),
               np.ascontiguousarray(mass, dtype=np.float64),
               np.ascontiguousarray(species, dtype=np.int32),
               np.ascontiguousarray(ids, dtype=np.int64)]
        self._check(self.ctx.lib.tb_dd_load(self.h, n, *[P(a) for a in arr]), "tb_dd_load")

    def export(self):
        c = self.counts()
        n = int(c[0])
        ids, pos, vel, f = (np.zeros(n, np.int64), np.zeros((n, 3)), np.zeros((n, 3)),
                            np.zeros((n, 3)))
        P = self.native.ptr
        self._check(self.ctx.lib.tb_dd_export(self.h, P(ids), P(pos), P(vel), P(f)),
                    "tb_dd_export")
        return ids, pos, vel, f

    def local_ids(self):
        c = self.counts()
        return self._view(_IDS, 0, int(c[0] + c[1] + c[2]), 0, "i8").cpu().numpy()

    # ---- rebuild ----
    def migrate_pack(self):
        a, b = self._i64
        self._check(self.ctx.lib.tb_dd_migrate_pack(self.h, ctypes.byref(a), ctypes.byref(b)),
                    "tb_dd_migrate_pack")
        return self._split(_SEND, a.value, b.value, 9)

    def migrate_recv(self, nl, nr):
        self._recv(nl + nr, 9)
        return self._split(_RECV, nl, nr, 9)

    def migrate_unpack(self, nl, nr):
        self._check(self.ctx.lib.tb_dd_migrate_unpack(self.h, nl, nr), "tb_dd_migrate_unpack")

    def halo_pack(self):
        a, b = self._i64
        self._check(self.ctx.lib.tb_dd_halo_pack(self.h, ctypes.byref(a), ctypes.byref(b)),
                    "tb_dd_halo_pack")
        return self._split(_SEND, a.value, b.value, 2)

    def halo_recv(self, nl, nr):
        self._recv(nl + nr, 2)
        return self._split(_RECV, nl, nr, 2)

    def halo_unpack(self, nl, nr):
        self._check(self.ctx.lib.tb_dd_halo_unpack(self.h, nl, nr), "tb_dd_halo_unpack")
        self._layout()

    def _layout(self):
        """Views of the per-evaluation message blocks (fixed until the next
        rebuild: graph-capturable)."""
        c = self.counts()
        n, ngl, ngr, nsl, nsr = (int(v) for v in c[:5])
        self.n_owned, self.n_local = n, n + ngl + ngr
        self.pos_ghosts = (self._view(_POS, n, ngl, 3), self._view(_POS, n + ngl, ngr, 3))
        self.force_ghosts = (self._view(_FORCES, n, ngl, 3), self._view(_FORCES, n + ngl, ngr, 3))
        self.pos_send = self._split(_SEND, nsl, nsr, 3) if nsl + nsr else (
            self._view(_SEND, 0, 0, 3), self._view(_SEND, 0, 0, 3))
        self._recv(nsl + nsr, 3)
        self.force_recv = self._split(_RECV, nsl, nsr, 3)

    def build(self):
        self._check(self.ctx.lib.tb_dd_build(self.h, self.nl.handle), "tb_dd_build")
        self._layout()

    # ---- every evaluation ----
    def pack_positions(self):
        self._check(self.ctx.lib.tb_dd_pack_positions(self.h), "tb_dd_pack_positions")

    def compute(self, result, stats=None):
        P = self.native.ptr
        self._check(self.ctx.lib.tb_dd_compute(self.h, self.nl.handle, self.prec, self.scat,
                                               P(result), P(stats)), "tb_dd_compute")

    def reverse_add(self):
        self._check(self.ctx.lib.tb_dd_reverse_add(self.h), "tb_dd_reverse_add")

    # ---- integration ----
    def kick_drift(self, dt, accel):
        self._check(self.ctx.lib.tb_dd_kick_drift(self.h, self.nl.handle, float(dt), float(accel),
                                                  self.native.ptr(self.drift2)),
                    "tb_dd_kick_drift")
        return self.drift2

    def kick(self, dt, accel, result):
        self._check(self.ctx.lib.tb_dd_kick(self.h, float(dt), float(accel),
                                            self.native.ptr(result)), "tb_dd_kick")

    def pairs(self):
        """Owned rows as global-id pairs (gid_i, gid_j), for parity checks."""
        n, m, _ = self.nl.info()
        off = np.zeros(n + 1, np.int64)
        nbr = np.zeros(max(m, 1), np.int64)
        P = self.native.ptr
        self.ctx.check(self.ctx.lib.tb_nlist_export(self.ctx.handle, self.nl.handle, P(off),
                                                    P(nbr)), "tb_nlist_export")
        ids = self.local_ids()
        i = np.repeat(np.arange(n), np.diff(off))
        return np.stack([ids[i], ids[nbr[:m]]], axis=1)

    def check_errors(self):
        self.ctx.check(self.ctx.lib.tb_check_errors(self.ctx.handle), "tb_check_errors")


# ---------------------------------------------------------------------------
# the decomposed evaluation and NVE run (engine-agnostic)
# ---------------------------------------------------------------------------


class DomainMD:
    """Slab-decomposed evaluation / velocity-Verlet NVE over `engine` (the
    rank's atoms) and `comm` (the transport).

    result (device tensor, 8 doubles): [E, W xx yy zz xy xz yz, E_kin], summed
    over ranks after every step."""

    def __init__(self, engine, comm, skin=0.3, dt=1.0, rebuild_every=0, accel=None):
        from .state import ACCEL
        self.eng, self.comm = engine, comm
        self.skin, self.dt, self.rebuild_every = skin, dt, int(rebuild_every or 0)
        self.accel = ACCEL if accel is None else accel
        self.device = engine.device
        self.result = torch.zeros(8, dtype=torch.float64, device=self.device)
        self.rebuilds = 0
        self.step_no = 0

    # ---- rebuild: migration, send lists, ghost identities, list ----
    def rebuild(self):
        eng, comm = self.eng, self.comm
        if comm.nranks > 1:
            sl, sr = eng.migrate_pack()
            nfl, nfr = comm.exchange_counts(sl.shape[0], sr.shape[0], self.device)
            comm.exchange((sl, sr), eng.migrate_recv(nfl, nfr))
            eng.migrate_unpack(nfl, nfr)
            ml, mr = eng.halo_pack()
            ngl, ngr = comm.exchange_counts(ml.shape[0], mr.shape[0], self.device)
            comm.exchange((ml, mr), eng.halo_recv(ngl, ngr))
            eng.halo_unpack(ngl, ngr)
            self.forward_positions()
        eng.build()
        self.rebuilds += 1

    # ---- every evaluation ----
    def forward_positions(self):
        if self.comm.nranks > 1:
            self.eng.pack_positions()
            self.comm.exchange(self.eng.pos_send, self.eng.pos_ghosts)

    def evaluate_local(self, stats=None):
        """Halo + evaluation + reverse halo: complete forces on the owned atoms,
        this rank's [E, W6] in result[:7] (not yet summed)."""
        self.forward_positions()
        self.eng.compute(self.result, stats)
        if self.comm.nranks > 1:
            self.comm.exchange(self.eng.force_ghosts, self.eng.force_recv)
            self.eng.reverse_add()
        return self.result

    def evaluate(self, stats=None):
        """One decomposed E+F+virial evaluation; [E, W6] summed over ranks."""
        self.evaluate_local(stats)
        self.result[7] = 0.0
        return self.comm.allreduce(self.result)

    # ---- NVE ----
    def setup(self):
        """List, F(0), E(0) and E_kin(0) (run_nve's first ForceField call)."""
        self.rebuild()
        self.evaluate_local()
        self.eng.kick(0.0, self.accel, self.result)  # zero-length kick: E_kin of v(0)
        return self.comm.allreduce(self.result)

    def step(self):
        d2 = self.eng.kick_drift(self.dt, self.accel)
        d2 = float(self.comm.allreduce(d2.clone(), op="max")[0])
        self.step_no += 1
        if d2 > (0.5 * self.skin) ** 2 or \
                (self.rebuild_every and self.step_no % self.rebuild_every == 0):
            self.rebuild()
        self.evaluate_local()
        self.eng.kick(self.dt, self.accel, self.result)
        return self.comm.allreduce(self.result)

    def run(self, steps, record_every=1):
        """NVE record as the reference's run_nve: potential / kinetic / total
        per recorded step (row 0 = the setup state), rebuild count."""
        rec = [self.setup().clone()]
        for s in range(1, steps + 1):
            r = self.step()
            if s % record_every == 0:
                rec.append(r.clone())
        a = torch.stack(rec).cpu().numpy()
        return {"kind": "nve", "steps": steps, "dt": self.dt, "potential": a[:, 0],
                "kinetic": a[:, 7], "total": a[:, 0] + a[:, 7], "rebuilds": self.rebuilds,
                "virial": a[:, 1:7]}


def decompose(state, params, rank, nranks, comm=None, skin=0.3, device=0, precision="double",
              scatter="atomic", dt=1.0, rebuild_every=0):
    """Rank `rank`'s DomainMD on the B200 for a global (seeded) state."""
    d = SlabDecomposition(state.box.lengths, state.box.periodic, params.r_cut + skin, nranks)
    ids = owned_atoms(d, state, rank)
    eng = B200Domain(params, state.box, rank, nranks, skin, device, precision, scatter)
    vel = state.velocities if state.velocities is not None else np.zeros_like(state.positions)
    eng.load(ids, state.positions[ids], vel[ids], state.atom_masses[ids], state.species[ids])
    return DomainMD(eng, comm or Comm(rank, nranks), skin, dt, rebuild_every)


def gather_global(comm, ids, values, n_global, device="cpu"):
    """Sum-gather per-atom rows (owned ids) into the global order (tests)."""
    out = torch.zeros((n_global,) + tuple(values.shape[1:]), dtype=torch.float64,
                      device=comm.route or device)
    out[torch.as_tensor(ids, device=out.device)] = torch.as_tensor(values, dtype=torch.float64,
                                                                   device=out.device)
    return comm.allreduce(out)
