"""Spatial (slab) domain decomposition of the Tersoff evaluation across ranks.

BASELINE north_star (4) / SURVEY.md 8(e): one slab of whole cell columns along
x per rank (one process per GPU), ghost halos one cell column (>= rc + skin)
wide on both faces, forces on ghosts reverse-communicated to their owners.
The reference has no decomposition; parity target is the
single-domain result:

* columns are the global cell grid of the neighbour build (neighbor.py:54-88):
  ncx = floor(Lx / bc), width = Lx / ncx, column = floor(remainder(x, Lx) /
  width) clipped -- numpy arithmetic identical to the GPU binning, so an atom's
  column is the same on every rank and in the single-domain build;
* ghosts keep their unshifted coordinates and every displacement uses the
  global-box minimum image, so each owned atom's neighbour row, displacement
  bits and energy terms equal the single-domain ones;
* only owned atoms get rows (tb_build_neighbors_owned), so every energy term is
  evaluated exactly once across ranks.

Per evaluation: forward halo (positions of the send lists to the +-1 ranks,
torch.distributed P2P: NCCL over NVLink on GPUs, gloo in the CPU tests),
compute on [owned | left ghosts | right ghosts], reverse halo (ghost forces
back to their owners), all-reduce of [E, W6].  At a rebuild: migration of
atoms that changed column owner, new send lists, ghost ids/species.

The per-rank force engine is pluggable (`engine.rebuild`, `engine.compute`):
B200Engine drives the CUDA kernels; the CPU tests plug in the oracle.
"""

import numpy as np
import torch
import torch.distributed as dist

from .errors import ConfigurationError


def _np_remainder(x, L):
    return np.remainder(x, L)


class SlabDecomposition:
    """Static slab geometry: which cell columns each rank owns."""

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
        """Cell column of each x (neighbor.py:83-88 arithmetic, x axis)."""
        c = np.floor(_np_remainder(np.asarray(x, dtype=np.float64) - 0.0, self.Lx)
                     / self.width).astype(np.int64)
        return np.clip(c, 0, self.ncx - 1)

    def owner(self, x):
        return self._owner[self.columns(x)]

    def first_col(self, r):
        return self.bounds[r]

    def last_col(self, r):
        return self.bounds[r + 1] - 1


class LocalDomain:
    """The atoms one rank owns (global ids, state) plus its ghost bookkeeping."""

    def __init__(self, ids, positions, velocities, species, masses):
        self.ids = ids                    # int64 (n_own,)   global ids, host
        self.pos = positions              # (n_own, 3) float64 tensor (engine device)
        self.vel = velocities             # (n_own, 3)
        self.species = species            # (n_own,) int32 tensor
        self.masses = masses              # (n_own,) float64 tensor (per atom)
        self.send_left = None             # owned indices sent to rank-1 (their right ghosts)
        self.send_right = None            # owned indices sent to rank+1 (their left ghosts)
        self.n_ghost_left = 0
        self.n_ghost_right = 0
        self.ghost_ids = None
        self.ghost_species = None

    @property
    def n_owned(self):
        return int(self.pos.shape[0])


def scatter_state(decomp, state, rank, device):
    """Initial distribution: every rank takes the atoms in its columns (all
    ranks see the same global state, e.g. a seeded generator)."""
    own = decomp.owner(state.positions[:, 0]) == rank
    ids = np.nonzero(own)[0].astype(np.int64)
    t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)
    return LocalDomain(ids, t(state.positions[ids], torch.float64),
                       t(state.velocities[ids], torch.float64),
                       t(state.species[ids], torch.int32),
                       t(state.atom_masses[ids], torch.float64))


def _padded(shape):
    # zero-row messages are sent as one dummy row (backends reject empty P2P)
    return (max(shape[0], 1),) + tuple(shape[1:])


_COMM_DEVICE = {}  # process-wide override: exchange through this device (e.g. "cpu" for gloo)


def _exchange(sends, recv_shapes, dtype, device, left, right):
    """Two-way P2P with the left and right ranks.  sends: (to_left, to_right)
    tensors; recv_shapes: (from_left, from_right) row counts x width.  Message
    order per peer is fixed (to_left before to_right), which also resolves the
    two-rank ring where left == right.  Returns (from_left, from_right)."""
    comm = _COMM_DEVICE.get("device")
    if comm is not None and str(comm) != str(device):
        fl, fr = _exchange(tuple(t.to(comm) for t in sends), recv_shapes, dtype, comm, left,
                           right)
        return fl.to(device), fr.to(device)
    bufs = []
    for t in sends:
        t = t.contiguous()
        if t.shape[0] == 0:
            t = torch.zeros(_padded(tuple(t.shape)), dtype=dtype, device=device)
        bufs.append(t)
    from_left = torch.empty(_padded(recv_shapes[0]), dtype=dtype, device=device)
    from_right = torch.empty(_padded(recv_shapes[1]), dtype=dtype, device=device)
    ops = [dist.P2POp(dist.isend, bufs[0], left),
           dist.P2POp(dist.irecv, from_right, right),
           dist.P2POp(dist.isend, bufs[1], right),
           dist.P2POp(dist.irecv, from_left, left)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    return from_left[:recv_shapes[0][0]], from_right[:recv_shapes[1][0]]


def _exchange_into(sends, recvs, left, right):
    """_exchange with caller-owned receive buffers (contiguous row blocks,
    written in place), as the per-step halos use them: no allocation, no
    concatenation.  Zero-row messages and the gloo routing take _exchange
    (both ends of a zero-row message do, so the padding stays matched)."""
    dev = recvs[0].device
    comm = _COMM_DEVICE.get("device")
    if (comm is not None and str(comm) != str(dev)) or \
            any(t.shape[0] == 0 for t in (*sends, *recvs)):
        fl, fr = _exchange(sends, (tuple(recvs[0].shape), tuple(recvs[1].shape)), recvs[0].dtype,
                           dev, left, right)
        recvs[0].copy_(fl)
        recvs[1].copy_(fr)
        return
    ops = [dist.P2POp(dist.isend, sends[0], left),
           dist.P2POp(dist.irecv, recvs[1], right),
           dist.P2POp(dist.isend, sends[1], right),
           dist.P2POp(dist.irecv, recvs[0], left)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()


def _exchange_counts(a_left, a_right, device, left, right):
    s = (torch.tensor([a_left], dtype=torch.int64, device=device),
         torch.tensor([a_right], dtype=torch.int64, device=device))
    fl, fr = _exchange(s, ((1,), (1,)), torch.int64, device, left, right)
    return int(fl.item()), int(fr.item())


class DecomposedForceField:
    """Halo exchange + per-rank engine + reverse forces + all-reduce.

    `engine` implements rebuild(pos_local, species_local, n_owned, box) and
    compute(pos_local, species_local) -> (forces_local (n_local,3) tensor,
    result tensor [E, W6]) on the domain's device."""

    def __init__(self, decomp, box, engine, rank, nranks, device):
        self.decomp = decomp
        self.box = box
        self.engine = engine
        self.rank = rank
        self.nranks = nranks
        self.device = device
        self.left = (rank - 1) % nranks
        self.right = (rank + 1) % nranks
        self.rebuilds = 0

    # ---- rebuild: migration, send lists, ghost identities ----
    def migrate(self, dom):
        """Hand atoms whose column now belongs to a neighbour over to it."""
        x = dom.pos[:, 0].detach().cpu().numpy()
        own = self.decomp.owner(x)
        to_l = np.nonzero(own == self.left)[0] if self.nranks > 1 else np.zeros(0, np.int64)
        to_r = np.nonzero((own == self.right) & (own != self.left))[0] if self.nranks > 1 \
            else np.zeros(0, np.int64)
        stray = np.nonzero((own != self.rank) & (own != self.left) & (own != self.right))[0]
        if stray.size:
            raise ConfigurationError("an atom moved more than one slab between rebuilds")
        keep = np.nonzero(own == self.rank)[0]
        if self.nranks == 1:
            return dom
        dev = self.device
        nl_, nr_ = _exchange_counts(len(to_l), len(to_r), dev, self.left, self.right)
        idx = lambda a: torch.as_tensor(a, dtype=torch.long, device=dev)

        def pack(sel):
            s = idx(sel)
            f = torch.cat([dom.pos[s], dom.vel[s], dom.masses[s, None],
                           dom.species[s, None].to(torch.float64),
                           torch.as_tensor(dom.ids[sel], dtype=torch.float64, device=dev)[:, None]],
                          dim=1)
            return f

        fl, fr = _exchange((pack(to_l), pack(to_r)), ((nl_, 9), (nr_, 9)), torch.float64, dev,
                           self.left, self.right)
        k = idx(keep)
        inc = torch.cat([fl, fr], dim=0)
        dom.pos = torch.cat([dom.pos[k], inc[:, 0:3]], dim=0).contiguous()
        dom.vel = torch.cat([dom.vel[k], inc[:, 3:6]], dim=0).contiguous()
        dom.masses = torch.cat([dom.masses[k], inc[:, 6]], dim=0).contiguous()
        dom.species = torch.cat([dom.species[k], inc[:, 7].to(torch.int32)], dim=0).contiguous()
        dom.ids = np.concatenate([dom.ids[keep], inc[:, 8].cpu().numpy().astype(np.int64)])
        return dom

    def rebuild(self, dom):
        dom = self.migrate(dom)
        d = self.decomp
        x = dom.pos[:, 0].detach().cpu().numpy()
        col = d.columns(x)
        dom.send_left = np.nonzero(col == d.first_col(self.rank))[0]
        dom.send_right = np.nonzero(col == d.last_col(self.rank))[0]
        if self.nranks > 1:
            dev = self.device
            ngl, ngr = _exchange_counts(len(dom.send_left), len(dom.send_right), dev,
                                        self.left, self.right)
            # from_left = rank-1's right-column atoms = my left ghosts
            dom.n_ghost_left, dom.n_ghost_right = ngl, ngr
            idl = torch.as_tensor(dom.send_left, dtype=torch.long, device=dev)
            idr = torch.as_tensor(dom.send_right, dtype=torch.long, device=dev)
            meta = lambda sel: torch.stack(
                [torch.as_tensor(dom.ids, dtype=torch.float64, device=dev)[sel],
                 dom.species[sel].to(torch.float64)], dim=1)
            gl, gr = _exchange((meta(idl), meta(idr)), ((ngl, 2), (ngr, 2)), torch.float64, dev,
                               self.left, self.right)
            g = torch.cat([gl, gr], dim=0)
            dom.ghost_ids = g[:, 0].cpu().numpy().astype(np.int64)
            dom.ghost_species = g[:, 1].to(torch.int32).contiguous()
            dom._idl, dom._idr = idl, idr
        else:
            dom.n_ghost_left = dom.n_ghost_right = 0
            dom.ghost_ids = np.zeros(0, np.int64)
            dom.ghost_species = dom.species[:0]
        self.rebuilds += 1
        # per-step buffers (fixed until the next rebuild): [owned | left ghosts |
        # right ghosts] positions, the packed send rows and the returning forces;
        # species of [owned | ghosts] only change at a rebuild
        if self.nranks > 1:
            nsend = len(dom.send_left) + len(dom.send_right)
            dom._idx_send = torch.cat([dom._idl, dom._idr]).contiguous()
            dom._pos_l = torch.empty((dom.n_owned + dom.n_ghost_left + dom.n_ghost_right, 3),
                                     dtype=torch.float64, device=self.device)
            dom._send = torch.empty((nsend, 3), dtype=torch.float64, device=self.device)
            dom._back = torch.empty((nsend, 3), dtype=torch.float64, device=self.device)
        pos_l = self.halo_positions(dom)
        dom._sp_l = torch.cat([dom.species, dom.ghost_species]).contiguous()
        self.engine.rebuild(pos_l, dom._sp_l, dom.n_owned, self.box)
        return dom

    # ---- every evaluation ----
    def halo_positions(self, dom):
        """[owned | left ghosts | right ghosts] positions (forward halo)."""
        if self.nranks == 1:
            return dom.pos
        n, ngl = dom.n_owned, dom.n_ghost_left
        pos_l, send, nsl = dom._pos_l, dom._send, len(dom.send_left)
        pos_l[:n].copy_(dom.pos)
        torch.index_select(dom.pos, 0, dom._idx_send, out=send)
        _exchange_into((send[:nsl], send[nsl:]), (pos_l[n:n + ngl], pos_l[n + ngl:]),
                       self.left, self.right)
        return pos_l

    def __call__(self, dom):
        """Forces on the owned atoms, global energy and virial.  The returned
        force tensor is a view of the engine's buffer: valid until the next
        call (copy it to keep it)."""
        pos_l = self.halo_positions(dom)
        sp_l = getattr(dom, "_sp_l", None)
        if sp_l is None:
            sp_l = torch.cat([dom.species, dom.ghost_species]).contiguous() \
                if self.nranks > 1 else dom.species
        forces_l, result = self.engine.compute(pos_l, sp_l)
        n = dom.n_owned
        f = forces_l[:n]
        if self.nranks > 1:
            # reverse halo: forces on my left ghosts belong to rank-1's right
            # column atoms and vice versa; from_left carries forces on my
            # left-column atoms (rank-1's right ghosts)
            ngl, nsl, back = dom.n_ghost_left, len(dom.send_left), dom._back
            _exchange_into((forces_l[n:n + ngl], forces_l[n + ngl:]), (back[:nsl], back[nsl:]),
                           self.left, self.right)
            f.index_add_(0, dom._idx_send, back)
            comm = _COMM_DEVICE.get("device")
            if comm is not None and str(comm) != str(self.device):
                r = result.to(comm)
                dist.all_reduce(r)
                result.copy_(r)
            else:
                dist.all_reduce(result)
        return f, result


class B200Engine:
    """Per-rank force engine on the sm_100a kernels (device tensors)."""

    def __init__(self, params, skin=0.3, device=0, precision="double", scatter="atomic"):
        from . import _native
        self.native = _native
        self.ctx = _native.default_context(device)
        self.ctx.set_table(params)
        self.params = params
        self.skin = skin
        self.prec = _native.PRECISION[precision]
        self.scat = _native.SCATTER[scatter]
        self.nl = _native.NList(self.ctx)
        self.device = torch.device("cuda", device)

    def rebuild(self, pos_l, sp_l, n_owned, box):
        P = self.native.ptr
        L = np.ascontiguousarray(np.asarray(box.lengths, dtype=np.float64))
        per = np.ascontiguousarray(np.asarray(box.periodic, dtype=np.int32))
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)
        self.ctx.check(self.ctx.lib.tb_build_neighbors_owned(
            self.ctx.handle, self.nl.handle, pos_l.shape[0], n_owned, P(pos_l), P(L), P(per),
            float(self.params.r_cut), float(self.skin)), "tb_build_neighbors_owned")

    def compute(self, pos_l, sp_l):
        """Forces on [owned | ghosts] and [E, W6] into engine-owned buffers
        (reused while the atom count is unchanged: capturable in a graph)."""
        P = self.native.ptr
        n = pos_l.shape[0]
        if getattr(self, "_n", None) != n:
            self._forces = torch.empty((n, 3), dtype=torch.float64, device=self.device)
            self._result = torch.zeros(8, dtype=torch.float64, device=self.device)
            self._n = n
        self.ctx.check(self.ctx.lib.tb_compute_device(
            self.ctx.handle, self.nl.handle, P(pos_l), P(sp_l), float(self.params.r_cut),
            self.prec, self.scat, P(self._forces), None, P(self._result), None),
            "tb_compute_device")
        return self._forces, self._result[:7]


def set_comm_device(device):
    """Route the P2P/all-reduce traffic through `device` (e.g. "cpu" when the
    process group is gloo but the domain lives on a GPU)."""
    _COMM_DEVICE["device"] = device


def gather_global(dom, forces_owned, n_global, device):
    """All-gather owned forces into the global atom order (tests/diagnostics)."""
    comm = _COMM_DEVICE.get("device") or device
    out = torch.zeros((n_global, 3), dtype=torch.float64, device=comm)
    out[torch.as_tensor(dom.ids, dtype=torch.long, device=comm)] = forces_owned.to(comm)
    dist.all_reduce(out)
    return out.to(device)
