"""Device-resident Verlet neighbour list with skin.

Drop-in for reference pkg/src/tersoffmd/neighbor.py:
  build_neighbor_list(state, r_cut, skin=0.3)  (:194-217) -> cell binning +
      full symmetric list on the GPU (kernels K1/K2 in csrc/tb_kernels.cuh);
      the pair set equals the reference's bit for bit.
  needs_rebuild(state, nl)                      (:220-229) -> K3 on the GPU.
  NeighborList                                  (:170-191) -> handle to the
      device CSR; .offsets / .neighbors export it as int64 numpy arrays.
  pack_adjacency(state, nl, r_cut)              (:330-360) -> the packed rows
      at current positions (for parity checks; the force kernel packs on the
      fly inside its own tile and never materialises this).
"""

import math

import numpy as np

from . import _native
from .errors import ConfigurationError, InputError


def _box_args(box):
    L = np.ascontiguousarray(np.asarray(box.lengths, dtype=np.float64).reshape(3))
    per = np.ascontiguousarray(np.asarray([bool(p) for p in box.periodic], dtype=np.int32))
    return L, per


def _positions(state):
    """float64 (n,3) C-contiguous positions: numpy array or CUDA tensor."""
    pos = state.positions
    if isinstance(pos, np.ndarray):
        if pos.dtype != np.float64 or not pos.flags.c_contiguous:
            pos = np.ascontiguousarray(pos, dtype=np.float64)
        return pos
    # torch tensor (device-resident path)
    if pos.dtype.is_floating_point and str(pos.dtype) == "torch.float64" and pos.is_contiguous():
        return pos
    raise ConfigurationError("device positions must be a contiguous float64 tensor")


class NeighborList:
    """Full symmetric neighbour list held on the GPU (CSR, rows ascending)."""

    def __init__(self, handle, n, build_cutoff, r_cut, skin, reference_positions, box):
        self._nl = handle
        self._n = n
        self.build_cutoff = build_cutoff
        self.r_cut = r_cut
        self.skin = skin
        self.reference_positions = reference_positions
        self.box = box
        self._csr = None

    @property
    def context(self):
        return self._nl.ctx

    @property
    def natoms(self):
        return self._n

    @property
    def n_entries(self):
        return self._nl.info()[1]

    @property
    def max_row(self):
        return self._nl.info()[2]

    def _export(self):
        if self._csr is None:
            n, m, _ = self._nl.info()
            off = np.zeros(n + 1, dtype=np.int64)
            nbr = np.zeros(max(m, 1), dtype=np.int64)
            ctx = self._nl.ctx
            ctx.check(ctx.lib.tb_nlist_export(ctx.handle, self._nl.handle, _native.ptr(off),
                                              _native.ptr(nbr)), "tb_nlist_export")
            self._csr = (off, nbr[:m])
        return self._csr

    @property
    def offsets(self):
        return self._export()[0]

    @property
    def neighbors(self):
        return self._export()[1]

    def row(self, i):
        off, nbr = self._export()
        return nbr[off[i]:off[i + 1]]

    def rebuild_on_device(self, positions, species, scatter="atomic"):
        """Rebuild in place at `positions` (cuda float64 (n,3)) with the
        device-side builder of the graph MD loop (tb_nlist_rebuild_device):
        same pair set and row order as build_neighbor_list."""
        ctx = self._nl.ctx
        sp = species if species.dtype == torch_int32() else species.to(torch_int32())
        ctx.check(ctx.lib.tb_nlist_rebuild_device(ctx.handle, self._nl.handle,
                                                  _native.ptr(positions), _native.ptr(sp),
                                                  _native.SCATTER[scatter]),
                  "tb_nlist_rebuild_device")
        self.reference_positions = positions.clone()
        self._csr = None
        return self


def torch_int32():
    import torch
    return torch.int32


def build_neighbor_list(state, r_cut, skin=0.3, device=None, reuse=None):
    """Full list at build_cutoff = r_cut + skin (neighbor.py:194-217).
    reuse (extension): a NeighborList whose device buffers are rebuilt in
    place (ForceField keeps one list alive across rebuilds)."""
    if skin < 0:
        raise ConfigurationError(f"negative skin {skin:g}")
    pos = _positions(state)
    if device is None:
        device = 0 if isinstance(pos, np.ndarray) else pos.device.index
    ctx = _native.default_context(device)
    nl = reuse._nl if reuse is not None and reuse._nl.ctx is ctx else _native.NList(ctx)
    L, per = _box_args(state.box)
    n = int(pos.shape[0])
    ctx.check(ctx.lib.tb_build_neighbors(ctx.handle, nl.handle, n, _native.ptr(pos),
                                         _native.ptr(L), _native.ptr(per), float(r_cut),
                                         float(skin)), "tb_build_neighbors")
    ref = pos.copy() if isinstance(pos, np.ndarray) else pos.clone()
    return NeighborList(nl, n, float(r_cut) + float(skin), float(r_cut), float(skin), ref,
                        state.box)


def needs_rebuild(state, nl):
    """True once any atom drifted more than skin/2 since the build
    (neighbor.py:220-229), evaluated on the GPU."""
    pos = _positions(state)
    out = np.zeros(1, dtype=np.int32)
    ctx = nl.context
    ctx.check(ctx.lib.tb_needs_rebuild(ctx.handle, nl._nl.handle, _native.ptr(pos),
                                       _native.ptr(out)), "tb_needs_rebuild")
    return bool(out[0])


class PackedAdjacency:
    """Packed rows at current positions (neighbor.py:259-327 data layout)."""

    def __init__(self, offsets, i, j, dx, dy, dz, r, r_cut):
        self.offsets, self.i, self.j = offsets, i, j
        self.dx, self.dy, self.dz, self.r = dx, dy, dz, r
        self.r_cut = r_cut

    @property
    def natoms(self):
        return self.offsets.shape[0] - 1

    @property
    def npairs(self):
        return self.j.shape[0]


def pack_adjacency(state, nl, r_cut=None):
    """Re-filter the skin list to r < r_cut at current positions
    (neighbor.py:330-360).  Uses the GPU list; the filter arithmetic is the
    reference's (min image, r2 = (dx^2 + dy^2) + dz^2).  Host-side helper for
    inspection and parity tests; the force kernel packs on the device."""
    if r_cut is None:
        r_cut = nl.r_cut
    if r_cut > nl.r_cut:
        raise ConfigurationError(
            f"cutoff {r_cut:g} A exceeds the {nl.r_cut:g} A the neighbor "
            f"list was built for")
    pos = np.asarray(state.positions if isinstance(state.positions, np.ndarray)
                     else state.positions.cpu().numpy(), dtype=np.float64)
    off, nbr = nl.offsets, nl.neighbors
    n = nl.natoms
    i_all = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    d = pos[nbr] - pos[i_all]
    for ax in range(3):
        if state.box.periodic[ax]:
            edge = state.box.lengths[ax]
            d[:, ax] -= edge * np.round(d[:, ax] / edge)
    r2 = (d * d).sum(axis=1)
    keep = r2 < r_cut * r_cut
    i_k, j_k, d_k = i_all[keep], nbr[keep], d[keep]
    if i_k.size and r2[keep].min() < 1e-16:
        at = int(np.argmin(r2[keep]))
        raise InputError(f"atoms {int(i_k[at])} and {int(j_k[at])} are coincident "
                         f"(r = {math.sqrt(r2[keep].min()):.3e} A)")
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(i_k, minlength=n), out=offsets[1:])
    return PackedAdjacency(offsets, i_k, j_k, np.ascontiguousarray(d_k[:, 0]),
                           np.ascontiguousarray(d_k[:, 1]), np.ascontiguousarray(d_k[:, 2]),
                           np.sqrt(r2[keep]), float(r_cut))
