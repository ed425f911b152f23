"""The Tersoff energy/force/virial entry points, on B200.

Drop-in for reference pkg/src/tersoffmd/kernels.py:
  make_variant / KernelVariant   (:43-77)   selector (tag, backend); tag "B200"
                                            or any reference tag -- all run the
                                            same sm_100a kernel
  ForceEnergyResult              (:80-92)   + .virial (xx,yy,zz,xy,xz,yz)
  compute(state, nl, params, variant, threads=1)   (:517-527)
  kernel_function / count_flops_and_visits         (:530-544)

compute() takes this package's device NeighborList or the reference's own
NeighborList (numpy CSR; imported once per list object with
tb_nlist_import), and the reference's KernelVariant(tag, backend) objects as
well as this package's.  One C-ABI crossing per evaluation (tb_compute):
host positions are copied to HBM, the kernel re-packs the skin list at the
current positions and evaluates E, F, per-atom E and the virial.  There is no
CPU path: a missing library raises NativeUnavailable.

Instrumentation counters follow the reference's contract
(pkg/tests/test_kernels.py:218-249): zeta_visits = sum n_i^2 over the packed
rows for single-pass variants and 2 sum n_i^2 for "Reference" (Algorithm 1
walks k twice, kernels.py:172-243); the scalar tags (Reference, ScalarOpt)
report no lanes (lane_utilization None) and no gathers; the lane tags (VecJ,
VecI, B200) report the warp lanes of the B200 chunk layout: lane_total = 32 x
warp chunks, lane_active = lanes holding a list entry, gathers = one neighbour
gather per active lane.
"""

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigurationError
from .neighbor import NeighborList, _box_args, _positions

REFERENCE_TAGS = ("Reference", "ScalarOpt", "VecJ", "VecI")
KERNEL_TAGS = ("B200",) + REFERENCE_TAGS
SCALAR_TAGS = ("Reference", "ScalarOpt")
PRECISIONS = ("double", "single")


@dataclass(frozen=True)
class DeviceBackend:
    """Execution model in the shape of the reference's simd.Backend
    (simd.py:151-181): a warp of 32 lanes."""

    name: str = "sm_100a"
    width: int = 32
    precision: str = "double"
    strict: bool = False


@dataclass(frozen=True)
class KernelVariant:
    """(tag, backend) as the reference's selector, plus B200 options:
    precision "double" (fp64) or "single" (fp64 positions/displacements/
    accumulators, fp32 potential math, kernels.py:154-165) -- taken from the
    backend when not given; scatter "atomic" (red.global.add.f64 of the
    neighbour forces) or "gather" (per-entry buffer + deterministic gather)."""

    tag: str = "B200"
    backend: object = None
    precision: str = None
    scatter: str = "atomic"
    device: int = 0

    def __post_init__(self):
        if self.tag not in KERNEL_TAGS:
            raise ConfigurationError(f"unknown kernel tag {self.tag!r}")
        prec = self.precision or getattr(self.backend, "precision", None) or "double"
        if prec not in PRECISIONS:
            raise ConfigurationError(f"unknown precision {prec!r}")
        if self.scatter not in _native.SCATTER:
            raise ConfigurationError(f"unknown scatter mode {self.scatter!r}")
        object.__setattr__(self, "precision", prec)
        if self.backend is None:
            object.__setattr__(self, "backend", DeviceBackend(precision=prec))

    def describe(self):
        return f"{self.tag}[sm_100a,{self.precision},{self.scatter}]"


def make_variant(tag="B200", backend="scalar", width=None, precision="double", strict=False,
                 scatter="atomic", device=0):
    """Mirror of kernels.make_variant (kernels.py:73-77).  A reference Backend
    object supplies the precision; backend names / width / strict describe the
    reference's CPU lane emulation and are accepted for compatibility."""
    if backend is not None and not isinstance(backend, str):
        return KernelVariant(tag, backend, getattr(backend, "precision", precision), scatter,
                             device)
    return KernelVariant(tag, None, precision, scatter, device)


def resolve_variant(variant):
    """This package's KernelVariant for None, one of ours, or the reference's
    KernelVariant(tag, backend) (duck-typed: .tag and .precision/.backend)."""
    if variant is None:
        return KernelVariant()
    if isinstance(variant, KernelVariant):
        return variant
    tag = getattr(variant, "tag", None)
    prec = getattr(variant, "precision", None) or \
        getattr(getattr(variant, "backend", None), "precision", None)
    return KernelVariant(tag, getattr(variant, "backend", None), prec,
                         getattr(variant, "scatter", "atomic"), getattr(variant, "device", 0))


@dataclass
class ForceEnergyResult:
    forces: np.ndarray
    potential_energy: float
    per_atom_energy: np.ndarray
    stats: dict
    virial: np.ndarray = field(default_factory=lambda: np.zeros(6))

    @property
    def lane_utilization(self):
        total = self.stats.get("lane_total", 0)
        if total == 0:
            return None
        return self.stats["lane_active"] / total


def _species_i32(state, n):
    sp = state.species
    if isinstance(sp, np.ndarray) or sp is None or isinstance(sp, (list, tuple)):
        sp = np.zeros(n, np.int32) if sp is None else np.asarray(sp)
        if sp.shape != (n,):
            raise ConfigurationError(f"species shape {sp.shape} does not match {n} atoms")
        return np.ascontiguousarray(sp, dtype=np.int32)
    if sp.dtype != __import__("torch").int32:
        raise ConfigurationError("device species must be an int32 tensor")
    return sp


_PTRS = {}  # id(array) -> (weakref, shape, raw pointer): per-call pointer lookups cost ~1 us each


def _ptr(a):
    """Raw data pointer of an array or tensor, cached per live numpy array (a
    changed shape -- the only way a live array's buffer can move -- misses)."""
    if not isinstance(a, np.ndarray):
        return _native.ptr(a)
    e = _PTRS.get(id(a))
    if e is not None and e[0]() is a and e[1] == a.shape:
        return e[2]
    p = _native.ptr(a)
    if len(_PTRS) > 64:
        _PTRS.clear()
    _PTRS[id(a)] = (weakref.ref(a), a.shape, p)
    return p


class _Scratch:
    """Per-context host buffers for the scalar results of tb_compute."""

    def __init__(self):
        self.energy = np.zeros(1)
        self.virial = np.zeros(6)
        self.stats = np.zeros(_native.NSTATS, dtype=np.int64)
        self.p = (_native.ptr(self.energy), _native.ptr(self.virial), _native.ptr(self.stats))
        self.chunks, self.used = ctypes.c_int64(), ctypes.c_int64()
        self.refs = (ctypes.byref(self.chunks), ctypes.byref(self.used))


# the reference's NeighborList objects -> imported device lists
_IMPORTED = weakref.WeakKeyDictionary()


def device_list(nl, state, device=0):
    """This package's NeighborList for `nl`: itself, or the device import of a
    reference NeighborList (offsets / neighbors / reference_positions CSR,
    neighbor.py:170-191), cached for the lifetime of that object."""
    if isinstance(nl, NeighborList):
        return nl
    try:
        hit = _IMPORTED.get(nl)
    except TypeError:  # not weak-referenceable
        hit = None
    if hit is not None and hit[1] is nl.offsets and hit[2] is nl.neighbors:
        return hit[0]
    off = np.ascontiguousarray(nl.offsets, dtype=np.int64)
    nbr = np.ascontiguousarray(nl.neighbors, dtype=np.int64)
    ref = np.ascontiguousarray(nl.reference_positions, dtype=np.float64)
    n = off.shape[0] - 1
    skin = float(getattr(nl, "skin", 0.0))
    r_cut = float(getattr(nl, "r_cut", nl.build_cutoff - skin))
    ctx = _native.default_context(device)
    h = _native.NList(ctx)
    L, per = _box_args(state.box)
    ctx.check(ctx.lib.tb_nlist_import(ctx.handle, h.handle, n, _native.ptr(off),
                                      _native.ptr(nbr), _native.ptr(ref), _native.ptr(L),
                                      _native.ptr(per), r_cut, skin), "tb_nlist_import")
    dl = NeighborList(h, n, r_cut + skin, r_cut, skin, ref, state.box)
    dl._csr = (off, nbr)
    try:
        _IMPORTED[nl] = (dl, nl.offsets, nl.neighbors)
    except TypeError:
        pass
    return dl


def _stats(tag, counts, chunks, used):
    nsq = int(counts[0])
    lanes = tag not in SCALAR_TAGS
    return {"zeta_visits": 2 * nsq if tag == "Reference" else nsq,
            "gathers": int(used) if lanes else 0,
            "lane_active": int(used) if lanes else 0,
            "lane_total": 32 * int(chunks) if lanes else 0,
            "packed_pairs": int(counts[1]), "live_pairs": int(counts[2]),
            "live_triplets": int(counts[3]), "taper_pairs": int(counts[4]),
            "taper_triplets": int(counts[5])}


def compute(state, nl, params, variant=None, threads=1, out=None):
    """One E+F(+virial) evaluation (kernels.py:517-527).

    state.positions may be a numpy array (copied to the GPU inside the call)
    or a contiguous float64 CUDA tensor (used in place; forces then come back
    as a CUDA tensor).  `threads` is accepted for signature compatibility.
    `out` (extension): a ForceEnergyResult whose forces / per_atom_energy
    arrays are overwritten instead of allocating new ones (e.g. pinned host
    buffers for a streaming driver); it is returned updated."""
    variant = resolve_variant(variant)
    pos = _positions(state)
    nl = device_list(nl, state, variant.device if isinstance(pos, np.ndarray)
                     else pos.device.index)
    ctx = nl.context
    ctx.set_table(params)
    n = int(pos.shape[0])
    if n != nl.natoms:
        raise ConfigurationError(f"state has {n} atoms but the neighbor list {nl.natoms}")
    sp = _species_i32(state, n)
    on_device = not isinstance(pos, np.ndarray)
    if out is not None:
        forces, per_atom = out.forces, out.per_atom_energy
        if tuple(forces.shape) != (n, 3) or tuple(per_atom.shape) != (n,):
            raise ConfigurationError("out buffers do not match the number of atoms")
    elif on_device:
        import torch
        forces = torch.empty((n, 3), dtype=torch.float64, device=pos.device)
        per_atom = torch.empty(n, dtype=torch.float64, device=pos.device)
    else:
        forces = np.empty((n, 3))
        per_atom = np.empty(n)
    scr = getattr(ctx, "_scratch", None)
    if scr is None:
        scr = ctx._scratch = _Scratch()
    lib = ctx.lib
    rc = lib.tb_compute(ctx.handle, nl._nl.handle, _ptr(pos), _ptr(sp), float(params.r_cut),
                        _native.PRECISION[variant.precision], _native.SCATTER[variant.scatter],
                        _ptr(forces), _ptr(per_atom), *scr.p)
    if rc:
        ctx.check(rc, "tb_compute")
    rc = lib.tb_nlist_lanes(nl._nl.handle, *scr.refs)
    if rc:
        ctx.check(rc, "tb_nlist_lanes")
    st = _stats(variant.tag, scr.stats, scr.chunks.value, scr.used.value)
    energy, virial = float(scr.energy[0]), scr.virial.copy()
    if out is not None:
        out.potential_energy, out.stats, out.virial = energy, st, virial
        return out
    return ForceEnergyResult(forces, energy, per_atom, st, virial)


def kernel_function(variant, threads=1):
    """Bind a variant to a (state, nl, params) -> ForceEnergyResult call."""
    def fn(state, nl, params):
        return compute(state, nl, params, variant, threads)
    return fn


def count_flops_and_visits(state, nl, params, variant):
    """Run once and report the instrumentation counters (kernels.py:537-544),
    plus the live pair / triplet counts the roofline is charged on."""
    res = compute(state, nl, params, variant)
    return {"zeta_visits": res.stats["zeta_visits"], "gathers": res.stats["gathers"],
            "lane_utilization": res.lane_utilization,
            "live_pairs": res.stats["live_pairs"],
            "live_triplets": res.stats["live_triplets"]}
