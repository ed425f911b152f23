"""The Tersoff energy/force/virial entry points, on B200.

Drop-in for reference pkg/src/tersoffmd/kernels.py:
  make_variant / KernelVariant   (:46-77)   selector; tag "B200" (the reference
                                            tags are accepted and all map onto
                                            the same sm_100a kernel)
  ForceEnergyResult              (:80-92)   + .virial (xx,yy,zz,xy,xz,yz)
  compute(state, nl, params, variant, threads=1)   (:517-527)
  kernel_function / count_flops_and_visits         (:530-544)

compute() crosses the C ABI once (tb_compute): host positions are copied to
HBM, the kernel re-packs the skin list at the current positions and
evaluates E, F, per-atom E and the virial, and the results come back.
There is no CPU path: a missing library raises NativeUnavailable.
"""

import ctypes
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigurationError
from .neighbor import _positions

REFERENCE_TAGS = ("Reference", "ScalarOpt", "VecJ", "VecI")
KERNEL_TAGS = ("B200",) + REFERENCE_TAGS
PRECISIONS = ("double", "single")


@dataclass(frozen=True)
class KernelVariant:
    """Kernel selector.  precision: "double" (fp64) or "single" (mixed: fp64
    positions/displacements/accumulators, fp32 potential math, as
    kernels.py:154-165).  scatter: "atomic" (red.global.add.f64 of the
    neighbour forces) or "gather" (per-entry buffer + deterministic gather)."""

    tag: str = "B200"
    precision: str = "double"
    scatter: str = "atomic"
    device: int = 0

    def __post_init__(self):
        if self.tag not in KERNEL_TAGS:
            raise ConfigurationError(f"unknown kernel tag {self.tag!r}")
        if self.precision not in PRECISIONS:
            raise ConfigurationError(f"unknown precision {self.precision!r}")
        if self.scatter not in _native.SCATTER:
            raise ConfigurationError(f"unknown scatter mode {self.scatter!r}")

    def describe(self):
        return f"{self.tag}[sm_100a,{self.precision},{self.scatter}]"

    @property
    def backend(self):
        """Execution model in the shape of the reference's simd.Backend
        (simd.py:151-181): name, lane width (a warp), precision."""
        return DeviceBackend("sm_100a", 32, self.precision)


@dataclass(frozen=True)
class DeviceBackend:
    name: str
    width: int
    precision: str
    strict: bool = False


def make_variant(tag="B200", backend=None, width=None, precision="double", strict=False,
                 scatter="atomic", device=0):
    """Mirror of kernels.make_variant (kernels.py:73-77).  backend/width/strict
    describe the reference's CPU lane emulation and are accepted for
    signature compatibility; the B200 kernel has one execution model."""
    if backend is not None and hasattr(backend, "precision"):
        precision = backend.precision
    return KernelVariant(tag, precision, scatter, device)


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
    if isinstance(sp, np.ndarray) or sp is None:
        sp = np.zeros(n, np.int32) if sp is None else sp
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


def compute(state, nl, params, variant=None, threads=1, out=None):
    """One E+F(+virial) evaluation (kernels.py:517-527).

    state.positions may be a numpy array (copied to the GPU inside the call)
    or a contiguous float64 CUDA tensor (used in place; forces then come back
    as a CUDA tensor).  `threads` is accepted for signature compatibility.
    `out` (extension): a ForceEnergyResult whose forces / per_atom_energy
    arrays are overwritten instead of allocating new ones (e.g. pinned host
    buffers for a streaming driver); it is returned updated."""
    variant = variant or KernelVariant()
    ctx = nl.context
    ctx.set_table(params)
    pos = _positions(state)
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
    stats = scr.stats.tolist()
    st = {"zeta_visits": stats[0], "gathers": 0,
          "lane_active": scr.used.value, "lane_total": 32 * scr.chunks.value,
          "packed_pairs": stats[1], "live_pairs": stats[2],
          "live_triplets": stats[3], "taper_pairs": stats[4],
          "taper_triplets": stats[5]}
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
    """Run once and report the work counters (kernels.py:537-544)."""
    res = compute(state, nl, params, variant)
    return {"zeta_visits": res.stats["zeta_visits"], "gathers": 0,
            "lane_utilization": res.lane_utilization,
            "live_pairs": res.stats["live_pairs"],
            "live_triplets": res.stats["live_triplets"]}
