"""ctypes binding of lib/libtersoff_b200.so (C ABI: include/tersoff_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, every entry point raises NativeUnavailable.  Status codes map onto
the reference's exception classes (errors.py:9-14): TB_ERR_CONFIG ->
ConfigurationError, TB_ERR_INPUT -> InputError.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import ConfigurationError, InputError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TB_LIB_PATH") or os.path.join(_HERE, "lib", "libtersoff_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "tersoff_b200.h")

TB_OK, TB_ERR_CONFIG, TB_ERR_INPUT, TB_ERR_CUDA, TB_ERR_ARG, TB_ERR_UNSUPPORTED = range(6)
PRECISION = {"double": 0, "single": 1, "mixed": 1}
SCATTER = {"atomic": 0, "gather": 1}
NSTATS = 6
OPT_TILE_KERNEL = 1
OPT_LIST_MARGIN = 2  # percent of spare list entries / warp chunks (tb_md_run)
OPT_LIVE_PACK = 3  # 0 off / 1 on / 2 auto: rows cut to r < r_cut and re-chunked per evaluation
OPT_MD_LOOSE_SKIN = 4  # tb_md_run list skin extra in 1/100 A (default 30; 0 = exact list)
OPT_REPACK_MARGIN = 5  # live repack margin in 1/1000 A (default 1; 0 = repack every evaluation)
OPT_STREAM_RANGE = 6  # tb_compute with pinned host buffers: atoms per streamed range (default 131072; 0 = off)
OPT_ROW_KERNEL = 7  # atom-per-lane kernel for rows of <= 4 entries (one species, lam3 = 0); 0 = warp kernel only

# symbol -> (restype, argtypes); the exported surface of the C ABI
_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double
SIGNATURES = {
    "tb_create": (_I, [_I, ctypes.POINTER(_P)]),
    "tb_destroy": (None, [_P]),
    "tb_last_error": (ctypes.c_char_p, [_P]),
    "tb_set_stream": (_I, [_P, _P]),
    "tb_set_option": (_I, [_P, _I, _I]),
    "tb_synchronize": (_I, [_P]),
    "tb_set_params": (_I, [_P, _I, _P, _P, _P]),
    "tb_nlist_create": (_I, [_P, ctypes.POINTER(_P)]),
    "tb_nlist_destroy": (None, [_P]),
    "tb_build_neighbors": (_I, [_P, _P, _I64, _P, _P, _P, _D, _D]),
    "tb_build_neighbors_owned": (_I, [_P, _P, _I64, _I64, _P, _P, _P, _D, _D]),
    "tb_nlist_info": (_I, [_P, _P, _P, _P]),
    "tb_nlist_export": (_I, [_P, _P, _P, _P]),
    "tb_needs_rebuild": (_I, [_P, _P, _P, _P]),
    "tb_compute": (_I, [_P, _P, _P, _P, _D, _I, _I, _P, _P, _P, _P, _P]),
    "tb_compute_device": (_I, [_P, _P, _P, _P, _D, _I, _I, _P, _P, _P, _P]),
    "tb_check_errors": (_I, [_P]),
    "tb_md_step": (_I, [_P, _P, _I64, _P, _P, _P, _P, _P, _P, _P, _D, _D, _D, _D, _I, _I,
                        _I, _P, _P, _P]),
    "tb_md_run": (_I, [_P, _P, _I64, _P, _P, _P, _P, _P, _D, _D, _D, _D, _I, _I, _I, _I64, _I,
                       _P, _P, _P]),
    "tb_nlist_rebuild_device": (_I, [_P, _P, _P, _P, _I]),
    "tb_nlist_lanes": (_I, [_P, _P, _P]),
    "tb_nlist_refilter": (_I, [_P, _P]),
    "tb_nlist_import": (_I, [_P, _P, _I64, _P, _P, _P, _P, _P, _D, _D]),
    "tb_dd_create": (_I, [_P, _I, _I, _P, _P, _D, _D, ctypes.POINTER(_P)]),
    "tb_dd_destroy": (None, [_P]),
    "tb_dd_load": (_I, [_P, _I64, _P, _P, _P, _P, _P]),
    "tb_dd_counts": (_I, [_P, _P]),
    "tb_dd_buffer": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "tb_dd_recv_buffer": (_I, [_P, _I64, _I, ctypes.POINTER(_P)]),
    "tb_dd_migrate_pack": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "tb_dd_migrate_unpack": (_I, [_P, _I64, _I64]),
    "tb_dd_halo_pack": (_I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "tb_dd_halo_unpack": (_I, [_P, _I64, _I64]),
    "tb_dd_pack_positions": (_I, [_P]),
    "tb_dd_build": (_I, [_P, _P]),
    "tb_dd_compute": (_I, [_P, _P, _I, _I, _P, _P]),
    "tb_dd_reverse_add": (_I, [_P]),
    "tb_dd_kick_drift": (_I, [_P, _P, _D, _D, _P]),
    "tb_dd_kick": (_I, [_P, _D, _D, _P]),
    "tb_dd_export": (_I, [_P, _P, _P, _P, _P]),
    "tb_profile": (_I, [_P, _I]),
    "tb_profile_read": (_I, [_P, _P, _P]),
    "tb_measure_peak": (_I, [_P, _I, ctypes.POINTER(_D)]),
    "tb_version": (ctypes.c_char_p, []),
}


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built or no GPU is usable (no fallback)."""


_lib = None
_lock = threading.Lock()


def load_library():
    """Load the shared library and bind every declared symbol."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeUnavailable(
                    f"{LIB_PATH} is missing: build it with "
                    f"`python -c 'import __graft_entry__ as g; g.build()'` "
                    f"(make -C paper_1710_00882_b200/csrc)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def version():
    return load_library().tb_version().decode()


def ptr(a):
    """Raw pointer of a numpy array or torch tensor (None passes through)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        # (the array interface is ~10x cheaper than ndarray.ctypes per call)
        return a.__array_interface__["data"][0]
    return a.data_ptr()


class Context:
    """One tb_context: a device, a stream and the uploaded parameter table."""

    def __init__(self, device=0):
        lib = load_library()
        h = ctypes.c_void_p()
        rc = lib.tb_create(int(device), ctypes.byref(h))
        if rc != TB_OK or not h:
            raise NativeUnavailable(f"tb_create(device={device}) failed with status {rc}: "
                                    f"no usable CUDA device")
        self.lib = lib
        self.handle = h
        self.device = int(device)
        self._table_key = None
        self.r_cut = None

    def close(self):
        if getattr(self, "handle", None):
            self.lib.tb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc, what=""):
        if rc == TB_OK:
            return
        msg = self.lib.tb_last_error(self.handle).decode()
        if rc == TB_ERR_CONFIG:
            raise ConfigurationError(msg)
        if rc == TB_ERR_INPUT:
            raise InputError(msg)
        raise RuntimeError(f"{what}: {msg} (status {rc})")

    def set_stream(self, stream_ptr):
        self.check(self.lib.tb_set_stream(self.handle, ctypes.c_void_p(stream_ptr or 0)),
                   "tb_set_stream")

    def set_option(self, option, value):
        self.check(self.lib.tb_set_option(self.handle, int(option), int(value)), "tb_set_option")

    def synchronize(self):
        self.check(self.lib.tb_synchronize(self.handle), "tb_synchronize")

    def set_table(self, table):
        """Upload a ParamTable (flattened as ParamTable.views, potential.py:127-155)."""
        key = id(table)
        if key == self._table_key:
            return self.r_cut
        v = table.views("double")
        pair = np.ascontiguousarray(v["pair_matrix"], dtype=np.float64)
        trip = np.ascontiguousarray(v["trip_matrix"], dtype=np.float64)
        rc_out = ctypes.c_double()
        self.check(self.lib.tb_set_params(self.handle, table.nspecies, ptr(pair), ptr(trip),
                                          ctypes.byref(rc_out)), "tb_set_params")
        self._table_key = key
        self._table_ref = table
        self.r_cut = rc_out.value
        return self.r_cut


_contexts = {}


def default_context(device=0):
    """Process-wide context per device (created lazily)."""
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts[device] = ctx
    return ctx


class NList:
    """Owning wrapper of a tb_nlist bound to a Context."""

    def __init__(self, ctx):
        self.ctx = ctx
        h = ctypes.c_void_p()
        ctx.check(ctx.lib.tb_nlist_create(ctx.handle, ctypes.byref(h)), "tb_nlist_create")
        self.handle = h

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.tb_nlist_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def info(self):
        n, m, mr = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self.ctx.check(self.ctx.lib.tb_nlist_info(self.handle, ctypes.byref(n), ctypes.byref(m),
                                                  ctypes.byref(mr)), "tb_nlist_info")
        return n.value, m.value, mr.value
