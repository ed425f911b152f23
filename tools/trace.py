"""Per-warp timeline of the warp Tersoff kernel (debug build with -DTB_TRACE).
Usage: TB_LIB_PATH=paper_1710_00882_b200/lib/libtb_trace.so python tools/trace.py [config]"""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st, tn = structures.config(cfg)
t = B.builtin_params(tn)
n = st.natoms
ctx = _native.default_context(0); ctx.set_table(t)
s = torch.cuda.current_stream(); ctx.set_stream(s.cuda_stream)
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
lib = ctx.lib
lib.tb_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {}
for prec in (0, 1):
    for fl in (True, False):
        for _ in range(3):
            if fl:
                flush.zero_()
            lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, 0,
                                  P(f), P(pa), P(res), None)
        torch.cuda.synchronize()
        buf = np.zeros(4096 * 16, np.uint64)
        assert lib.tb_debug_trace(buf.ctypes.data, buf.nbytes) == 0
        blk = buf[-2048:].reshape(1024, 2).astype(np.int64)
        blk = blk[blk[:, 0] != 0]
        tr = buf.reshape(4096, 16).astype(np.int64)[:3968]
        nw = int(np.count_nonzero(tr[:, 0]))
        tr = tr[:nw]
        g0 = tr[:, 0] - tr[:, 0].min()
        gend = tr[:, 15] - tr[:, 0].min()
        ctx.lib.tb_profile(ctx.handle, 1)
        for _ in range(20):
            if fl:
                flush.zero_()
            lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, 0,
                                  P(f), P(pa), P(res), None)
        ctx.lib.tb_profile(ctx.handle, 0)
        tot = ctypes.c_double(); l = ctypes.c_int64()
        ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
        out[f"event_us_{prec}_{fl}"] = 1e3 * tot.value / l.value
        nd = tr[:, 14]
        clk = tr[:, 2:15]
        d_first = clk[:, 1] - clk[:, 0]
        later = [clk[w, k + 1] - clk[w, k] for w in range(nw) for k in range(1, min(nd[w], 12))]
        b0 = blk[:, 0].min()
        key = f"{'f64' if prec == 0 else 'mix'}/{'flush' if fl else 'warm'}"
        out[key + "/blocks"] = {"entry_ns_p50_max": [int(np.median(blk[:, 0] - b0)), int((blk[:, 0] - b0).max())],
                                "exit_ns_min_p50_max": [int((blk[:, 1] - b0).min()), int(np.median(blk[:, 1] - b0)), int((blk[:, 1] - b0).max())],
                                "first_warp_start_after_entry_ns": int(tr[:, 0].min() - b0)}
        out[key] = {
            "warps": nw, "chunks_per_warp": np.bincount(nd).tolist(),
            "start_ns_p50_p100": [int(np.median(g0)), int(g0.max())],
            "end_ns_p0_p50_p100": [int(gend.min()), int(np.median(gend)), int(gend.max())],
            "first_chunk_cycles_p50": int(np.median(d_first)),
            "later_chunk_cycles_p50": int(np.median(later)) if later else None,
            "warp_total_cycles_p50_max": [int(np.median(clk[np.arange(nw), np.minimum(nd, 12)] - clk[:, 0])),
                                          int((clk[np.arange(nw), np.minimum(nd, 12)] - clk[:, 0]).max())],
        }
print(json.dumps(out, indent=1))
