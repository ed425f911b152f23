"""Quick kernel timing on config 2 (64k Si): fp64 + mixed, atomic + gather,
warp + tile paths.  Usage: TB_LIB_PATH=... python tools/kbench.py [tag]"""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
cfg = int(os.environ.get("KB_CONFIG", "2"))
st, tn = structures.config(cfg, small=os.environ.get("KB_SMALL") == "1")
t = B.builtin_params(tn)
n = st.natoms
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = _native.default_context(0); ctx.set_stream(s.cuda_stream); ctx.set_table(t)
if os.environ.get("KB_LIVE"):
    ctx.set_option(_native.OPT_LIVE_PACK, int(os.environ["KB_LIVE"]))
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda"); stt = torch.zeros(6, dtype=torch.int64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {"tag": sys.argv[1] if len(sys.argv) > 1 else "", "n": n, "entries": nl.n_entries, "max_row": nl.max_row}
for path in ("warp", "tile"):
    ctx.set_option(_native.OPT_TILE_KERNEL, path == "tile")
    for prec in (0, 1):
        for scat in (0, 1):
            def step():
                ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, scat, P(f), P(pa), P(res), None))
            for _ in range(5): step()
            torch.cuda.synchronize()
            ctx.lib.tb_profile(ctx.handle, 1)
            K = 50
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
            for a_, b_ in ev:
                flush.zero_(); a_.record(s); step(); b_.record(s)
            torch.cuda.synchronize()
            ctx.lib.tb_profile(ctx.handle, 0)
            tot = ctypes.c_double(); l = ctypes.c_int64()
            ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
            step_ms = sum(a_.elapsed_time(b_) for a_, b_ in ev) / K
            out[f"{path}/{'f64' if prec == 0 else 'mix'}/{'atomic' if scat == 0 else 'gather'}"] = \
                {"kernel_us": round(1e3 * tot.value / l.value, 2), "step_us": round(1e3 * step_ms, 2)}
ctx.set_option(_native.OPT_TILE_KERNEL, 0)
print(json.dumps(out))
