"""Step timing with the evaluation captured in a CUDA graph (torch.cuda.graph).
Prints kernel-only time (profile events, non-graph) and graph-replay step time."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
cfg = int(os.environ.get("KB_CONFIG", "2"))
if os.environ.get("KB_CELLS"):
    st = structures.seed_velocities(structures.displace(structures.gen_diamond(int(os.environ["KB_CELLS"]), 5.431), 0.1, 1002), 1000.0, 2002)
    tn = "Si"
else:
    st, tn = structures.config(cfg)
t = B.builtin_params(tn)
n = st.natoms
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = _native.default_context(0); ctx.set_stream(s.cuda_stream); ctx.set_table(t)
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {"tag": sys.argv[1] if len(sys.argv) > 1 else "", "n": n}
for prec in (0, 1):
    for scat in (0, 1):
        def step():
            ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, scat, P(f), P(pa), P(res), None))
        for _ in range(5): step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        ctx.set_stream(s.cuda_stream)
        torch.cuda.synchronize()
        K = 100
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for a_, b_ in ev:
            flush.zero_(); a_.record(s); g.replay(); b_.record(s)
        torch.cuda.synchronize()
        gstep = sum(a_.elapsed_time(b_) for a_, b_ in ev) / K
        # back-to-back replays without flush (L2-warm throughput)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(K): g.replay()
        e1.record(s); torch.cuda.synchronize()
        warm = e0.elapsed_time(e1) / K
        ctx.lib.tb_profile(ctx.handle, 1)
        for _ in range(20):
            flush.zero_(); step()
        torch.cuda.synchronize(); ctx.lib.tb_profile(ctx.handle, 0)
        tot = ctypes.c_double(); l = ctypes.c_int64()
        ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
        out[f"{'f64' if prec == 0 else 'mix'}/{'atomic' if scat == 0 else 'gather'}"] = {
            "kernel_us": round(1e3 * tot.value / l.value, 2), "graph_step_us": round(1e3 * gstep, 2),
            "graph_step_warm_us": round(1e3 * warm, 2)}
print(json.dumps(out))
