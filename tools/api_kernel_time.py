import ctypes, json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
st, tn = structures.config(5); t = B.builtin_params(tn)
ctx = _native.default_context(0); ctx.set_table(t)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
P = _native.ptr; n = st.natoms
pos = torch.from_numpy(st.positions).cuda(); sp = torch.zeros(n, dtype=torch.int32, device="cuda")
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); res = torch.zeros(8, dtype=torch.float64, device="cuda")
stt = torch.zeros(8, dtype=torch.int64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
out = {}
for prec in (0, 1):
    for stats in (False, True):
        def step():
            ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, 0, P(f), None, P(res), P(stt) if stats else None))
        for _ in range(3): step()
        torch.cuda.synchronize(); K = 15
        ctx.lib.tb_profile(ctx.handle, 1)
        for _ in range(K): step()
        torch.cuda.synchronize(); ctx.lib.tb_profile(ctx.handle, 0)
        tot = ctypes.c_double(); l = ctypes.c_int64()
        ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
        out[f"p{prec}_stats{int(stats)}_us"] = round(1e3 * tot.value / K, 1)
print(json.dumps(out), stt.cpu().numpy().tolist())
