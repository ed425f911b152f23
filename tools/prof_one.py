"""Run a few device-resident evaluations of one configuration (for ncu).
Usage: python tools/prof_one.py [double|single] [atomic|gather] [config] [warp|tile]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
prec = sys.argv[1] if len(sys.argv) > 1 else "double"
scat = sys.argv[2] if len(sys.argv) > 2 else "atomic"
cfg = int(sys.argv[3]) if len(sys.argv) > 3 else 2
path = sys.argv[4] if len(sys.argv) > 4 else "warp"
st, tn = structures.config(cfg)
t = B.builtin_params(tn)
n = st.natoms
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = _native.default_context(0); ctx.set_stream(s.cuda_stream); ctx.set_table(t)
ctx.set_option(_native.OPT_TILE_KERNEL, path == "tile")
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda"); stt = torch.zeros(6, dtype=torch.int64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
for _ in range(6):
    ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut),
                                        _native.PRECISION[prec], _native.SCATTER[scat], P(f), P(pa), P(res), P(stt)))
torch.cuda.synchronize()
ctx.check(ctx.lib.tb_check_errors(ctx.handle))
print("ok", float(res[0]))
