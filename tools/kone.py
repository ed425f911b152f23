"""Run one Tersoff evaluation configuration a few times (for ncu captures).
Usage: python tools/kone.py CONFIG PREC(0=fp64,1=mixed) SCAT(0=atomic,1=gather) [reps]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
cfg, prec, scat = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
st, tn = structures.config(cfg, small=os.environ.get("KB_SMALL") == "1")
t = B.builtin_params(tn)
n = st.natoms
ctx = _native.default_context(0); ctx.set_table(t)
if os.environ.get("KB_LIVE"):
    ctx.set_option(_native.OPT_LIVE_PACK, int(os.environ["KB_LIVE"]))
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
for _ in range(reps):
    ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut),
                                        prec, scat, P(f), P(pa), P(res), None))
torch.cuda.synchronize()
print("E", res[0].item())
