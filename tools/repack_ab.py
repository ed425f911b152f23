"""A/B timing of one evaluation (live repack + Tersoff + finalize) for the
library named by TB_LIB_PATH.  Usage: python tools/repack_ab.py CONFIG [reps]
Prints ms per evaluation (CUDA events, eager, no L2 flush) and the energy."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
cfg = int(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
st, tn = structures.config(cfg)
t = B.builtin_params(tn); n = st.natoms
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = _native.default_context(0); ctx.set_table(t); ctx.set_stream(s.cuda_stream)
pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); pa = torch.empty(n, dtype=torch.float64, device="cuda")
res = torch.zeros(8, dtype=torch.float64, device="cuda")
class D: pass
ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
P = _native.ptr
def one(prec):
    ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut),
                                        prec, 0, P(f), P(pa), P(res), None))
for prec in (0, 1):
    for _ in range(5): one(prec)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(reps): one(prec)
    e1.record(s); torch.cuda.synchronize()
    print(f"lib={os.path.basename(os.environ.get('TB_LIB_PATH', 'default'))} cfg={cfg} prec={prec} "
          f"ms={e0.elapsed_time(e1) / reps:.4f} E={res[0].item():.10f} "
          f"Fsum={f.abs().sum().item():.10f} pa={pa.sum().item():.10f}")
