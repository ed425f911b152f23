"""Neighbour-list build timing (device positions, includes the host syncs of
the two-pass build)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
out = {}
for cells in [int(c) for c in os.environ.get("NB_CELLS", "20,64").split(",")]:
    st = structures.displace(structures.gen_diamond(cells, 5.431), 0.1, 1002)
    pos = torch.from_numpy(st.positions).cuda()
    ctx = _native.default_context(0)
    nl = _native.NList(ctx)
    L = np.ascontiguousarray(st.box.lengths); per = np.ones(3, np.int32)
    def build():
        ctx.check(ctx.lib.tb_build_neighbors(ctx.handle, nl.handle, st.natoms, _native.ptr(pos), _native.ptr(L), _native.ptr(per), 3.0, 0.3))
    for _ in range(3): build()
    torch.cuda.synchronize()
    K = 20
    t0 = time.perf_counter()
    for _ in range(K): build()
    torch.cuda.synchronize()
    out[st.natoms] = round((time.perf_counter() - t0) / K * 1e6, 1)
print(json.dumps({"nl_build_us": out}))
