"""Row kernel vs warp-chunk kernel by system size (Si diamond, sigma 0.1): Tersoff
kernel time per evaluation (tb_profile events), fp64 and mixed.
Usage: python tools/row_crossover.py CELLS..."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
t = B.builtin_params("Si")
ctx = _native.default_context(0); ctx.set_table(t)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); ctx.set_stream(s.cuda_stream)
P = _native.ptr
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for cells in [int(x) for x in sys.argv[1:]]:
    st = structures.displace(structures.gen_diamond(cells), 0.1, 7)
    n = st.natoms
    pos = torch.from_numpy(st.positions).cuda(); sp = torch.zeros(n, dtype=torch.int32, device="cuda")
    f = torch.empty((n, 3), dtype=torch.float64, device="cuda"); res = torch.zeros(8, dtype=torch.float64, device="cuda")
    class D: pass
    ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
    nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
    rec = {"cells": cells, "atoms": n}
    for row in (0, 2):
        ctx.set_option(_native.OPT_ROW_KERNEL, row)
        for prec in (0, 1):
            def step():
                ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, 0, P(f), None, P(res), None))
            for _ in range(3): step()
            torch.cuda.synchronize()
            K = 20
            ctx.lib.tb_profile(ctx.handle, 1)
            for _ in range(K):
                flush.zero_(); step()
            torch.cuda.synchronize(); ctx.lib.tb_profile(ctx.handle, 0)
            tot = ctypes.c_double(); l = ctypes.c_int64()
            ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
            rec[f"{'row' if row else 'warp'}_{'fp64' if prec == 0 else 'mixed'}_us"] = round(1e3 * tot.value / K, 2)
    ctx.set_option(_native.OPT_ROW_KERNEL, 1)
    print(json.dumps(rec), flush=True)
    del pos, sp, f, nl
