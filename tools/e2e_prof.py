"""Break down the end-to-end compute() call (config 2): full API call, raw C-ABI
call, copies alone, device-only call.  Usage: python tools/e2e_prof.py [config]"""
import ctypes, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
st, tn = structures.config(cfg)
t = B.builtin_params(tn)
n = st.natoms
nl = B.build_neighbor_list(st, t.r_cut, 0.3, device=0)
ctx = nl.context
P = _native.ptr
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()
pos_t, sp_t = pin((n, 3), torch.float64), pin(n, torch.int32)
pos_t.numpy()[:] = st.positions
sp_t.numpy()[:] = st.species
f_t, e_t = pin((n, 3), torch.float64), pin(n, torch.float64)


class HS:
    pass


hs = HS(); hs.positions, hs.species, hs.box = pos_t.numpy(), sp_t.numpy(), st.box
var = B.make_variant("B200")
out = B.ForceEnergyResult(f_t.numpy(), 0.0, e_t.numpy(), {})
res = {}


def timeit(name, fn, k=300, rep=5):
    for _ in range(10):
        fn()
    best = 1e9
    for _ in range(rep):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / k)
    res[name] = round(1e6 * best, 1)


timeit("api_compute_us", lambda: B.compute(hs, nl, t, var, out=out))
energy = np.zeros(1); vir = np.zeros(6); stats = np.zeros(_native.NSTATS, np.int64)
args = (ctx.handle, nl._nl.handle, P(hs.positions), P(hs.species), float(t.r_cut), 0, 0,
        P(out.forces), P(out.per_atom_energy), P(energy), P(vir), P(stats))
timeit("raw_tb_compute_us", lambda: ctx.lib.tb_compute(*args))
timeit("raw_tb_compute_no_peratom_us",
       lambda: ctx.lib.tb_compute(*args[:8], None, *args[9:]))
dpos, dsp = pos_t.cuda(), sp_t.cuda()
df, de = torch.empty((n, 3), dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()


def copies():
    dpos.copy_(pos_t, non_blocking=True); dsp.copy_(sp_t, non_blocking=True)
    f_t.copy_(df, non_blocking=True); e_t.copy_(de, non_blocking=True)
    s.synchronize()


timeit("copies_only_us", copies)
ctx.set_stream(s.cuda_stream)
r8 = torch.zeros(8, dtype=torch.float64, device="cuda")
dargs = (ctx.handle, nl._nl.handle, P(dpos), P(dsp), float(t.r_cut), 0, 0, P(df), P(de), P(r8), None)


def dev():
    ctx.lib.tb_compute_device(*dargs)
    s.synchronize()


timeit("device_call_sync_us", dev)
timeit("raw_tb_compute_on_device_ptrs_us",
       lambda: ctx.lib.tb_compute(ctx.handle, nl._nl.handle, P(dpos), P(dsp), float(t.r_cut), 0, 0,
                                  P(df), P(de), P(energy), P(vir), P(stats)))
res["atoms"] = n
print(json.dumps(res))
