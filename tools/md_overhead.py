"""Fixed cost of one tb_md_run call (config 2): event-timed runs of 10 and 1000
steps after a warm-up run, with the loose list on (default) and off."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.system import ACCEL

st, tn = structures.config(2)
t = B.builtin_params(tn)
n = st.natoms
d = torch.device("cuda", 0)
s = torch.cuda.current_stream(d)
ctx = _native.default_context(0)
ctx.set_stream(s.cuda_stream)
ctx.set_table(t)
out = {}
for loose in (30, 0):
    ctx.set_option(_native.OPT_MD_LOOSE_SKIN, loose)
    pos = torch.from_numpy(st.positions.copy()).to(d)
    vel = torch.from_numpy(st.velocities.copy()).to(d)
    mass = torch.from_numpy(np.ascontiguousarray(st.atom_masses, dtype=np.float64)).to(d)
    sp = torch.from_numpy(st.species.astype(np.int32)).to(d)
    f = torch.empty((n, 3), dtype=torch.float64, device=d)
    res = torch.zeros(8, dtype=torch.float64, device=d)
    ser = torch.zeros((200, 2), dtype=torch.float64, device=d)

    class DS:
        pass
    ds = DS(); ds.positions, ds.species, ds.box = pos, sp, st.box
    nl = B.build_neighbor_list(ds, t.r_cut, 0.3, device=0)
    P = _native.ptr
    ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut),
                                        0, 0, P(f), None, P(res), None))
    nreb = ctypes.c_int64()

    def run(k):
        ctx.check(ctx.lib.tb_md_run(ctx.handle, nl._nl.handle, n, P(pos), P(vel), P(f), P(mass),
                                    P(sp), 1.0, float(ACCEL), float(t.r_cut), 0.3, 10, 0, 0, k,
                                    100, P(ser), P(res), ctypes.byref(nreb)))

    run(20)
    for k in (10, 1000, 10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(s); run(k); b.record(s)
        torch.cuda.synchronize()
        out[f"loose{loose}_steps{k}_ms"] = round(a.elapsed_time(b), 3)
ctx.set_option(_native.OPT_MD_LOOSE_SKIN, 30)
print(json.dumps(out))
