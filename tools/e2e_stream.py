"""End-to-end compute() with pinned host buffers: streamed (TB_OPT_STREAM_RANGE)
vs plain, wall clock per call, plus copy-only floors (H2D alone, D2H alone,
both directions at once).  Usage: python tools/e2e_stream.py [config] [ranges...]"""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
ranges = [int(a) for a in sys.argv[2:]] or [0, 131072]
prec = os.environ.get("PREC", "double")
st, tn = structures.config(cfg)
t = B.builtin_params(tn)
n = st.natoms
nl = B.build_neighbor_list(st, t.r_cut, 0.3, device=0)
ctx = nl.context
pin = lambda shape, dt: torch.empty(shape, dtype=dt).pin_memory()
pos_t = pin((n, 3), torch.float64)
pos_t.numpy()[:] = st.positions
sp_d = torch.from_numpy(st.species.astype(np.int32)).cuda()
f_t, e_t = pin((n, 3), torch.float64), pin(n, torch.float64)


class HS:
    pass


hs = HS(); hs.positions, hs.species, hs.box = pos_t.numpy(), sp_d, st.box
var = B.make_variant("B200", precision=prec)
out = B.ForceEnergyResult(f_t.numpy(), 0.0, e_t.numpy(), {})
res = {"config": cfg, "atoms": n, "precision": prec}
ref = None
for r in ranges:
    ctx.set_option(_native.OPT_STREAM_RANGE, r)
    for _ in range(2):
        B.compute(hs, nl, t, var, out=out)
    k = 5
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(k):
            rr = B.compute(hs, nl, t, var, out=out)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / k)
    f = out.forces.copy()
    if ref is None:
        ref = (f, rr.potential_energy, out.per_atom_energy.copy())
    res[f"range_{r}"] = {"ms_per_call": round(1e3 * best, 3), "atom_steps_per_s": n / best,
                         "energy": rr.potential_energy,
                         "max_dF_vs_first": float(np.abs(f - ref[0]).max()),
                         "per_atom_equal": bool(np.array_equal(out.per_atom_energy, ref[2]))}

# copy floors
dpos = torch.empty((n, 3), dtype=torch.float64, device="cuda")
df = torch.empty((n, 3), dtype=torch.float64, device="cuda")
de = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def tm(fn, k=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return round(1e3 * (time.perf_counter() - t0) / k, 3)


def h2d():
    with torch.cuda.stream(s1):
        dpos.copy_(pos_t, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        f_t.copy_(df, non_blocking=True); e_t.copy_(de, non_blocking=True)


res["h2d_only_ms"] = tm(h2d)
res["d2h_only_ms"] = tm(d2h)
res["both_directions_ms"] = tm(lambda: (h2d(), d2h()))
print(json.dumps(res))
