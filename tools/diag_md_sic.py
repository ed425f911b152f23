"""Graph loop vs step loop on small SiC: rebuild counts and energy divergence."""
import numpy as np
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.paramfile import builtin_params
from paper_1710_00882_b200.system import RunConfig, run_nve_device

st, tname = structures.config(3, small=True)
t = builtin_params(tname)
cfg = RunConfig(dt=0.5, steps=200, skin=0.3, rebuild_every=10)
runs = {}
for loop in ("graph", "step", "graph", "step"):
    for sc in ("atomic", "gather"):
        r = run_nve_device(st.copy(), t, cfg, loop=loop, scatter=sc, record_every=1)
        runs.setdefault((loop, sc), []).append(r)
        print(loop, sc, "rebuilds", r["rebuilds"], "E_end", repr(r["total"][-1]))
a = runs[("graph", "gather")][0]["total"]
b = runs[("step", "gather")][0]["total"]
d = np.abs(a - b) / abs(b[0])
print("gather graph vs step: first step with diff > 1e-12:", int(np.argmax(d > 1e-12)), "max", d.max())
print("gather graph vs graph:", np.abs(a - runs[("graph", "gather")][1]["total"]).max())
print("gather step vs step:", np.abs(b - runs[("step", "gather")][1]["total"]).max())
