import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.md import RunConfig, run_nve
st, tn = structures.config(5); t = B.builtin_params(tn)
v = B.make_variant("B200")
done = 0
for upto in (0, 10, 20, 50, 100, 200):
    if upto > done:
        r = run_nve(st, t, RunConfig(dt=1.0, steps=upto - done, skin=0.3, rebuild_every=10, variant=v, record_every=10))
        st.positions[:] = r["positions"]; st.velocities[:] = r["velocities"]; done = upto
    rec = {"t": upto}
    for skin in (0.3, 0.4, 0.45, 0.5, 0.6):
        nl = B.build_neighbor_list(st, t.r_cut, skin)
        L = np.diff(nl.offsets)
        rec[f"f_short_{skin}"] = round(float((L <= 4).mean()), 4)
        del nl
    print(json.dumps(rec), flush=True)
