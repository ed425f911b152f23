import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.md import RunConfig, run_nve
st, tn = structures.config(2)
t = B.builtin_params(tn)
for k in range(4):
    for steps in (10, 200, 1000):
        r = run_nve(st.copy(), t, RunConfig(dt=1.0, steps=steps, skin=0.3, rebuild_every=10, record_every=10))
        print(k, steps, round(r["wall_clock"]["loop"] / steps * 1e6, 1), "us/step", r["rebuilds"], flush=True)
