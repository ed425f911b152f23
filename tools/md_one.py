"""One device-resident NVE run (tb_md_run) of a BASELINE config, for launch
lists under ncu.  Usage: python tools/md_one.py CONFIG STEPS [PREC]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.md import RunConfig, run_nve
c, steps = int(sys.argv[1]), int(sys.argv[2])
prec = sys.argv[3] if len(sys.argv) > 3 else "double"
st, tn = structures.config(c)
t = B.builtin_params(tn)
r = run_nve(st, t, RunConfig(dt=1.0, steps=steps, skin=0.3, rebuild_every=10, record_every=10,
                             variant=B.make_variant("B200", precision=prec)))
print(r["loop"], r["rebuilds"], r["wall_clock"])
