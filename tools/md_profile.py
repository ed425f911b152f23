"""One device-resident NVE run of BASELINE config 2 (64k Si) for launch lists."""
import os
import sys

from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.paramfile import builtin_params
from paper_1710_00882_b200.system import RunConfig, run_nve_device

steps = int(os.environ.get("MP_STEPS", "100"))
loop = os.environ.get("MP_LOOP", "graph")
prec = os.environ.get("MP_PREC", "double")
st, tn = structures.config(2)
t = builtin_params(tn)
r = run_nve_device(st.copy(), t, RunConfig(dt=1.0, steps=steps, skin=0.3, rebuild_every=10),
                   precision=prec, loop=loop)
print(loop, prec, "steps", steps, "rebuilds", r["rebuilds"], "loop_s", r["wall_clock"]["loop"],
      file=sys.stderr)
