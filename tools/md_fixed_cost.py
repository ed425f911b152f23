"""Fixed cost of a tb_md_run call at a config: the same call at several step
counts, CUDA events around each (bench.py's md protocol).
Usage: python tools/md_fixed_cost.py CONFIG STEPS..."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
c = int(sys.argv[1])
st, tn = structures.config(c)
t = B.builtin_params(tn)
ctx = _native.default_context(0)
for k in [int(x) for x in sys.argv[2:]]:
    t0 = time.perf_counter()
    r = bench.md_measure(B, _native, ctx, st, t, 0, 0, k, warm=int(os.environ.get("WARM", "20")))
    print(json.dumps({"steps": k, "ms_per_step": r["ms_per_step"], "total_ms": r["ms_per_step"] * k,
                      "rebuilds": r["rebuilds"], "wall_s": time.perf_counter() - t0}), flush=True)
