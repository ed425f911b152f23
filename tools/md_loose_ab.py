"""NVE config N with different loose-list skins (TB_OPT_MD_LOOSE_SKIN): ms/step.
Usage: python tools/md_loose_ab.py CONFIG STEPS 30 0 15 ..."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.md import RunConfig, run_nve
c, steps = int(sys.argv[1]), int(sys.argv[2])
st, tn = structures.config(c)
t = B.builtin_params(tn)
ctx = _native.default_context(0)
v = B.make_variant("B200")
for loose in [int(x) for x in sys.argv[3:]]:
    ctx.set_option(_native.OPT_MD_LOOSE_SKIN, loose)
    run_nve(st.copy(), t, RunConfig(dt=1.0, steps=10, skin=0.3, rebuild_every=10, variant=v))
    for n in (steps, 2 * steps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = run_nve(st.copy(), t, RunConfig(dt=1.0, steps=n, skin=0.3, rebuild_every=10, variant=v, record_every=10))
        torch.cuda.synchronize(); el = time.perf_counter() - t0
        print(json.dumps({"loose": loose, "steps": n, "loop_ms_per_step": r["wall_clock"]["loop"] / n * 1e3,
                          "call_ms_total": el * 1e3, "rebuilds": r["rebuilds"], "wall": r["wall_clock"]}), flush=True)
