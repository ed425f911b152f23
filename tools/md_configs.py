"""Device-resident NVE (md.run_nve, tb_md_run graph loop) on BASELINE configs:
us/step and atom-steps/s, rebuild counts.  CUDA events around the run call.
Usage: MC_CONFIGS=2,3 MC_STEPS=200 python tools/md_configs.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.md import RunConfig, run_nve

out = {}
steps = int(os.environ.get("MC_STEPS", "200"))
for c in [int(x) for x in os.environ.get("MC_CONFIGS", "2,3").split(",")]:
    st, tn = structures.config(c)
    t = B.builtin_params(tn)
    dt = 1.0
    for prec in ("double", "single"):
        v = B.make_variant("B200", precision=prec)
        run_nve(st.copy(), t, RunConfig(dt=dt, steps=10, skin=0.3, rebuild_every=10, variant=v))
        r = run_nve(st.copy(), t, RunConfig(dt=dt, steps=steps, skin=0.3, rebuild_every=10,
                                            variant=v, record_every=10))
        us = r["wall_clock"]["loop"] / steps * 1e6
        key = f"c{c}_{prec}"
        out[key] = {"atoms": st.natoms, "steps": steps, "us_per_step": us,
                    "atom_steps_per_s": st.natoms * steps / r["wall_clock"]["loop"],
                    "rebuilds": r["rebuilds"], "loop": r["loop"],
                    "rel_drift": float(abs(r["total"][-1] - r["total"][0]) / abs(r["total"][0]))}
        print(json.dumps({key: out[key]}), flush=True)
json.dump(out, open(os.environ.get("MC_OUT", "gpurun_out/md_configs.json"), "w"), indent=1)
