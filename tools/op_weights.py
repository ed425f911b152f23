"""Turn the ncu metrics of tools/native/op_weights.cu into per-call flop
weights (flops = add + mul + 2 fma, minus the baseline kernel's per-call
cost) and freeze them in profiles/roofline.json.
Usage: python tools/op_weights.py gpurun_out/op_weights.csv profiles/roofline.json"""
import collections
import csv
import json
import re
import sys

THREADS, ITER = 148 * 256, 64
OPS = ["base", "div", "sqrt", "exp", "sin", "cos", "pow"]
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, im, iv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = collections.defaultdict(dict)
order = []
for r in rows[1:]:
    key = (r[h.index("ID")], r[ik])
    if key not in per:
        order.append(key)
    per[key][r[im]] = float(r[iv].replace(",", ""))
res = {"fp64": {}, "fp32": {}}
for key in order:
    m = re.search(r"k_op<(double|float), (\d)>", key[1])
    if not m:
        continue
    prec = "fp64" if m.group(1) == "double" else "fp32"
    p = "d" if prec == "fp64" else "f"
    v = per[key]
    g = lambda s: v.get(f"smsp__sass_thread_inst_executed_op_{p}{s}_pred_on.sum", 0.0)
    flops = (g("add") + g("mul") + 2 * g("fma")) / (THREADS * ITER)
    res[prec][OPS[int(m.group(2))]] = flops
out = {"method": "ncu dynamic SASS counts, flops = add + mul + 2*fma per call, "
                 "baseline loop subtracted (tools/native/op_weights.cu)",
       "weights": {}}
for prec, d in res.items():
    base = d.get("base", 0.0)
    out["weights"][prec] = {k: round(x - base, 2) for k, x in d.items() if k != "base"}
    out["weights"][prec]["add"] = 1
    out["weights"][prec]["mul"] = 1
print(json.dumps(out, indent=1))
json.dump(out, open(sys.argv[2], "w"), indent=1)
