"""Summarise `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv` launch lists: per kernel name, mean duration (us)
and DRAM bytes per launch.  Usage: python tools/ncu_launch_table.py FILE..."""
import csv
import io
import json
import re
import sys
from collections import defaultdict


def parse(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    agg = defaultdict(lambda: defaultdict(list))
    for r in rows:
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        name = re.sub(r"<.*", "", name) if "cub" in name else name
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        unit = r["Metric Unit"]
        m = r["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}[unit]
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        agg[name][m].append(v)
    out = {}
    for name, ms in agg.items():
        d = ms.get("gpu__time_duration.sum", [])
        rd = ms.get("dram__bytes_read.sum", [0])
        wr = ms.get("dram__bytes_write.sum", [0])
        out[name] = {"launches": len(d), "us_mean": sum(d) / max(len(d), 1),
                     "dram_bytes_mean": (sum(rd) + sum(wr)) / max(len(d), 1)}
    return out


if __name__ == "__main__":
    res = {p: parse(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
