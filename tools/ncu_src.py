"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export by
CUDA source line: executed warp instructions and stall samples.
Usage: python tools/ncu_src.py file.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None; hdr = None
lines = collections.defaultdict(lambda: [0.0, 0.0, "", collections.Counter()])
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r; iE = hdr.index("Instructions Executed"); iW = hdr.index("Warp Stall Sampling (All Samples)"); continue
    if hdr is None:
        continue
    # cuda line rows have a line number in col 0; sass rows have empty col 0 and address in col 2
    if r[0].strip():
        cur_line = (fname, int(r[0]))
        lines[cur_line][2] = r[1][:70]
        continue
    try:
        n = float(r[iE] or 0); s = float(r[iW] or 0)
    except ValueError:
        continue
    L = lines[cur_line]; L[0] += n; L[1] += s
    op = r[3].split()[0] if r[3] else "";
    if op.startswith("@"): op = r[3].split()[1]
    L[3][op.split(".")[0]] += n
tn = sum(v[0] for v in lines.values()); ts = sum(v[1] for v in lines.values())
print(f"total warp inst {tn:.0f} samples {ts:.0f}")
byf = collections.Counter()
for k, v in lines.items(): byf[k[0]] += v[0]
print({k: round(100 * v / tn, 1) for k, v in byf.most_common()})
for k, v in sorted(lines.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{k[0]:>22}:{k[1]:<4} inst {100*v[0]/tn:5.1f}% stall {100*v[1]/ts:5.1f}%  {v[2]!s:70} {dict(v[3].most_common(4))}")
