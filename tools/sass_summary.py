"""Summarise an ncu --page source --print-source sass CSV: executed warp
instructions and stall samples per opcode, plus the hottest instructions."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); st = collections.Counter(); tot = 0; tots = 0
hot = []
for r in rows[2:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    base = op.split(".")[0]
    n = int(r[ix["Instructions Executed"]] or 0); s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ops[base] += n; st[base] += s; tot += n; tots += s
    hot.append((s, n, r[ix["Address"]], src))
print(f"total warp instr {tot}, stall samples {tots}")
for op, n in ops.most_common(30):
    print(f"{op:12s} {n:10d} {100*n/tot:5.1f}%   stalls {100*st[op]/max(tots,1):5.1f}%")
print("--- hottest by stall samples")
for s, n, a, src in sorted(hot, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{s:6d} {n:8d} {a} {src}")
