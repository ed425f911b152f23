"""Attribute ncu SASS-level samples/instructions to source lines.
usage: sass_lines.py <ncu sass csv> <nvdisasm -g -c output> <mangled kernel name> [top]"""
import csv, re, sys, collections
csvf, sassf, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# nvdisasm: offset -> file:line
lines = open(sassf).read().split("\n")
start = None
for k, l in enumerate(lines):
    if l.startswith(f".text.{fn}:"):
        start = k
        break
assert start is not None, "function not found"
cur = "?"
off2line = {}
for l in lines[start + 1:]:
    if l.startswith("//---") or l.startswith(".text.") and not l.startswith(f".text.{fn}"):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
h = rows[1]
ix = {x: i for i, x in enumerate(h)}
base = None
agg = collections.defaultdict(lambda: [0, 0])
tot_s = tot_i = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    a = int(r[ix["Address"]], 16)
    if base is None:
        base = a
    ln = off2line.get(a - base, "?")
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    agg[ln][0] += s
    agg[ln][1] += n
    tot_s += s
    tot_i += n
print(f"samples {tot_s} instr {tot_i}")
for ln, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}% samp {100*n/tot_i:5.1f}% inst  {ln}")
