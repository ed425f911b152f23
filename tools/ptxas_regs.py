"""Registers / spills per kernel from an `nvcc -Xptxas -v` log: python tools/ptxas_regs.py LOG [name filter]"""
import re, subprocess, sys
t = open(sys.argv[1]).read()
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for m in re.finditer(r"X (\d+) registers([^\n]*)", t, re.S):
    name = m.group(1)
    try:
        name = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    except OSError:
        pass
    if flt in name:
        sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", m.group(2))
        print(name[:110], "| regs", m.group(3), "| spill", sp.groups() if sp else None)
