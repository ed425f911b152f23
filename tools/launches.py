"""Print an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
for r in rows[1:]:
    print(r[iv].rjust(10), r[ik][:100])
