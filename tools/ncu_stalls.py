"""Print warp-stall breakdown (per issued instruction) from an ncu report."""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, v = rows[0], rows[-1]
d = dict(zip(h, v))
st = {}
for k, x in d.items():
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(x.replace(",", ""))
        except ValueError:
            pass
for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:12]:
    print(f"{x:8.3f}  {k}")
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "gpu__time_duration.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]:
    if k in d:
        print(k, d[k])
