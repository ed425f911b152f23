"""Summarise an ncu --set full report into JSON (profiles/): duration, DRAM
bytes, pipe utilisation, occupancy, registers, stall breakdown."""
import csv, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
res = []
for v in rows[2:]:
    d = dict(zip(h, v))
    def f(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
    stalls = {}
    for k in d:
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            x = f(k)
            if x and x > 0.05:
                stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    unit_r = d.get("dram__bytes_read.sum", "")
    res.append({
        "kernel": d.get("Kernel Name", "")[:120],
        "duration_us": f("gpu__time_duration.sum"),
        "dram_read": rd, "dram_write": wr,
        "registers": f("launch__registers_per_thread"),
        "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
        "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": f("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "ipc": f("sm__inst_executed.avg.per_cycle_active"),
        "inst_executed": f("smsp__inst_executed.sum"),
        "l2_hit_pct": f("lts__t_sector_hit_rate.pct"),
        "stalls_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])),
    })
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
