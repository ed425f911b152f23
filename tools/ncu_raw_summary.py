"""Key metrics of one `ncu --page raw --csv` export: python tools/ncu_raw_summary.py FILE.csv [more.csv ...]"""
import csv, sys
KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum"]
for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, unit, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(val, unit)))
    print("==", f, d.get("Kernel Name", ("", ""))[0][:80])
    for k in KEYS:
        if k in d:
            print(f"  {k:75s} {d[k][0]:>18s} {d[k][1]}")
    stalls = [(float(v[0].replace(",", "")), k) for k, v in d.items()
              if k.startswith("smsp__average_warp") and "issue_stalled" in k and k.endswith("_per_warp_active.pct") is False
              and "per_issue_active" in k and "not_issued" not in k]
    for v, k in sorted(stalls, reverse=True)[:8]:
        print(f"  stall {k.split('issue_stalled_')[1].split('_per')[0]:30s} {v:8.3f}")
