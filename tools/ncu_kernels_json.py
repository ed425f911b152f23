"""Summarise the ncu raw exports of tools/ncu_kernels.sh into profiles/ JSON:
duration, DRAM bytes and GB/s against the measured HBM peak, pipe / issue /
L1 utilisation, lane efficiency.  Usage: python tools/ncu_kernels_json.py OUT.json [INDIR]"""
import csv, glob, json, sys
TS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"method": "ncu --set full --clock-control none, one k_tersoff_warp launch after two "
                 "warm-up evaluations (tools/ncu_kernels.sh, tools/kone.py CONFIG PREC 0); "
                 "cold caches (ncu default cache control)",
       "peaks": {"dram_GBs_measured": 6552.3, "source": "MEASURED_PEAKS.json hbm_gbs"},
       "kernels": {}}
indir = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
for f in sorted(glob.glob(f"{indir}/ncu_tk_c*_p*_raw.csv")):
    rows = list(csv.reader(open(f)))
    u = dict(zip(rows[0], rows[1]))
    # the dominant kernel of the evaluation (row kernel, or the warp kernel alone)
    cands = [dict(zip(rows[0], r)) for r in rows[2:] if len(r) == len(rows[0])]
    d = max(cands, key=lambda c: float(c["gpu__time_duration.sum"].replace(",", "")) *
            TS[u["gpu__time_duration.sum"]])
    others = [c for c in cands if c is not d]

    def g(k):
        try:
            return float(d[k].replace(",", ""))
        except (KeyError, ValueError):
            return None
    tag = f.split("ncu_tk_")[1].replace("_raw.csv", "")
    dur = g("gpu__time_duration.sum") * TS[u["gpu__time_duration.sum"]]
    byts = sum((g(k) or 0.0) * BS[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    out["kernels"][tag] = {
        "kernel": d.get("Kernel Name", "")[:90],
        "duration_us": round(dur, 2), "dram_bytes": byts,
        "dram_GBs": round(byts / dur / 1e3, 1),
        "dram_frac_of_measured": round(byts / dur / 1e3 / 6552.3, 4),
        "fp64_pipe_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct": g("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "l1tex_pct": g("l1tex__throughput.avg.pct_of_peak_sustained_active"),
        "sm_active_of_elapsed_pct": round(100 * g("sm__cycles_active.avg") / g("sm__cycles_elapsed.avg"), 1),
        "threads_per_inst": g("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "registers": g("launch__registers_per_thread"),
        "occupancy_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "other_kernels_us": [round(float(c["gpu__time_duration.sum"].replace(",", "")) *
                                   TS[u["gpu__time_duration.sum"]], 2) for c in others],
    }
    # executed fp64 / fp32 flops of the dominant kernel from the SASS-level export
    # (thread-level DFMA x2 + DMUL + DADD, resp. FFMA x2 + FMUL + FADD)
    try:
        srows = list(csv.reader(open(f.replace("_raw.csv", "_sass.csv"))))
    except OSError:
        srows = []
    hdr, ops, kname, best = None, {}, None, {}
    for r in srows:
        if r and r[0] in ("Function Name", "Kernel Name"):
            kname = r[1]
            # (a multi-kernel report prints every kernel's block twice: keep the first)
            ops = {} if kname in best else best.setdefault(kname, {})
        if r and r[0] in ("Line No", "Address", "#"):
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or "Thread Instructions Executed" not in hdr:
            continue
        src = r[hdr.index("Source")] if "Source" in hdr else ""
        tok = src.split()
        if not tok:
            continue
        op = (tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]).split(".")[0]
        try:
            ops[op] = ops.get(op, 0.0) + float(r[hdr.index("Thread Instructions Executed")] or 0)
        except ValueError:
            pass
    if best:
        o = max(best.values(), key=lambda v: sum(v.values()))
        pre = "D" if tag.endswith("p0") else "F"
        out["kernels"][tag]["executed_flops"] = 2 * o.get(pre + "FMA", 0) + o.get(pre + "MUL", 0) + o.get(pre + "ADD", 0)
        out["kernels"][tag]["thread_inst_executed"] = sum(o.values())
json.dump(out, open(sys.argv[1], "w"), indent=1)
for k, v in out["kernels"].items():
    print(k, {a: v[a] for a in ("duration_us", "dram_GBs", "fp64_pipe_pct", "fma_pipe_pct",
                                "issue_active_pct", "l1tex_pct", "sm_active_of_elapsed_pct")})
