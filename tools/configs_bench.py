"""Throughput of every BASELINE configuration on one GPU (kernel-only step:
Tersoff kernel + finalize as a CUDA-graph replay, L2 flushed between steps),
fp64 and mixed, with the algorithmic-flop roofline fraction; plus the
device-resident NVE step of config 2.  Writes one JSON object."""
import ctypes, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1710_00882_b200 as B
from paper_1710_00882_b200 import _native, structures
from paper_1710_00882_b200.md import RunConfig, run_nve
import bench

cfgs = [int(c) for c in os.environ.get("CB_CONFIGS", "1,2,3,4,5").split(",")]
steps = int(os.environ.get("CB_STEPS", "100"))
scat = int(os.environ.get("CB_SCATTER", "0"))  # 0 atomic, 1 gather
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = _native.default_context(0); ctx.set_stream(s.cuda_stream)
peak64 = bench.measure_peak(ctx.lib, ctx, 0)["tflops"]
peak32 = bench.measure_peak(ctx.lib, ctx, 1)["tflops"]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
out = {"peaks_tflops": {"fp64": peak64, "fp32": peak32}, "scatter": ["atomic", "gather"][scat], "configs": {}}
for cfg in cfgs:
    t0 = time.time()
    st, tn = structures.config(cfg)
    gen_s = time.time() - t0
    t = B.builtin_params(tn)
    ctx.set_table(t)
    n = st.natoms
    pos = torch.from_numpy(st.positions).cuda(); sp = torch.from_numpy(st.species.astype(np.int32)).cuda()
    f = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    res = torch.zeros(8, dtype=torch.float64, device="cuda"); stt = torch.zeros(6, dtype=torch.int64, device="cuda")
    class D: pass
    ds = D(); ds.positions = pos; ds.species = sp; ds.box = st.box
    torch.cuda.synchronize(); t1 = time.perf_counter()
    nl = B.build_neighbor_list(ds, t.r_cut, 0.3)
    torch.cuda.synchronize(); nl_ms = (time.perf_counter() - t1) * 1e3
    P = _native.ptr
    rec = {"atoms": n, "species": tn, "entries": nl.n_entries, "max_row": nl.max_row,
           "nl_build_ms": nl_ms, "generate_s": gen_s}
    for prec in (0, 1):
        def step(with_stats=False):
            ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(sp), float(t.r_cut), prec, scat,
                                                P(f), None, P(res), P(stt) if with_stats else None))
        step(True); torch.cuda.synchronize()
        cnt = stt.cpu().numpy()
        for _ in range(3): step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        ctx.set_stream(s.cuda_stream)
        torch.cuda.synchronize()
        K = steps if n < 4_000_000 else max(5, steps // 10)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        for a_, b_ in ev:
            flush.zero_(); a_.record(s); g.replay(); b_.record(s)
        torch.cuda.synchronize()
        step_ms = sum(a_.elapsed_time(b_) for a_, b_ in ev) / K
        ctx.lib.tb_profile(ctx.handle, 1)
        for _ in range(K):
            flush.zero_(); step()
        torch.cuda.synchronize(); ctx.lib.tb_profile(ctx.handle, 0)
        tot = ctypes.c_double(); l = ctypes.c_int64()
        ctx.lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(l))
        kms = tot.value / K  # per evaluation: the row kernel + the warp kernel when the list is split
        fl = bench.algorithmic_flops(cnt) if prec == 0 else bench.algorithmic_flops32(cnt)
        pk = peak64 if prec == 0 else peak32
        rec["fp64" if prec == 0 else "mixed"] = {
            "atom_steps_per_s": n / (step_ms * 1e-3), "step_ms": step_ms, "kernel_ms": kms,
            "kernel_launches_per_step": l.value / K,
            "achieved_tflops": fl / (kms * 1e-3) / 1e12, "frac": fl / (kms * 1e-3) / 1e12 / pk,
            "live_pairs": int(cnt[2]), "live_triplets": int(cnt[3])}
        del g
    out["configs"][cfg] = rec
    print(json.dumps({cfg: rec}), flush=True)
    del pos, sp, f, nl
    torch.cuda.empty_cache()
if 2 in cfgs and os.environ.get("CB_MD", "1") == "1":
    st, tn = structures.config(2)
    t = B.builtin_params(tn)
    for prec in ("double", "single"):
        for loop in ("graph", "step"):
            v = B.make_variant("B200", precision=prec)
            cfgr = RunConfig(dt=1.0, steps=int(os.environ.get("CB_MD_STEPS", "500")), skin=0.3, rebuild_every=10, variant=v)
            run_nve(st.copy(), t, RunConfig(dt=1.0, steps=20, skin=0.3, rebuild_every=10, variant=v), loop=loop)
            r = run_nve(st.copy(), t, cfgr, loop=loop)
            drift = float(np.max(np.abs(r["total"] - r["total"][0])) / abs(r["total"][0]))
            key = f"md_config2_{prec}_{loop}"
            out[key] = {"atom_steps_per_s": st.natoms * cfgr.steps / r["wall_clock"]["loop"],
                        "us_per_step": r["wall_clock"]["loop"] / cfgr.steps * 1e6,
                        "steps": cfgr.steps, "rebuilds": r["rebuilds"], "drift": drift,
                        "timing": "host wall clock around the step loop (synchronised), incl. graph capture for loop=graph"}
            print(json.dumps({key: out[key]}), flush=True)
json.dump(out, open(os.environ.get("CB_OUT", "gpurun_out/configs_bench.json"), "w"), indent=1)
