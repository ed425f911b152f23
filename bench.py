#!/usr/bin/env python
"""Benchmark of the B200 Tersoff hot path (driver contract: one JSON line).

Metric (BASELINE.json): Tersoff atom-steps/s -- atoms x E+F evaluations per
second -- with the achieved fraction of the FP64 pipe peak.

Workload: BASELINE config 2, the largest single-GPU configuration the metric
is quoted on: 64,000-atom Si diamond (20^3 cells, a=5.431, sigma=0.1 seed
1002), Si(C) Tersoff parameters, skin 0.3, fp64.  One "step" = one energy +
force + virial evaluation at the current positions: the kernel re-packs the
skin list at r_cut (pack_adjacency) and evaluates every Tersoff term
(kernels.compute semantics).  The neighbour list is built once outside the
timed region, as the reference harness does (bench.py:116-118).  Inputs are
resident in HBM for `value`; the 64k-atom working set (~6 MB) fits in L2, so
L2 is flushed (a 256 MiB write) between timed steps.

  e2e         the same evaluation through the public API compute() with the
              positions in pinned host memory: H2D of positions+species and
              D2H of forces, per-atom energies, energy/virial/stats per step.
  roofline    the Tersoff kernel's algorithmic fp64 flops (SURVEY 8(d) op
              counts per live pair / live triplet) / its CUDA-event time, against
              the FP64 DFMA peak measured on this GPU at start-up.
  cpu_baseline  the CPU oracle (a C restatement of the reference ScalarOpt,
              oracle/) on this host's cores, rank 0, N=1.

  --impl reference   the reference's CPU implementation of the path on the
              host cores (the oracle port; the Python reference cannot travel).

Multi-GPU (torchrun, N>1): every rank evaluates its own replica of the
workload (weak scaling); time = max over ranks of the device-timed loop.
"""

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Tersoff atom-steps/s (E+F evals)"
UNIT = "atom-steps/s"

# the reference ScalarOpt expression tree charged once per
# live pair / triplet, math-library calls weighted by their dynamic flop counts
# on sm_100a (ncu, tools/native/op_weights.cu -> profiles/roofline.json);
# the static SASS counts of SURVEY 8(d) are the fallback.
_W_STATIC = {"fp64": {"div": 15, "sqrt": 13, "exp": 31, "sin": 26, "cos": 26, "pow": 125},
             "fp32": {"div": 10, "sqrt": 5, "exp": 10, "sin": 20, "cos": 20, "pow": 63}}


def _op_weights():
    try:
        with open(os.path.join(ROOT, "profiles", "roofline.json")) as fh:
            w = json.load(fh)["weights"]
        return {p: {k: float(w[p][k]) for k in _W_STATIC[p]} for p in _W_STATIC}, "ncu-dynamic"
    except (OSError, KeyError, ValueError):
        return _W_STATIC, "static-sass"


OP_WEIGHTS, OP_WEIGHTS_SOURCE = _op_weights()


def _costs(w, distance):
    pair = 19 + 25 + 3 * w["div"] + 2 * w["exp"] + 4 * w["pow"] + (8 + w["sqrt"] if distance else 0)
    trip = 32 + 55 + 4 * w["div"] + w["exp"]
    taper = 2 + 3 + w["div"] + w["sin"] + w["cos"]  # per tapered f_C
    return pair, trip, taper


def _jsonable(o):
    return o.item() if hasattr(o, "item") else str(o)


FLOPS_PAIR, FLOPS_TRIP, FLOPS_TAPER = _costs(OP_WEIGHTS["fp64"], True)
# mixed mode: the distance stays fp64 and is not charged to the fp32 pipe
FLOPS32_PAIR, FLOPS32_TRIP, FLOPS32_TAPER = _costs(OP_WEIGHTS["fp32"], False)


def algorithmic_flops32(stats):
    return int(FLOPS32_PAIR * stats[2] + FLOPS32_TAPER * stats[4]
               + FLOPS32_TRIP * stats[3] + FLOPS32_TAPER * stats[5])


def algorithmic_flops(stats):
    return int(FLOPS_PAIR * stats[2] + FLOPS_TAPER * stats[4]
            + FLOPS_TRIP * stats[3] + FLOPS_TAPER * stats[5])


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
            0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, torch_dev):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                uuid = str(torch.cuda.get_device_properties(torch_dev).uuid)
                if not uuid.startswith("GPU-"):
                    uuid = "GPU-" + uuid
                h = pynvml.nvmlDeviceGetHandleByUUID(uuid)
            except Exception:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                idx = int(vis.split(",")[torch_dev]) if vis and vis.split(",")[0].isdigit() \
                    else torch_dev
                h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nv, self.h = pynvml, h
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def _run(self):
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.BITS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_baseline(state, table, budget_s=12.0, min_evals=2, threads=None):
    """Time the CPU oracle (reference ScalarOpt restated in C, OpenMP over
    atom ranges) on this host: NL built outside the timer, then E+F
    evaluations (pack + kernel) until `budget_s`."""
    from oracle import oracle as O
    threads = threads or cpu_cores()
    off, nb = O.build_neighbor_list(state.positions, state.box.lengths, state.box.periodic,
                                    table.r_cut, 0.3, threads=threads)
    t0 = time.perf_counter()
    evals = 0
    while True:
        O.compute(state.positions, state.species, state.box.lengths, state.box.periodic,
                  off, nb, table, threads=threads)
        evals += 1
        el = time.perf_counter() - t0
        if (el >= budget_s and evals >= min_evals) or evals >= 10000:
            break
    return state.natoms * evals / el, threads, evals, el


def reference_arm(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1710_00882_b200 import structures
    from paper_1710_00882_b200.paramfile import builtin_params
    from oracle import oracle as O
    state, tname = structures.config(args.config)
    table = builtin_params(tname)
    threads = cpu_cores()
    off, nb = O.build_neighbor_list(state.positions, state.box.lengths, state.box.periodic,
                                    table.r_cut, 0.3, threads=threads)

    def one():
        O.compute(state.positions, state.species, state.box.lengths, state.box.periodic,
                  off, nb, table, precision=args.precision_ref, threads=threads)

    for _ in range(args.warmup):
        one()
    # bounded sample: the whole run stays within ~2 minutes
    t0 = time.perf_counter()
    one()
    per = time.perf_counter() - t0
    steps = args.steps
    budget = 120.0
    timed = max(1, min(steps, int(budget / max(per, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(timed):
        one()
    el = time.perf_counter() - t0
    value = state.natoms * timed / el
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": timed, "warmup": args.warmup, "ms_per_step": 1e3 * el / timed,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if args.precision_ref == "double" else "f32/f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"BASELINE config {args.config}: {state.natoms} Si diamond "
                               f"E+F(+virial) evaluation, skin 0.3",
                   "atoms": state.natoms, "precision": args.precision_ref},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{timed} full E+F evaluations of the {state.natoms}-atom "
                                   f"system (of {steps} requested; bounded to ~{budget:.0f} s), "
                                   f"NL built outside the timer; oracle/ C restatement of "
                                   f"ScalarOpt, OpenMP over {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line, default=_jsonable), flush=True)


def gpu_arm_decomposed(args):
    """N > 1: slab decomposition (decomp.py) with NCCL P2P halos, weak scaling:
    every GPU owns a 20^3-cell (64,000-atom) slab of a (20N x 20 x 20)-cell Si
    crystal (config 2 per GPU, same seeds).  A step = forward halo + Tersoff
    evaluation on [owned | ghosts] + reverse ghost forces + all-reduce of
    [E, W6]; device-timed (CUDA events) per rank, max over ranks."""
    import ctypes
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_setup()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1710_00882_b200 import _native, decomp, structures
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: single-GPU smoke test only
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
        decomp.set_comm_device("cpu")
    from paper_1710_00882_b200.paramfile import builtin_params
    cells = (20 * ws, 20, 20)
    st = structures.displace(structures.gen_diamond(cells, 5.431), 0.1, 1002)
    table = builtin_params("Si")
    n_total = st.natoms
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    d = decomp.SlabDecomposition(st.box.lengths, st.box.periodic, table.r_cut + 0.3, ws)
    dom = decomp.scatter_state(d, st, rank, dev)
    eng = decomp.B200Engine(table, 0.3, device=local, precision=args.precision,
                            scatter=args.scatter)
    ff = decomp.DecomposedForceField(d, st.box, eng, rank, ws, dev)
    dom = ff.rebuild(dom)
    for _ in range(max(3, args.warmup)):
        f, res = ff(dom)
    torch.cuda.synchronize()
    # the whole decomposed step (halo P2P, Tersoff kernel + finalize, reverse
    # forces, all-reduce) as one CUDA graph: NCCL ops are capturable
    # (tools/nccl_capture_probe.py); any capture error falls back to eager
    launch = f"eager (Python host loop, {backend} batch_isend_irecv)"
    graph = None
    step_fn = lambda: ff(dom)  # noqa: E731
    if backend == "nccl" and os.environ.get("BENCH_DD_GRAPH", "1") == "1":
        try:
            dist.barrier()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                f_g, res_g = ff(dom)
            graph.replay()
            torch.cuda.synchronize()
            step_fn = lambda: (graph.replay(), (f_g, res_g))[1]  # noqa: E731
            launch = ("one CUDA graph per step: halo P2P + Tersoff kernel + finalize + reverse "
                      "forces + all-reduce (NCCL ops captured)")
        except Exception as e:  # noqa: BLE001
            graph = None
            launch = f"eager (graph capture failed: {str(e)[:80]})"
            torch.cuda.synchronize()
        # every rank must take the same path (their NCCL call sequences must match)
        ok = torch.tensor([1 if graph is not None else 0], dtype=torch.int32,
                          device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and graph is not None:
            del graph
            graph = None
            step_fn = lambda: ff(dom)  # noqa: E731
            launch = "eager (graph capture failed on another rank)"
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    k = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    sampler = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for s_ in range(k):
            flush.zero_()
            starts[s_].record(stream)
            f, res = step_fn()
            ends[s_].record(stream)
        torch.cuda.synchronize()
    t_local = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / 1e3
    comm = "cpu" if backend != "nccl" else dev
    t = torch.tensor([t_local], dtype=torch.float64, device=comm)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t[0])
    value = n_total * k / t_max
    energy = float(res[0])
    # kernel share on this rank
    lib, ctx = eng.ctx.lib, eng.ctx
    lib.tb_profile(ctx.handle, 1)
    for _ in range(min(k, 100)):
        flush.zero_()
        f, res = ff(dom)
    torch.cuda.synchronize()
    lib.tb_profile(ctx.handle, 0)
    tot, cnt = ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(cnt)))
    kern_ms = tot.value / max(cnt.value, 1)
    # rank 0's algorithmic flops (its owned rows) for the kernel roofline
    roof = {"bound": "fp64" if args.precision == "double" else "fp32",
            "kernel_ms_rank0": kern_ms, "achieved": None, "peak": None,
            "unit": "TFLOP/s", "frac": None, "traffic": None}
    if rank == 0:
        pcode = _native.PRECISION[args.precision]
        st_t = torch.zeros(_native.NSTATS, dtype=torch.int64, device=dev)
        r8 = torch.zeros(8, dtype=torch.float64, device=dev)
        pos_l = dom._pos_l  # [owned | ghosts] of the last step (no collective on one rank)
        f_t = torch.empty((pos_l.shape[0], 3), dtype=torch.float64, device=dev)
        rc = lib.tb_compute_device(ctx.handle, eng.nl.handle, _native.ptr(pos_l),
                                   _native.ptr(dom._sp_l), float(table.r_cut), pcode,
                                   _native.SCATTER[args.scatter], _native.ptr(f_t), None,
                                   _native.ptr(r8), _native.ptr(st_t))
        torch.cuda.synchronize()
        pk = measure_peak(lib, ctx, pcode)
        if rc == 0 and pk:
            stv = st_t.cpu().numpy()
            flops = algorithmic_flops(stv) if pcode == 0 else algorithmic_flops32(stv)
            ach = flops / (kern_ms * 1e-3) / 1e12
            roof.update({"achieved": ach, "peak": pk["tflops"], "frac": ach / pk["tflops"],
                         "flops_per_launch_rank0": flops, "peak_source": pk["source"],
                         "kernel": "k_tersoff_warp (rank 0: its owned rows of [owned | ghosts])"})
    # e2e: owned positions from pinned host memory each step, forces back
    pos_h = torch.empty(tuple(dom.pos.shape), dtype=torch.float64).pin_memory()
    pos_h.copy_(dom.pos)
    f_h = torch.empty(tuple(dom.pos.shape), dtype=torch.float64).pin_memory()
    ke = max(10, min(k, args.e2e_steps))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        dom.pos.copy_(pos_h, non_blocking=True)
        f, res = step_fn()
        f_h.copy_(f, non_blocking=True)
        e_host = float(res[0])
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=comm)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": k,
        "warmup": args.warmup, "ms_per_step": t_max * 1e3 / k, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if args.precision == "double" else "f32/f64", "data": "synthetic",
        "config": {"workload": f"config 2 per GPU, weak scaling: {cells[0]}x{cells[1]}x{cells[2]}"
                               f"-cell Si diamond ({n_total} atoms), slab decomposition along x, "
                               f"{backend.upper()} P2P halo + reverse forces + all-reduce per step",
                   "backend": backend,
                   "atoms": n_total, "atoms_per_gpu": n_total // ws,
                   "precision": args.precision, "scatter": args.scatter,
                   "parallelism": f"spatial slabs x{ws}",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "launch": launch},
        "e2e": {"value": n_total * ke / float(te[0]), "unit": UNIT, "steps": ke,
                "h2d_bytes_per_step": int(dom.pos.numel() * 8),
                "d2h_bytes_per_step": int(dom.pos.numel() * 8 + 8),
                "path": "decomp.DecomposedForceField per rank, pinned host positions in, "
                        "forces out, energy to host"},
        "gpu_launches": 2 * k,
        "roofline": roof,
        "clocks": sampler.summary(), "energy_eV": energy,
    }
    if rank == 0:
        print(json.dumps(line, default=_jsonable), flush=True)
    dist.barrier()
    if graph is not None:
        # tearing the process group down under a live captured graph can
        # block at exit: release the graph, then leave without the teardown
        del graph, step_fn
        torch.cuda.synchronize()
        sys.stdout.flush()
        os._exit(0)
    dist.destroy_process_group()


def gpu_arm(args):
    import ctypes
    import torch
    ws, rank, local = dist_setup()
    if ws > 1 and not args.replicas:
        return gpu_arm_decomposed(args)
    dev = local if ws > 1 else 0
    torch.cuda.set_device(dev)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    import paper_1710_00882_b200 as B
    from paper_1710_00882_b200 import _native, structures
    from paper_1710_00882_b200.paramfile import builtin_params

    state, tname = structures.config(args.config)
    table = builtin_params(tname)
    n = state.natoms
    stream = torch.cuda.Stream(device=dev)   # one explicit stream for torch and the C ABI
    torch.cuda.set_stream(stream)
    ctx = _native.default_context(dev)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_table(table)
    lib = ctx.lib

    pos = torch.from_numpy(state.positions).to(f"cuda:{dev}").contiguous()
    species = torch.from_numpy(state.species.astype(np.int32)).to(f"cuda:{dev}")
    forces = torch.empty((n, 3), dtype=torch.float64, device=pos.device)
    per_atom = torch.empty(n, dtype=torch.float64, device=pos.device)
    result = torch.zeros(8, dtype=torch.float64, device=pos.device)
    stats = torch.zeros(_native.NSTATS, dtype=torch.int64, device=pos.device)

    class DevState:
        pass

    ds = DevState()
    ds.positions, ds.species, ds.box = pos, species, state.box
    nl = B.build_neighbor_list(ds, table.r_cut, 0.3, device=dev)
    scat = _native.SCATTER[args.scatter]
    P = _native.ptr

    def step(precision, with_stats=False):
        rc = lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(species),
                                   float(table.r_cut), precision, scat, P(forces),
                                   P(per_atom), P(result), P(stats) if with_stats else None)
        if rc:
            ctx.check(rc, "tb_compute_device")

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=pos.device)

    def capture(precision):
        """The evaluation (Tersoff kernel + finalize) as one CUDA graph."""
        for _ in range(3):
            step(precision)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step(precision)
        ctx.set_stream(stream.cuda_stream)
        torch.cuda.synchronize()
        return g

    def timed_graph(g, k):
        """k steps, L2 flushed between steps (outside the event bracket)."""
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        for s_ in range(k):
            flush.zero_()
            starts[s_].record(stream)
            g.replay()
            ends[s_].record(stream)
        torch.cuda.synchronize()
        return sum(a_.elapsed_time(b_) for a_, b_ in zip(starts, ends))

    def kernel_time(precision, k):
        """Average Tersoff-kernel duration (CUDA events bracketing each launch on
        the launch stream, tb_profile), same flush protocol."""
        lib.tb_profile(ctx.handle, 1)
        for _ in range(k):
            flush.zero_()
            step(precision)
        torch.cuda.synchronize()
        lib.tb_profile(ctx.handle, 0)
        tot, cnt = ctypes.c_double(), ctypes.c_int64()
        ctx.check(lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(cnt)))
        return tot.value / max(cnt.value, 1)

    prec = _native.PRECISION[args.precision]
    for _ in range(max(3, args.warmup)):
        step(prec)
    step(prec, with_stats=True)
    torch.cuda.synchronize()
    ctx.check(lib.tb_check_errors(ctx.handle), "warm-up")
    st = stats.cpu().numpy().astype(np.int64)
    energy0 = float(result[0])
    g = capture(prec)

    sampler = ClockSampler(dev)
    with sampler:
        step_ms = timed_graph(g, args.steps)
    ctx.check(lib.tb_check_errors(ctx.handle), "timed loop")
    t_local = step_ms / 1e3
    if ws > 1:
        t = torch.tensor([t_local], dtype=torch.float64, device=pos.device)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_max = float(t[0])
    else:
        t_max = t_local
    value = ws * n * args.steps / t_max

    # roofline of the Tersoff kernel (the dominant launch of the step)
    kern_ms = kernel_time(prec, min(args.steps, 200))
    flops = algorithmic_flops(st) if args.precision == "double" else algorithmic_flops32(st)
    peak = measure_peak(lib, ctx, prec) if rank == 0 else None
    achieved = flops / (kern_ms / 1e3) / 1e12
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_tersoff_fp64.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    extra = {}
    if args.extras and rank == 0 and args.precision == "double":
        # mixed precision on the same workload, against the FP32 pipe
        gm = capture(1)
        k2 = max(10, args.steps // 2)
        mixed_ms = timed_graph(gm, k2)
        mk = kernel_time(1, min(k2, 200))
        mflops = algorithmic_flops32(st)
        mpeak = measure_peak(lib, ctx, 1)
        extra["mixed"] = {
            "value": n * k2 / (mixed_ms / 1e3), "unit": UNIT, "steps": k2,
            "ms_per_step": mixed_ms / k2, "dtype": "f32 math / f64 positions+accumulators",
            "roofline": {"bound": "fp32", "achieved": mflops / (mk / 1e3) / 1e12,
                         "peak": mpeak["tflops"] if mpeak else None, "unit": "TFLOP/s",
                         "frac": (mflops / (mk / 1e3) / 1e12) / mpeak["tflops"] if mpeak else None,
                         "kernel_ms": mk, "flops_per_launch": mflops,
                         "peak_source": mpeak["source"] if mpeak else None}}
        step(prec)  # restore the fp64 result buffers
        torch.cuda.synchronize()

    if args.extras and rank == 0 and args.config == 2:
        # SURVEY 8(d) "full MD step": velocity Verlet + rebuilds amortised,
        # BASELINE config 2 protocol, the whole run one CUDA-graph launch
        extra["md"] = {}
        for pname, pcode in (("double", 0), ("single", 1)):
            r = md_measure(B, _native, ctx, state, table, dev, pcode, scat)
            fl = algorithmic_flops(st) if pcode == 0 else algorithmic_flops32(st)
            pk = peak if pcode == 0 else measure_peak(lib, ctx, 1)
            r["roofline_frac"] = (fl / (r["ms_per_step"] / 1e3) / 1e12 / pk["tflops"]
                                  if pk else None)
            extra["md"][pname] = r
        ctx.set_stream(stream.cuda_stream)
        step(prec)
        torch.cuda.synchronize()

    e2e = None
    if rank == 0:
        e2e = e2e_arm(args, B, state, table, nl, dev)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if args.precision == "double" else "f32/f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {args.config}: {n}-atom "
                               f"{'Si diamond' if tname == 'Si' else tname}, one E+F+virial "
                               f"evaluation per step (skin-list repack at r_cut, Tersoff "
                               f"terms, force/energy/virial reduction), neighbour list built "
                               f"outside the timed region",
                   "atoms": n, "precision": args.precision, "scatter": args.scatter,
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "launch": "each step is one CUDA-graph replay (Tersoff kernel + finalize)"},
        "e2e": e2e,
        "gpu_launches": 2 * args.steps,
        "roofline": {"bound": "fp64" if args.precision == "double" else "fp32",
                     "achieved": achieved,
                     "peak": peak["tflops"] if peak else None, "unit": "TFLOP/s",
                     "frac": achieved / peak["tflops"] if peak else None,
                     "traffic": traffic,
                     "kernel": f"k_tersoff_warp<{'double' if prec == 0 else 'float'},S=1,{args.scatter}>",
                     "kernel_ms": kern_ms,
                     "flops_per_launch": flops,
                     "flop_convention": "SURVEY 8(d): reference ScalarOpt expression tree "
                                        "charged once per live pair and live triplet; "
                                        f"library-call weights {OP_WEIGHTS_SOURCE} "
                                        "(profiles/roofline.json)",
                     "flops_per_unit": {"pair": FLOPS_PAIR, "triplet": FLOPS_TRIP,
                                        "taper": FLOPS_TAPER},
                     "peak_source": peak["source"] if peak else None,
                     "counts": {"live_pairs": int(st[2]), "live_triplets": int(st[3]),
                                "taper_pairs": int(st[4]), "taper_triplets": int(st[5]),
                                "zeta_visits": int(st[0])}},
        "clocks": sampler.summary(),
        "energy_eV": energy0,
    }
    line.update(extra)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        v, cores, evals, el = oracle_baseline(state, table, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{evals} full E+F evaluations of the {n}-atom system "
                                          f"in {el:.1f} s (NL outside the timer); oracle/ C "
                                          f"restatement of ScalarOpt, OpenMP {cores} threads"}
    if rank == 0:
        print(json.dumps(line, default=_jsonable), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def md_measure(B, _native, ctx, state, table, dev, precision, scat, steps=1000, warm=20):
    """Device-resident NVE (tb_md_run): BASELINE config 2 protocol -- dt 1 fs,
    skin 0.3, rebuild every 10 steps plus the skin/2 trigger -- timed with
    CUDA events around one graph launch of `steps` steps after a `warm`-step
    launch that captures the graph."""
    import ctypes

    import torch
    from paper_1710_00882_b200.state import ACCEL
    n = state.natoms
    d = torch.device("cuda", dev)
    pos = torch.from_numpy(state.positions.copy()).to(d)
    vel = torch.from_numpy(state.velocities.copy()).to(d)
    mass = torch.from_numpy(np.ascontiguousarray(state.atom_masses, dtype=np.float64)).to(d)
    species = torch.from_numpy(state.species.astype(np.int32)).to(d)
    forces = torch.empty((n, 3), dtype=torch.float64, device=d)
    result = torch.zeros(8, dtype=torch.float64, device=d)
    series = torch.zeros((steps // 100 + 1, 2), dtype=torch.float64, device=d)

    class DS:
        pass

    ds = DS()
    ds.positions, ds.species, ds.box = pos, species, state.box
    s = torch.cuda.current_stream(d)
    ctx.set_stream(s.cuda_stream)
    nl = B.build_neighbor_list(ds, table.r_cut, 0.3, device=dev)
    lib, P = ctx.lib, _native.ptr
    ctx.check(lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(species),
                                    float(table.r_cut), precision, scat, P(forces), None,
                                    P(result), None), "tb_compute_device")
    nreb = ctypes.c_int64()

    def run(k):
        ctx.check(lib.tb_md_run(ctx.handle, nl._nl.handle, n, P(pos), P(vel), P(forces), P(mass),
                                P(species), 1.0, float(ACCEL), float(table.r_cut), 0.3, 10,
                                precision, scat, k, 100, P(series), P(result),
                                ctypes.byref(nreb)), "tb_md_run")
        return int(nreb.value)

    run(warm)
    torch.cuda.synchronize(d)
    e0 = float(result[0]) + float(result[7])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    rebuilds = run(steps)
    b.record(s)
    torch.cuda.synchronize(d)
    ms = a.elapsed_time(b)
    e1 = float(result[0]) + float(result[7])
    return {"value": n * steps / (ms / 1e3), "unit": UNIT, "steps": steps,
            "ms_per_step": ms / steps, "rebuilds": rebuilds,
            "rel_energy_change": abs(e1 - e0) / abs(e0),
            "workload": f"config 2 NVE ({n} Si, 1000 K, dt 1 fs, skin 0.3, rebuild every 10 "
                        f"steps + skin/2 trigger): velocity Verlet + device-side list rebuilds "
                        f"+ E/F/virial per step, one CUDA-graph launch (tb_md_run)",
            "l2": "not flushed: consecutive steps of one run",
            "gpu_launches": "1 graph launch (WHILE/IF conditional nodes)"}


def measure_peak(lib, ctx, precision):
    """FMA-pipe peak measured on this GPU (MEASURED_PEAKS.json has no fp64/fp32
    figure): an 8-chain FMA loop over all SMs, best of 5 (tb_measure_peak)."""
    import ctypes
    out = ctypes.c_double()
    if lib.tb_measure_peak(ctx.handle, int(precision), ctypes.byref(out)) != 0:
        return None
    return {"tflops": out.value,
            "source": f"measured {'DFMA' if precision == 0 else 'FFMA'} loop in bench.py "
                      f"(tb_measure_peak; MEASURED_PEAKS.json has no fp64/fp32 entry)"}


def e2e_arm(args, B, state, table, nl, dev):
    """compute() through the public API with pinned host arrays; wall clock
    with a device synchronise at both ends (compute() itself synchronises)."""
    import torch
    n = state.natoms
    pos_h = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    pos_h[:] = state.positions
    sp_h = torch.empty(n, dtype=torch.int32).pin_memory().numpy()
    sp_h[:] = state.species

    class HostState:
        pass

    hs = HostState()
    hs.positions, hs.species, hs.box = pos_h, sp_h, state.box
    variant = B.make_variant("B200", precision=args.precision, scatter=args.scatter)
    # caller-owned pinned result buffers (compute(..., out=)): D2H by DMA
    out = B.ForceEnergyResult(torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy(),
                              0.0, torch.empty(n, dtype=torch.float64).pin_memory().numpy(), {})
    for _ in range(3):
        B.compute(hs, nl, table, variant, out=out)
    k = max(10, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        res = B.compute(hs, nl, table, variant, out=out)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    assert np.isfinite(res.potential_energy)
    return {"value": n * k / el, "unit": UNIT, "steps": k,
            "h2d_bytes_per_step": n * 3 * 8 + n * 4,
            "d2h_bytes_per_step": n * 3 * 8 + n * 8 + 7 * 8 + 6 * 8,
            "path": "paper_1710_00882_b200.compute(state, nl, params, variant, out=pinned), "
                    "pinned host positions+species in, pinned host forces/per-atom energy out, "
                    "energy/virial/stats to host, wall clock per call (synchronous)"}


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--precision", choices=["double", "single"], default="double")
    ap.add_argument("--precision-ref", dest="precision_ref", default="double")
    ap.add_argument("--scatter", choices=["atomic", "gather"], default="atomic")
    ap.add_argument("--e2e-steps", type=int, default=300)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", dest="extras", action="store_false")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas instead of the slab decomposition")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
