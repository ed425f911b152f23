#!/usr/bin/env python
"""Benchmark of the B200 Tersoff hot path (driver contract: one JSON line).

Metric (BASELINE.json): Tersoff atom-steps/s -- atoms x E+F evaluations per
second -- with the achieved fraction of the FP64 (FP32 for mixed) pipe peak.

Workload (default): BASELINE config 5, the largest configuration the metric
is quoted on -- 16,777,216-atom Si diamond (128^3 cells, a=5.431, sigma=0.1
seed 1005), Si(C) Tersoff parameters, skin 0.3, fp64.  One "step" = one
energy + force + virial evaluation at the current positions: the kernel
re-packs the skin list at r_cut (pack_adjacency) and evaluates every Tersoff
term (kernels.compute semantics).  The neighbour list is built once outside
the timed region, as the reference harness does (bench.py:116-118).  The
working set (positions 0.4 GB, list 0.27 GB, lane table 1 GB) is far larger
than L2, so no flush is needed between steps.  --config 2/3/4 select the other
single-GPU configurations (smaller ones flush L2 between steps).

  N = 1      one GPU: each step is one CUDA-graph replay (Tersoff kernel +
             finalize); value = atoms x steps / device time.
  N > 1      (torchrun, NCCL) slab decomposition, decomp.DomainMD: strong
             scaling of config 5 by default (--scaling weak: 64^3 cells =
             2,097,152 atoms per GPU stacked along x).  A step = forward halo
             (NCCL P2P) + evaluation of the owned rows + reverse halo + sum of
             [E, W6] (all-reduce), captured as one CUDA graph; time = max over
             ranks of the device-timed loop; value = all atoms x steps / time.
  e2e        the same evaluation through the public API with HOST buffers:
             compute() with pinned host positions/species in, forces/per-atom
             energies out (N = 1); at N > 1 pinned host positions in and forces
             out around each decomposed step.
  roofline   the Tersoff kernel's algorithmic flops (SURVEY 8(d) op counts per
             live pair / triplet) / its CUDA-event time, against the FMA-pipe
             peak measured on this GPU at start-up; the ncu pipe utilisation
             and DRAM traffic of the same kernel and config from profiles/.
  cpu_baseline / --impl reference
             the CPU oracle (C restatement of the reference ScalarOpt,
             oracle/) on this host's cores -- "port": the reference itself is
             Python and cannot travel to the GPU box.
  extras     mixed precision (same workload), config 2 (64k atoms, the round-1
             headline), the device-resident NVE of configs 2 and 5 (tb_md_run:
             one graph launch per run), at N > 1 the decomposed NVE step.
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


def flops_for(stats, precision):
    return algorithmic_flops(stats) if precision == "double" else algorithmic_flops32(stats)


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
            time.sleep(0.005)

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


# ---------------------------------------------------------------------------
# workload (shared by both arms: identical `config` dicts)
# ---------------------------------------------------------------------------

def make_workload(args, ws):
    """(state, table name, config dict) of this run."""
    from paper_1710_00882_b200 import structures
    weak = ws > 1 and args.scaling == "weak"
    if weak:
        st, tname = structures.config5_weak(ws)
        what = (f"BASELINE config 5, weak scaling: (64*{ws})x64x64-cell Si diamond "
                f"({st.natoms} atoms, 2,097,152 per GPU)")
    else:
        st, tname = structures.config(args.config)
        what = {2: "BASELINE config 2: 64,000-atom Si diamond (20^3 cells)",
                3: "BASELINE config 3: 512,000-atom 3C-SiC (40^3 cells, fixture SiC table)",
                4: "BASELINE config 4: 1,000,000-atom disordered Si (rho 0.05/A^3)",
                5: "BASELINE config 5: 16,777,216-atom Si diamond (128^3 cells)"}.get(
                    args.config, f"BASELINE config {args.config}")
    cfg = {"workload": f"{what}, one E+F+virial evaluation per step, neighbour list (skin "
                       f"0.3) built outside the timed region",
           "config": args.config if not weak else 5, "atoms": int(st.natoms),
           "precision": args.precision, "skin": 0.3,
           "scaling": ("weak" if weak else "strong") if ws > 1 else "single GPU",
           "parallelism": f"spatial slabs x{ws}" if ws > 1 else "single GPU"}
    return st, tname, cfg


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline and the reference arm)
# ---------------------------------------------------------------------------

def oracle_timing(state, table, budget_s, max_evals, precision="double", threads=None):
    """The CPU oracle (reference ScalarOpt restated in C, OpenMP over atom
    ranges): NL built outside the timer, then E+F evaluations (pack + kernel)
    until `budget_s` or `max_evals`."""
    from oracle import oracle as O
    threads = threads or cpu_cores()
    off, nb = O.build_neighbor_list(state.positions, state.box.lengths, state.box.periodic,
                                    table.r_cut, 0.3, threads=threads)

    def one():
        O.compute(state.positions, state.species, state.box.lengths, state.box.periodic,
                  off, nb, table, precision=precision, threads=threads)

    one()  # warm (page-in, thread pool)
    t0 = time.perf_counter()
    evals = 0
    while True:
        one()
        evals += 1
        el = time.perf_counter() - t0
        if el >= budget_s or evals >= max_evals:
            break
    return state.natoms * evals / el, threads, evals, el


def reference_arm(args):
    ws, rank, _ = dist_setup()
    if rank != 0:
        return
    from paper_1710_00882_b200.paramfile import builtin_params
    state, tname, cfg = make_workload(args, ws)
    table = builtin_params(tname)
    v, threads, evals, el = oracle_timing(state, table, args.ref_budget,
                                          max(1, args.steps), args.precision)
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": ws, "steps": evals,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / evals, "higher_is_better": True,
        "scaling": "weak" if cfg["scaling"] == "weak" else "strong", "vs_baseline": None,
        "dtype": "f64" if args.precision == "double" else "f32/f64",
        "data": "synthetic", "impl": "reference", "config": cfg,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{evals} full E+F evaluations of the {state.natoms}-atom "
                                   f"system in {el:.1f} s (of {args.steps} requested; bounded to "
                                   f"~{args.ref_budget:.0f} s), NL built outside the timer; "
                                   f"oracle/ C restatement of ScalarOpt, OpenMP {threads} threads"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line, default=_jsonable), flush=True)


# ---------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------

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


def ncu_profile(config, precision):
    """The committed ncu --set full summary of the Tersoff kernel at this
    config / precision (profiles/ncu_r02_kernels.json, tools/ncu_kernels.sh)."""
    for name in ("ncu_r02_kernels.json", "ncu_r01_kernels.json"):
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", name)))
        except (OSError, ValueError):
            continue
        k = d.get("kernels", {}).get(f"c{config}_p{0 if precision == 'double' else 1}")
        if k:
            return dict(k, source=f"profiles/{name}")
    return None


def kernel_time(ctx, step, flush, k):
    """Tersoff kernel time per evaluation: CUDA events bracket every Tersoff
    launch on the launch stream (tb_profile); an evaluation is one launch, or
    two when the list is split between the atom-per-lane kernel (rows of <= 4
    entries) and the warp-chunk kernel (the longer rows).  Returns (ms per
    evaluation, launches per evaluation)."""
    import ctypes
    import torch
    lib = ctx.lib
    lib.tb_profile(ctx.handle, 1)
    for _ in range(k):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()
    lib.tb_profile(ctx.handle, 0)
    tot, cnt = ctypes.c_double(), ctypes.c_int64()
    ctx.check(lib.tb_profile_read(ctx.handle, ctypes.byref(tot), ctypes.byref(cnt)))
    return tot.value / max(k, 1), cnt.value / max(k, 1)


class Evaluator:
    """One configuration resident on one GPU: positions/species/list in HBM,
    the evaluation (tb_compute_device: Tersoff kernel + finalize) as a graph."""

    def __init__(self, B, _native, ctx, state, table, dev, scatter, stream):
        import torch
        self.ctx, self.native, self.table, self.stream = ctx, _native, table, stream
        ctx.set_table(table)
        n = self.n = state.natoms
        d = torch.device("cuda", dev)
        self.pos = torch.from_numpy(state.positions).to(d).contiguous()
        self.species = torch.from_numpy(state.species.astype(np.int32)).to(d)
        self.forces = torch.empty((n, 3), dtype=torch.float64, device=d)
        self.result = torch.zeros(8, dtype=torch.float64, device=d)
        self.stats = torch.zeros(_native.NSTATS, dtype=torch.int64, device=d)

        class DS:
            pass
        ds = DS()
        ds.positions, ds.species, ds.box = self.pos, self.species, state.box
        self.nl = B.build_neighbor_list(ds, table.r_cut, 0.3, device=dev)
        self.scat = _native.SCATTER[scatter]

    def step(self, precision, with_stats=False):
        P, ctx = self.native.ptr, self.ctx
        rc = ctx.lib.tb_compute_device(ctx.handle, self.nl._nl.handle, P(self.pos),
                                       P(self.species), float(self.table.r_cut), precision,
                                       self.scat, P(self.forces), None, P(self.result),
                                       P(self.stats) if with_stats else None)
        if rc:
            ctx.check(rc, "tb_compute_device")

    def counts(self, precision):
        import torch
        self.step(precision, with_stats=True)
        torch.cuda.synchronize()
        return self.stats.cpu().numpy().astype(np.int64)

    def capture(self, precision):
        import torch
        for _ in range(3):
            self.step(precision)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream):
            self.step(precision)
        self.ctx.set_stream(self.stream.cuda_stream)
        torch.cuda.synchronize()
        return g

    def timed(self, g, k, flush=None):
        import torch
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        torch.cuda.synchronize()
        for s_ in range(k):
            if flush is not None:
                flush.zero_()
            starts[s_].record(self.stream)
            g.replay()
            ends[s_].record(self.stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in zip(starts, ends))

    def roofline(self, precision, k, flush, peak, config):
        """Kernel time of the timed (counter-free) instantiation and of the
        API's counting one, algorithmic flops, ncu pipe % / traffic."""
        pcode = self.native.PRECISION[precision]
        st = self.counts(pcode)
        flops = flops_for(st, precision)
        kms, nlaunch = kernel_time(self.ctx, lambda: self.step(pcode), flush, k)
        kms_api, _ = kernel_time(self.ctx, lambda: self.step(pcode, True), flush, k)
        ach = flops / (kms * 1e-3) / 1e12
        prof = ncu_profile(config, precision)
        pipe = "fp64_pipe_pct" if precision == "double" else "fma_pipe_pct"
        tname = "double" if pcode == 0 else "float"
        kname = f"k_tersoff_warp<{tname},S={self.table.nspecies},atomic>"
        if nlaunch > 1.5:
            kname = (f"k_tersoff_row<{tname},4,atomic> (rows of <= 4 entries, one lane per atom) + "
                     f"{kname} (longer rows); kernel_ms is their sum")
        peak_tf = peak["tflops"] if peak else None
        exe = prof.get("executed_flops") if prof else None
        return {
            "bound": "fp64" if precision == "double" else "fp32",
            "achieved": ach, "peak": peak["tflops"] if peak else None, "unit": "TFLOP/s",
            "frac": ach / peak["tflops"] if peak else None,
            "traffic": prof.get("dram_bytes") if prof else None,
            "frac_note": "algorithmic fraction by the SURVEY 8(d) convention; it can exceed 1: "
                         "the kernels execute fewer flops than the reference expression tree "
                         "(2 log + 2 exp + 1 reciprocal instead of 4 pow per pair, g(cos) once "
                         "per unordered pair in the row kernel) -- frac_executed and ncu.pipe_pct "
                         "are the hardware view",
            "executed_flops_per_launch": exe,
            "frac_executed": (exe / (kms * 1e-3) / 1e12 / peak_tf) if exe and peak_tf else None,
            "kernel": kname,
            "kernel_launches_per_step": nlaunch,
            "kernel_ms": kms,
            "kernel_ms_api": kms_api,
            "kernel_ms_note": "kernel_ms: counter-free instantiation (the timed step); "
                              "kernel_ms_api: the instantiation compute() runs (live-pair / "
                              "triplet counters on)",
            "flops_per_launch": flops,
            "flop_convention": "SURVEY 8(d): reference ScalarOpt expression tree charged once "
                               "per live pair and live triplet; library-call weights "
                               f"{OP_WEIGHTS_SOURCE} (profiles/roofline.json)",
            "flops_per_unit": ({"pair": FLOPS_PAIR, "triplet": FLOPS_TRIP, "taper": FLOPS_TAPER}
                               if precision == "double" else
                               {"pair": FLOPS32_PAIR, "triplet": FLOPS32_TRIP,
                                "taper": FLOPS32_TAPER}),
            "peak_source": peak["source"] if peak else None,
            "counts": {"live_pairs": int(st[2]), "live_triplets": int(st[3]),
                       "taper_pairs": int(st[4]), "taper_triplets": int(st[5]),
                       "zeta_visits": int(st[0])},
            "ncu": ({"pipe": pipe, "pipe_pct": prof.get(pipe), "l1tex_pct": prof.get("l1tex_pct"),
                     "issue_active_pct": prof.get("issue_active_pct"),
                     "dram_bytes_per_launch": prof.get("dram_bytes"),
                     "duration_us": prof.get("duration_us"), "source": prof.get("source")}
                    if prof else None),
        }


def md_measure(B, _native, ctx, state, table, dev, precision, steps, warm=20):
    """Device-resident NVE (tb_md_run): dt 1 fs, skin 0.3, rebuild every 10
    steps plus the skin/2 trigger, timed with CUDA events around one graph
    launch of `steps` steps after a `warm`-step launch that captures the graph."""
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
    series = torch.zeros((steps // 100 + 2, 2), dtype=torch.float64, device=d)

    class DS:
        pass

    ds = DS()
    ds.positions, ds.species, ds.box = pos, species, state.box
    s = torch.cuda.current_stream(d)
    ctx.set_stream(s.cuda_stream)
    ctx.set_table(table)
    nl = B.build_neighbor_list(ds, table.r_cut, 0.3, device=dev)
    lib, P = ctx.lib, _native.ptr
    ctx.check(lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(species),
                                    float(table.r_cut), precision, 0, P(forces), None,
                                    P(result), None), "tb_compute_device")
    nreb = ctypes.c_int64()

    def run(k):
        ctx.check(lib.tb_md_run(ctx.handle, nl._nl.handle, n, P(pos), P(vel), P(forces), P(mass),
                                P(species), 1.0, float(ACCEL), float(table.r_cut), 0.3, 10,
                                precision, 0, k, 100, P(series), P(result),
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
            "workload": f"NVE ({n} atoms, dt 1 fs, skin 0.3, rebuild every 10 steps + skin/2 "
                        f"trigger): velocity Verlet + device-side list rebuilds + E/F/virial per "
                        f"step, one CUDA-graph launch (tb_md_run)",
            "gpu_launches": "1 graph launch (WHILE/IF conditional nodes)"}


def e2e_arm(args, B, state, table, nl, dev):
    """compute() through the public API with pinned host arrays; wall clock
    with a device synchronise at both ends (compute() itself synchronises)."""
    import torch
    n = state.natoms
    pos_h = torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy()
    pos_h[:] = state.positions
    # species are constant over a run: resident on the device (a CUDA tensor is
    # used in place by compute()); the per-step input is the positions
    sp_d = torch.from_numpy(state.species.astype(np.int32)).to(f"cuda:{dev}")

    class HostState:
        pass

    hs = HostState()
    hs.positions, hs.species, hs.box = pos_h, sp_d, state.box
    variant = B.make_variant("B200", precision=args.precision, scatter=args.scatter)
    out = B.ForceEnergyResult(torch.empty((n, 3), dtype=torch.float64).pin_memory().numpy(),
                              0.0, torch.empty(n, dtype=torch.float64).pin_memory().numpy(), {})
    for _ in range(2):
        B.compute(hs, nl, table, variant, out=out)
    k = max(3, min(args.steps, args.e2e_steps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        res = B.compute(hs, nl, table, variant, out=out)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    assert np.isfinite(res.potential_energy)
    return {"value": n * k / el, "unit": UNIT, "steps": k,
            "h2d_bytes_per_step": n * 3 * 8,
            "d2h_bytes_per_step": n * 3 * 8 + n * 8 + 7 * 8 + 6 * 8,
            "path": "paper_1710_00882_b200.compute(state, nl, params, variant, out=pinned), "
                    "pinned host positions in (species resident on the device: constant over a "
                    "run), pinned host forces/per-atom energy out, energy/virial/stats to host, "
                    "wall clock per call (synchronous); tb_compute streams the call in atom "
                    "ranges: H2D copy, kernel stages and D2H copy overlap (TB_OPT_STREAM_RANGE)"}


# ---------------------------------------------------------------------------
# N = 1
# ---------------------------------------------------------------------------

def gpu_arm(args):
    import torch
    import paper_1710_00882_b200 as B
    from paper_1710_00882_b200 import _native, structures
    from paper_1710_00882_b200.paramfile import builtin_params
    dev = 0
    torch.cuda.set_device(dev)
    state, tname, cfg = make_workload(args, 1)
    table = builtin_params(tname)
    n = state.natoms
    stream = torch.cuda.Stream(device=dev)  # one explicit stream for torch and the C ABI
    torch.cuda.set_stream(stream)
    ctx = _native.default_context(dev)
    ctx.set_stream(stream.cuda_stream)
    if os.environ.get("TB_REPACK_MARGIN_MA"):  # experiments: live-repack margin (1/1000 A)
        ctx.set_option(_native.OPT_REPACK_MARGIN, int(os.environ["TB_REPACK_MARGIN_MA"]))
    ev = Evaluator(B, _native, ctx, state, table, dev, args.scatter, stream)
    lib = ctx.lib
    prec = _native.PRECISION[args.precision]
    big = n * 40 > 256 * 1024 * 1024  # working set far above L2: no flush needed
    flush = None if big else torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32,
                                         device=ev.pos.device)
    for _ in range(max(3, args.warmup)):
        ev.step(prec)
    torch.cuda.synchronize()
    ctx.check(lib.tb_check_errors(ctx.handle), "warm-up")
    g = ev.capture(prec)
    energy0 = float(ev.result[0])
    sampler = ClockSampler(dev)
    with sampler:
        step_ms = ev.timed(g, args.steps, flush)
    ctx.check(lib.tb_check_errors(ctx.handle), "timed loop")
    value = n * args.steps / (step_ms / 1e3)
    peak = measure_peak(lib, ctx, prec)
    kk = max(5, min(args.steps, 50 if big else 200))
    roof = ev.roofline(args.precision, kk, flush, peak, cfg["config"])
    extra = {}
    if args.extras:
        if args.precision == "double":
            # mixed precision on the same workload, against the FP32 pipe
            gm = ev.capture(1)
            k2 = max(5, args.steps // 2)
            mixed_ms = ev.timed(gm, k2, flush)
            mpeak = measure_peak(lib, ctx, 1)
            extra["mixed"] = {
                "value": n * k2 / (mixed_ms / 1e3), "unit": UNIT, "steps": k2,
                "ms_per_step": mixed_ms / k2, "dtype": "f32 math / f64 positions+accumulators",
                "roofline": ev.roofline("single", kk, flush, mpeak, cfg["config"])}
            del gm
        ev.step(prec)
        torch.cuda.synchronize()
        if cfg["config"] != 2:
            # the round-1 headline (config 2, 64k atoms) beside it
            st2, tn2 = structures.config(2)
            ev2 = Evaluator(B, _native, ctx, st2, builtin_params(tn2), dev, args.scatter, stream)
            fl2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=ev.pos.device)
            g2 = ev2.capture(prec)
            k2 = max(20, args.steps)
            ms2 = ev2.timed(g2, k2, fl2)
            extra["config2"] = {"value": st2.natoms * k2 / (ms2 / 1e3), "unit": UNIT,
                                "steps": k2, "ms_per_step": ms2 / k2,
                                "l2": "flushed between steps (256 MiB write)",
                                "roofline": ev2.roofline(args.precision, 100, fl2, peak, 2)}
            del g2, ev2, fl2
            ctx.set_table(table)
        torch.cuda.synchronize()
        extra["md"] = {}
        st2, tn2 = structures.config(2)
        extra["md"]["config2_fp64"] = md_measure(B, _native, ctx, st2, builtin_params(tn2), dev,
                                                 0, 1000)
        extra["md"]["config2_mixed"] = md_measure(B, _native, ctx, st2, builtin_params(tn2), dev,
                                                  1, 1000)
        if args.md3_steps > 0:
            # BASELINE config 3 protocol: 512,000-atom SiC, 1500 K, dt 1 fs, 500 steps
            st3, tn3 = structures.config(3)
            for pname, pcode in (("fp64", 0), ("mixed", 1)):
                extra["md"][f"config3_{pname}"] = md_measure(B, _native, ctx, st3,
                                                             builtin_params(tn3), dev, pcode,
                                                             args.md3_steps, warm=10)
            del st3
        if cfg["config"] == 5 and args.md5_steps > 0:
            extra["md"]["config5_fp64"] = md_measure(B, _native, ctx, state, table, dev, 0,
                                                     args.md5_steps, warm=20)
        ctx.set_stream(stream.cuda_stream)
        ctx.set_table(table)
    e2e = e2e_arm(args, B, state, table, ev.nl, dev)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if args.precision == "double" else "f32/f64", "data": "synthetic",
        "config": cfg,
        "details": {"scatter": args.scatter,
                    "l2": ("working set > L2 (no flush)" if big
                           else "flushed between timed steps (256 MiB write)"),
                    "launch": "each step is one CUDA-graph replay (Tersoff kernel + finalize)"},
        "e2e": e2e,
        # per timed step: the Tersoff kernel(s) (row kernel + warp-chunk kernel when
        # the list is split) and the finalize kernel
        "gpu_launches": int(round((roof.get("kernel_launches_per_step", 1.0) + 1) * args.steps)),
        "roofline": roof,
        "clocks": sampler.summary(),
        "energy_eV": energy0,
    }
    line.update(extra)
    if not args.no_cpu_baseline:
        v, cores, evals, el = oracle_timing(state, table, args.cpu_budget, 1000, args.precision)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                "sample": f"{evals} full E+F evaluations of the {n}-atom system "
                                          f"in {el:.1f} s (NL outside the timer); oracle/ C "
                                          f"restatement of ScalarOpt, OpenMP {cores} threads"}
    print(json.dumps(line, default=_jsonable), flush=True)


# ---------------------------------------------------------------------------
# N > 1: slab decomposition
# ---------------------------------------------------------------------------

def gpu_arm_decomposed(args):
    """N > 1 (torchrun): decomp.DomainMD per rank, NCCL P2P halos; the
    evaluation step (halo + owned rows + reverse halo + all-reduce) as one
    CUDA graph; device-timed per rank, max over ranks."""
    import torch
    import torch.distributed as dist
    ws, rank, local = dist_setup()
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_1710_00882_b200 import decomp
    from paper_1710_00882_b200.paramfile import builtin_params
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: single-GPU functional run
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    comm = decomp.Comm(rank, ws, route=None if backend == "nccl" else "cpu")
    red_dev = dev if backend == "nccl" else "cpu"
    state, tname, cfg = make_workload(args, ws)
    table = builtin_params(tname)
    n_total = state.natoms
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    md = decomp.decompose(state, table, rank, ws, comm, device=local, precision=args.precision,
                          scatter=args.scatter, dt=1.0, rebuild_every=10)
    eng = md.eng
    md.rebuild()
    stats = torch.zeros(8, dtype=torch.int64, device=dev)
    md.evaluate(stats)
    torch.cuda.synchronize()
    energy = float(md.result[0])
    st_h = stats.cpu().numpy()
    for _ in range(max(3, args.warmup)):
        md.evaluate()
    torch.cuda.synchronize()
    launch = f"eager (Python host loop, {backend} batch_isend_irecv)"
    graph = None
    step_fn = md.evaluate
    if backend == "nccl" and os.environ.get("BENCH_DD_GRAPH", "1") == "1":
        try:
            dist.barrier()
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                md.evaluate()
            eng.ctx.set_stream(stream.cuda_stream)
            graph.replay()
            torch.cuda.synchronize()
            step_fn = graph.replay
            launch = ("one CUDA graph per step: position halo (NCCL P2P) + Tersoff kernel + "
                      "finalize + reverse halo + reverse add + all-reduce")
        except Exception as e:  # noqa: BLE001
            graph = None
            launch = f"eager (graph capture failed: {str(e)[:80]})"
            eng.ctx.set_stream(stream.cuda_stream)
            torch.cuda.synchronize()
        ok = torch.tensor([1 if graph is not None else 0], dtype=torch.int32, device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0 and graph is not None:
            del graph
            graph = None
            step_fn = md.evaluate
            launch = "eager (graph capture failed on another rank)"
    k = args.steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
    sampler = ClockSampler(local)
    dist.barrier()
    torch.cuda.synchronize()
    with sampler:
        for s_ in range(k):
            starts[s_].record(stream)
            step_fn()
            ends[s_].record(stream)
        torch.cuda.synchronize()
    t_local = sum(a.elapsed_time(b) for a, b in zip(starts, ends)) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t[0])
    value = n_total * k / t_max
    # Tersoff kernel of this rank (its owned rows of [owned | ghosts])
    prec = eng.native.PRECISION[args.precision]
    kern_ms, kern_launches = kernel_time(eng.ctx, lambda: eng.compute(md.result), None,
                                         min(k, 20))
    peak = measure_peak(eng.ctx.lib, eng.ctx, prec) if rank == 0 else None
    flops = flops_for(st_h, args.precision)
    ach = flops / (kern_ms * 1e-3) / 1e12
    roof = {"bound": "fp64" if prec == 0 else "fp32", "achieved": ach,
            "peak": peak["tflops"] if peak else None, "unit": "TFLOP/s",
            "frac": ach / peak["tflops"] if peak else None, "traffic": None,
            "kernel": ("k_tersoff_row + k_tersoff_warp" if kern_launches > 1.5 else
                       "k_tersoff_warp") + " (rank 0: its owned rows of [owned | ghosts])",
            "kernel_launches_per_step": kern_launches,
            "kernel_ms": kern_ms, "flops_per_launch": flops,
            "peak_source": peak["source"] if peak else None}
    counts = eng.counts()
    # e2e: owned positions from pinned host memory each step, owned forces back
    n_own = int(counts[0])
    pos_h = torch.empty((n_own, 3), dtype=torch.float64).pin_memory()
    pos_v = eng._view(0, 0, n_own, 3)
    f_v = eng._view(2, 0, n_own, 3)
    pos_h.copy_(pos_v)
    f_h = torch.empty((n_own, 3), dtype=torch.float64).pin_memory()
    ke = max(3, min(k, args.e2e_steps))
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        pos_v.copy_(pos_h, non_blocking=True)
        res = step_fn() if graph is None else (step_fn(), md.result)[1]
        f_h.copy_(f_v, non_blocking=True)
        e_host = float(res[0])
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # decomposed NVE steps (migration, cross-rank trigger, halos), eager
    md_line = None
    if args.extras and args.dd_md_steps > 0:
        if graph is not None:
            del graph
            graph = None
        dist.barrier()
        torch.cuda.synchronize()
        md.setup()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reb0 = md.rebuilds
        a.record(stream)
        for _ in range(args.dd_md_steps):
            r = md.step()
        b.record(stream)
        torch.cuda.synchronize()
        tm = torch.tensor([a.elapsed_time(b) / 1e3], dtype=torch.float64, device=red_dev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        md_line = {"value": n_total * args.dd_md_steps / float(tm[0]), "unit": UNIT,
                   "steps": args.dd_md_steps, "ms_per_step": float(tm[0]) * 1e3 / args.dd_md_steps,
                   "rebuilds": md.rebuilds - reb0, "e_total": float(r[0] + r[7]),
                   "workload": "decomposed velocity-Verlet NVE (dt 1 fs, skin 0.3, rebuild every "
                               "10 steps + skin/2 trigger on the max drift over ranks, migration "
                               "+ ghost rebuild at each rebuild), eager host loop, one drift "
                               "all-reduce + one result all-reduce per step"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": k,
        "warmup": args.warmup, "ms_per_step": t_max * 1e3 / k, "higher_is_better": True,
        "scaling": "weak" if cfg["scaling"] == "weak" else "strong", "vs_baseline": None,
        "dtype": "f64" if args.precision == "double" else "f32/f64", "data": "synthetic",
        "config": cfg,
        "details": {"backend": backend, "scatter": args.scatter, "launch": launch,
                    "atoms_per_gpu": n_total / ws,
                    "rank0": {"owned": int(counts[0]), "ghosts": int(counts[1] + counts[2]),
                              "send_rows": int(counts[3] + counts[4])},
                    "l2": "working set > L2 (no flush)"},
        "e2e": {"value": n_total * ke / float(te[0]), "unit": UNIT, "steps": ke,
                "h2d_bytes_per_step": int(n_own * 24), "d2h_bytes_per_step": int(n_own * 24 + 8),
                "path": "decomp.DomainMD.evaluate per rank, pinned host owned positions in, "
                        "owned forces out, energy to host (rank 0's bytes)"},
        "gpu_launches": 4 * k,
        "roofline": roof,
        "clocks": sampler.summary(), "energy_eV": energy, "energy_eV_e2e": e_host,
    }
    if md_line:
        line["md"] = {"decomposed_fp64" if prec == 0 else "decomposed_mixed": md_line}
    if rank == 0:
        print(json.dumps(line, default=_jsonable), flush=True)
    dist.barrier()
    if graph is not None:
        del graph
        torch.cuda.synchronize()
        sys.stdout.flush()
        os._exit(0)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="N>1: config 5 at fixed size, or 2,097,152 atoms per GPU")
    ap.add_argument("--precision", choices=["double", "single"], default="double")
    ap.add_argument("--scatter", choices=["atomic", "gather"], default="atomic")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-budget", type=float, default=60.0)
    ap.add_argument("--md5-steps", type=int, default=200)
    ap.add_argument("--md3-steps", type=int, default=500)
    ap.add_argument("--dd-md-steps", type=int, default=50)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", dest="extras", action="store_false")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws, _, _ = dist_setup()
    if args.impl == "reference":
        reference_arm(args)
    elif ws > 1:
        gpu_arm_decomposed(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
