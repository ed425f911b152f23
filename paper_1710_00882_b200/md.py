"""Molecular-dynamics drivers on the B200 path.

The reference drives compute() from a host loop: ForceField.__call__
(system.py:314-348) re-checks the skin/2 trigger and rebuilds the list before
every evaluation, velocity_verlet_step (:355-380) kicks/drifts on the host,
run_nve (:427-460) records E_pot/E_kin per step.  Here the state lives in HBM:

  ForceField(params, variant, skin)(state)
      drop-in force provider: one host->device copy of the positions (none for
      a CUDA-tensor state), drift check + rebuild on the device
      (tb_needs_rebuild, tb_nlist_rebuild_device), one evaluation, results
      back.  Callable by the reference's own velocity_verlet_step / run_nve.
  md_step(...)   one velocity-Verlet step as one C-ABI call (tb_md_step)
  run_nve(state, params, cfg)
      a whole NVE run as ONE CUDA-graph launch (tb_md_run: kick/drift, the
      rebuild decision and the device list rebuild in conditional nodes, the
      evaluation, the energy record), split only at XYZ dump points; systems
      the graph loop cannot take (free axes, rows > 32 entries, > 2 species)
      run tb_md_step per step.  Same record keys as the reference's run_nve.

Rebuild policy: the reference's skin/2 trigger, plus a fixed cadence when
cfg.rebuild_every > 0 (BASELINE config 2: "rebuilt every 10 steps").
"""

import ctypes
import time as _time
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigurationError, InputError
from .state import ACCEL


@dataclass
class RunConfig:
    """dt (fs), steps, variant (precision/scatter; None = fp64 atomic), skin (A),
    rebuild_every (0 = trigger only), record_every, dump_every/dump_path (XYZ)."""

    dt: float = 0.5
    steps: int = 100
    variant: object = None
    skin: float = 0.3
    threads: int = 1
    dump_every: int = 0
    dump_path: str = None
    rebuild_every: int = 0
    record_every: int = 1

    def __post_init__(self):
        if not self.dt > 0:
            raise ConfigurationError(f"dt must be positive, got {self.dt:g}")
        if self.steps < 0:
            raise ConfigurationError(f"steps must be >= 0, got {self.steps}")
        if self.dump_every < 0 or (self.dump_every and not self.dump_path):
            raise ConfigurationError("dump_every needs dump_path and must be >= 0")
        if self.record_every < 1:
            raise ConfigurationError(f"record_every must be >= 1, got {self.record_every}")


def _variant_modes(variant):
    from .kernels import resolve_variant
    v = resolve_variant(variant)
    return _native.PRECISION[v.precision], _native.SCATTER[v.scatter], v


class _DevState:
    """Duck-typed device state handed to compute()/build_neighbor_list()."""

    def __init__(self, positions, species, box):
        self.positions, self.species, self.box = positions, species, box


class ForceField:
    """Force provider owning a device-resident neighbour list.

    ff(state) -> ForceEnergyResult: rebuilds on the skin/2 trigger before the
    evaluation (system.py:332-337), counts rebuilds/evaluations and phase wall
    clock, raises InputError on non-finite forces (system.py:344-347).  Host
    numpy states get host results; CUDA-tensor states stay on the device."""

    def __init__(self, params, variant=None, skin=0.3, threads=1, device=0):
        self.params, self.skin, self.threads, self.device = params, skin, threads, device
        self.prec, self.scat, self.variant = _variant_modes(variant)
        self.nl = None
        self.rebuilds = self.evaluations = 0
        self.neighbor_s = self.force_s = 0.0
        self._dev = None  # device mirror of host positions / species

    def _device_state(self, state):
        import torch
        pos = state.positions
        if not isinstance(pos, np.ndarray):
            return state
        n = pos.shape[0]
        dev = torch.device("cuda", self.device)
        if self._dev is None or self._dev[0].shape[0] != n:
            self._dev = (torch.empty((n, 3), dtype=torch.float64, device=dev),
                         torch.empty(n, dtype=torch.int32, device=dev), None)
        p, s, sp_host = self._dev
        p.copy_(torch.from_numpy(np.ascontiguousarray(pos, dtype=np.float64)))
        spec = np.asarray(state.species)
        if sp_host is None or sp_host.shape != spec.shape or not np.array_equal(sp_host, spec):
            s.copy_(torch.from_numpy(spec.astype(np.int32)))
            self._dev = (p, s, spec.copy())
        return _DevState(p, s, state.box)

    def __call__(self, state):
        from .kernels import compute
        from .neighbor import build_neighbor_list, needs_rebuild
        t0 = _time.perf_counter()
        host = isinstance(state.positions, np.ndarray)
        ds = self._device_state(state)
        nl = self.nl
        if nl is None or nl.natoms != ds.positions.shape[0] or nl.box is not state.box:
            self.nl = build_neighbor_list(ds, self.params.r_cut, self.skin, device=self.device,
                                          reuse=nl)
            self.rebuilds += 1
        elif needs_rebuild(ds, nl):
            try:  # device builder: no host round trip between its kernels
                nl.rebuild_on_device(ds.positions, ds.species, scatter=self.variant.scatter)
            except RuntimeError:
                self.nl = build_neighbor_list(ds, self.params.r_cut, self.skin,
                                              device=self.device, reuse=nl)
            self.rebuilds += 1
        t1 = _time.perf_counter()
        self.neighbor_s += t1 - t0
        res = compute(ds, self.nl, self.params, self.variant, self.threads)
        if not bool(np.isfinite(float(res.potential_energy))) or \
                not bool(_all_finite(res.forces)):
            f = _host(res.forces)
            bad = int(np.argwhere(~np.isfinite(f))[0][0])
            raise InputError(f"non-finite force on atom {bad} at t={getattr(state, 'time', 0.0):g} fs")
        if host:
            res.forces = _host(res.forces)
            res.per_atom_energy = _host(res.per_atom_energy)
        self.force_s += _time.perf_counter() - t1
        self.evaluations += 1
        return res


def _host(a):
    return a if isinstance(a, np.ndarray) else a.detach().cpu().numpy()


def _all_finite(a):
    if isinstance(a, np.ndarray):
        return np.isfinite(a).all()
    import torch
    return bool(torch.isfinite(a).all())


def md_step(ctx, nl, pos, vel, forces, mass, species, box, dt, r_cut, skin, precision=0,
            scatter=0, force_rebuild=False, result=None):
    """One velocity-Verlet step on device tensors (tb_md_step): v += dt/2 a F/m,
    x += dt v, wrap, rebuild on the trigger (or force_rebuild), F(t+dt),
    v += dt/2 a F/m, E_kin.  Returns (rebuilt, result[8] device tensor)."""
    import torch
    if result is None:
        result = torch.zeros(8, dtype=torch.float64, device=pos.device)
    L = np.ascontiguousarray(np.asarray(box.lengths, dtype=np.float64))
    per = np.ascontiguousarray(np.asarray(box.periodic, dtype=np.int32))
    flag = np.zeros(1, dtype=np.int32)
    P = _native.ptr
    ctx.check(ctx.lib.tb_md_step(ctx.handle, nl._nl.handle, pos.shape[0], P(pos), P(vel),
                                 P(forces), P(mass), P(species), P(L), P(per), float(dt),
                                 float(ACCEL), float(r_cut), float(skin), int(precision),
                                 int(scatter), int(bool(force_rebuild)), None, P(result),
                                 P(flag)), "tb_md_step")
    return bool(flag[0]), result


def run_nve(state, params, cfg, device=0, loop="auto"):
    """NVE velocity Verlet with the trajectory resident in HBM.

    Returns the reference's run_nve record (kind, steps, dt, potential, kinetic,
    total, rebuilds, wall_clock) plus `loop` ("graph" = tb_md_run, "step" =
    tb_md_step per step) and the final positions / velocities; `state` is
    advanced in place (positions, velocities, forces, time).  Energies are
    recorded every cfg.record_every steps (default every step)."""
    import torch

    from .neighbor import build_neighbor_list
    from .xyz import write_xyz
    if loop not in ("auto", "graph", "step"):
        raise ConfigurationError(f"unknown loop {loop!r}")
    prec, scat, _ = _variant_modes(getattr(cfg, "variant", None))
    rebuild_every = int(getattr(cfg, "rebuild_every", 0) or 0)
    record_every = int(getattr(cfg, "record_every", 1) or 1)
    dump_every = int(getattr(cfg, "dump_every", 0) or 0)
    dev = torch.device("cuda", device)
    ctx = _native.default_context(device)
    ctx.set_table(params)
    ctx.set_stream(torch.cuda.current_stream(dev).cuda_stream)
    n = state.natoms
    t = lambda a, dt_: torch.as_tensor(np.ascontiguousarray(a), dtype=dt_, device=dev)  # noqa: E731
    pos = t(state.positions, torch.float64)
    vel = t(state.velocities, torch.float64)
    mass = t(state.atom_masses, torch.float64)
    species = t(state.species, torch.int32)
    forces = torch.empty((n, 3), dtype=torch.float64, device=dev)
    result = torch.zeros(8, dtype=torch.float64, device=dev)
    series = torch.zeros((cfg.steps // record_every + 1, 2), dtype=torch.float64, device=dev)
    P = _native.ptr
    t0 = _time.perf_counter()
    nl = build_neighbor_list(_DevState(pos, species, state.box), params.r_cut, cfg.skin,
                             device=device)
    rebuilds = 1
    ctx.check(ctx.lib.tb_compute_device(ctx.handle, nl._nl.handle, P(pos), P(species),
                                        float(params.r_cut), prec, scat, P(forces), None,
                                        P(result), None), "tb_compute_device")
    series[0, 0] = result[0]
    series[0, 1] = 0.5 * (mass[:, None] * vel * vel).sum() / ACCEL
    if dump_every:
        write_xyz(cfg.dump_path, _snapshot(state, pos, 0.0), append=False)
    torch.cuda.synchronize(dev)
    t_loop = _time.perf_counter()
    used = "step" if loop == "step" else "graph"
    if dump_every and (dump_every % record_every or (rebuild_every and dump_every % rebuild_every)):
        # graph segments restart their step count: dump points must keep the
        # record grid and the rebuild cadence aligned, else step per step
        if loop == "graph":
            raise ConfigurationError("loop='graph' with dumps needs dump_every to be a multiple "
                                     "of record_every and rebuild_every")
        used = "step"
    done = 0
    while done < cfg.steps:
        seg = cfg.steps - done if not dump_every else min(dump_every, cfg.steps - done)
        if used == "graph":
            nreb = ctypes.c_int64(0)
            rc = ctx.lib.tb_md_run(ctx.handle, nl._nl.handle, n, P(pos), P(vel), P(forces),
                                   P(mass), P(species), float(cfg.dt), float(ACCEL),
                                   float(params.r_cut), float(cfg.skin), rebuild_every, prec,
                                   scat, seg, record_every, P(series[done // record_every:]),
                                   P(result), ctypes.byref(nreb))
            if rc == _native.TB_OK:
                rebuilds += int(nreb.value)
            elif rc == _native.TB_ERR_UNSUPPORTED and loop == "auto":
                used = "step"
                continue
            else:
                ctx.check(rc, "tb_md_run")
        else:
            for s in range(done + 1, done + seg + 1):
                force = bool(rebuild_every) and s % rebuild_every == 0
                reb, _ = md_step(ctx, nl, pos, vel, forces, mass, species, state.box, cfg.dt,
                                 params.r_cut, cfg.skin, prec, scat, force, result)
                rebuilds += int(reb)
                if s % record_every == 0:
                    series[s // record_every].copy_(result[[0, 7]])
        done += seg
        if dump_every:
            write_xyz(cfg.dump_path, _snapshot(state, pos, done * cfg.dt), append=True)
    torch.cuda.synchronize(dev)
    t_end = _time.perf_counter()
    ctx.check(ctx.lib.tb_check_errors(ctx.handle), "run_nve")
    rec = series.cpu().numpy()
    state.positions = pos.cpu().numpy()
    state.velocities = vel.cpu().numpy()
    state.forces = forces.cpu().numpy()
    state.time = getattr(state, "time", 0.0) + cfg.steps * cfg.dt
    epot, ekin = rec[:, 0], rec[:, 1]
    return {"kind": "nve", "steps": cfg.steps, "dt": cfg.dt, "potential": epot,
            "kinetic": ekin, "total": epot + ekin, "rebuilds": rebuilds, "loop": used,
            "wall_clock": {"total": t_end - t0, "loop": t_end - t_loop},
            "positions": state.positions, "velocities": state.velocities}


def _snapshot(state, pos, time):
    class _F:
        pass
    f = _F()
    f.positions, f.species, f.symbols, f.box = pos, state.species, state.symbols, state.box
    f.time = getattr(state, "time", 0.0) + time
    return f
