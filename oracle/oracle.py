"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

The oracle is a C restatement (tersoff_oracle.c) of the reference
`tersoffmd` hot path: build_neighbor_list / pack_adjacency / needs_rebuild
(reference pkg/src/tersoffmd/neighbor.py:194-229, :330-360) and the ScalarOpt
kernel with its ordered merge (kernels.py:250-315, :119-151).  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import it; the
product package never does.

Parity of this restatement is pinned against vectors produced by running the
reference itself (tests/golden/make_golden.py -> tests/golden/*.npz) and
against the reference test-suite's frozen goldens (dimer energy/force).
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle_tersoff.so")
_lib = None

PRECISIONS = {"double": 0, "single": 1}


class OracleError(RuntimeError):
    pass


def build():
    """Compile the oracle library in place (make)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        d = ctypes.c_double
        ci = ctypes.c_int
        L.or_build_neighbors.argtypes = [i64, P, P, P, d, d, P, P, ci]
        L.or_build_neighbors.restype = ci
        L.or_needs_rebuild.argtypes = [i64, P, P, P, P, d]
        L.or_needs_rebuild.restype = ci
        L.or_pack_adjacency.argtypes = [i64, P, P, P, P, P, d, P, P, P, P, P, P, P]
        L.or_pack_adjacency.restype = ci
        L.or_compute_packed.argtypes = [i64, P, P, P, P, P, P, P, ci, P, P, ci, ci,
                                        P, P, P, P, P]
        L.or_compute_packed.restype = ci
        L.or_half_kick.argtypes = [i64, P, P, P, d]
        L.or_half_kick.restype = None
        L.or_drift_wrap.argtypes = [i64, P, P, d, P, P]
        L.or_drift_wrap.restype = None
        L.or_np_remainder.argtypes = [d, d]
        L.or_np_remainder.restype = d
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _box(lengths, periodic):
    L = np.ascontiguousarray(np.asarray(lengths, dtype=np.float64).reshape(3))
    per = np.ascontiguousarray(np.asarray([bool(x) for x in periodic], dtype=np.int32))
    return L, per


def flatten_table(table):
    """(S, pair_mat[S*S,8], trip_mat[S^3,8], r_cut) -- restates
    ParamTable._build_views (reference potential.py:127-155) and
    r_cut = max(R + D) (potential.py:106)."""
    s = table.nspecies
    pair = np.empty((s * s, 8))
    trip = np.empty((s * s * s, 8))
    rc = 0.0
    for ti in range(s):
        for tj in range(s):
            p = table.entry(ti, tj, tj)
            pair[ti * s + tj] = (p.R, p.D, p.A, p.lam1, p.B, p.lam2, p.beta, p.eta)
            for tk in range(s):
                q = table.entry(ti, tj, tk)
                trip[(ti * s + tj) * s + tk] = (q.R, q.D, q.gamma, q.c, q.d, q.h,
                                                q.lam3, float(q.m))
                rc = max(rc, q.R + q.D)
    return s, pair, trip, rc


def build_neighbor_list(positions, lengths, periodic, r_cut, skin=0.3, threads=0):
    """Full CSR (offsets, neighbors) at r_cut + skin, rows ascending."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    n = pos.shape[0]
    L, per = _box(lengths, periodic)
    offsets = np.zeros(n + 1, dtype=np.int64)
    rc = lib().or_build_neighbors(n, _p(pos), _p(L), _p(per), float(r_cut), float(skin),
                                  _p(offsets), None, threads)
    if rc:
        raise OracleError(f"or_build_neighbors failed ({rc})")
    nbr = np.zeros(max(int(offsets[-1]), 1), dtype=np.int64)
    rc = lib().or_build_neighbors(n, _p(pos), _p(L), _p(per), float(r_cut), float(skin),
                                  _p(offsets), _p(nbr), threads)
    if rc:
        raise OracleError(f"or_build_neighbors failed ({rc})")
    return offsets, nbr[: int(offsets[-1])]


def needs_rebuild(positions, reference_positions, lengths, periodic, skin):
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    ref = np.ascontiguousarray(reference_positions, dtype=np.float64)
    L, per = _box(lengths, periodic)
    return bool(lib().or_needs_rebuild(pos.shape[0], _p(pos), _p(ref), _p(L), _p(per),
                                       float(skin)))


def pack_adjacency(positions, lengths, periodic, offsets, neighbors, r_cut):
    """Packed adjacency dict(offsets, i, j, dx, dy, dz, r) at current positions."""
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    n = pos.shape[0]
    L, per = _box(lengths, periodic)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    nb = np.ascontiguousarray(neighbors, dtype=np.int64)
    if nb.size == 0:
        nb = np.zeros(1, dtype=np.int64)
    poff = np.zeros(n + 1, dtype=np.int64)
    bad = np.zeros(2, dtype=np.int64)
    rc = lib().or_pack_adjacency(n, _p(pos), _p(L), _p(per), _p(off), _p(nb), float(r_cut),
                                 _p(poff), None, None, None, None, None, _p(bad))
    m = int(poff[-1])
    j = np.zeros(max(m, 1), dtype=np.int64)
    dx, dy, dz, r = (np.zeros(max(m, 1)) for _ in range(4))
    rc = lib().or_pack_adjacency(n, _p(pos), _p(L), _p(per), _p(off), _p(nb), float(r_cut),
                                 _p(poff), _p(j), _p(dx), _p(dy), _p(dz), _p(r), _p(bad))
    if rc == 2:
        raise OracleError(f"atoms {bad[0]} and {bad[1]} are coincident")
    i = np.repeat(np.arange(n, dtype=np.int64), np.diff(poff))
    return dict(offsets=poff, i=i, j=j[:m], dx=dx[:m], dy=dy[:m], dz=dz[:m], r=r[:m])


def compute(positions, species, lengths, periodic, offsets, neighbors, table,
            precision="double", threads=1):
    """ScalarOpt energy/forces (+ derived virial) on the oracle.

    Returns dict(forces (n,3), energy, per_atom (n,), virial (6,)
    [xx,yy,zz,xy,xz,yz], zeta_visits)."""
    S, pair, trip, r_cut = flatten_table(table)
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    n = pos.shape[0]
    adj = pack_adjacency(pos, lengths, periodic, offsets, neighbors, r_cut)
    return compute_packed(adj, species, S, pair, trip, precision, threads, n)


def compute_packed(adj, species, S, pair, trip, precision="double", threads=1, n=None):
    if n is None:
        n = adj["offsets"].shape[0] - 1
    sp = np.ascontiguousarray(species, dtype=np.int64)
    forces = np.zeros((n, 3))
    per_atom = np.zeros(n)
    virial = np.zeros(6)
    energy = np.zeros(1)
    stats = np.zeros(1, dtype=np.int64)
    pad = lambda a, dt: np.ascontiguousarray(a if a.size else np.zeros(1, dt), dtype=dt)
    j = pad(adj["j"], np.int64)
    arrs = [pad(adj[k], np.float64) for k in ("dx", "dy", "dz", "r")]
    pair = np.ascontiguousarray(pair, dtype=np.float64)
    trip = np.ascontiguousarray(trip, dtype=np.float64)
    rc = lib().or_compute_packed(n, _p(adj["offsets"]), _p(j), *[_p(a) for a in arrs],
                                 _p(sp), int(S), _p(pair), _p(trip),
                                 PRECISIONS[precision], int(threads), _p(forces),
                                 _p(energy), _p(per_atom), _p(virial), _p(stats))
    if rc:
        raise OracleError(f"or_compute_packed failed ({rc})")
    return dict(forces=forces, energy=float(energy[0]), per_atom=per_atom, virial=virial,
                zeta_visits=int(stats[0]))


def np_remainder(a, b):
    return lib().or_np_remainder(float(a), float(b))


ACCEL = 1.602176634e-19 / 1.66053906660e-27 * 1e-10  # system.py:18-21


def run_nve(positions, velocities, species, masses, lengths, periodic, table, dt, steps,
            skin=0.3, precision="double", threads=1, rebuild_every=0):
    """NVE velocity Verlet (system.py:355-380, :427-460) on the oracle.

    The neighbour list is rebuilt on the skin/2 trigger (neighbor.py:220-229)
    and, when rebuild_every > 0, additionally every `rebuild_every` steps.
    Returns dict(potential, kinetic, total, rebuilds, positions, velocities)."""
    S, pair, trip, r_cut = flatten_table(table)
    pos = np.array(positions, dtype=np.float64)
    vel = np.array(velocities, dtype=np.float64)
    sp = np.asarray(species, dtype=np.int64)
    am = np.ascontiguousarray(np.asarray(masses, dtype=np.float64)[sp])
    L, per = _box(lengths, periodic)
    n = pos.shape[0]

    def forces(nl_state, step):
        off, nb, ref = nl_state[:3]
        if off is None or needs_rebuild(pos, ref, L, per, skin) or (
                rebuild_every and step % rebuild_every == 0):
            off, nb = build_neighbor_list(pos, L, per, r_cut, skin)
            ref = pos.copy()
            nl_state[3] += 1
        nl_state[0], nl_state[1], nl_state[2] = off, nb, ref
        adj = pack_adjacency(pos, L, per, off, nb, r_cut)
        return compute_packed(adj, sp, S, pair, trip, precision, threads, n)

    def kinetic():
        return 0.5 * float((am * (vel ** 2).sum(axis=1)).sum()) / ACCEL

    nl_state = [None, None, None, 0]
    res = forces(nl_state, 0)
    epot, ekin = [res["energy"]], [kinetic()]
    half = 0.5 * dt * ACCEL
    for step in range(1, steps + 1):
        lib().or_half_kick(n, _p(vel), _p(res["forces"]), _p(am), half)
        lib().or_drift_wrap(n, _p(pos), _p(vel), float(dt), _p(L), _p(per))
        res = forces(nl_state, step)
        lib().or_half_kick(n, _p(vel), _p(res["forces"]), _p(am), half)
        epot.append(res["energy"])
        ekin.append(kinetic())
    epot, ekin = np.array(epot), np.array(ekin)
    return dict(potential=epot, kinetic=ekin, total=epot + ekin, rebuilds=nl_state[3],
                positions=pos, velocities=vel)
