"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE names no public dataset: every configuration is a synthetic lattice
or random packing, generated here from fixed seeds:

  1  Si diamond 4^3 cells (512), a=5.431, sigma=0.1 (seed 1001), 1000 K (2001)
  2  Si diamond 20^3 (64,000), sigma=0.1 (1002), 1000 K (2002)
  3  3C-SiC zincblende 40^3 (512,000), a=4.359, sigma=0.08 (1003), 1500 K (2003)
  4  disordered Si, 1,000,000 atoms, rho=0.05/A^3, d_min=2.0 A (seed 1004)
  5  Si diamond 128^3 (16,777,216), sigma=0.1 (1005), 1000 K (2005)

gen_diamond follows the reference generator's site order (system.py:205-226);
zincblende puts species 0 (Si) on the fcc half of that basis and species 1 (C)
on the (1/4,1/4,1/4)-shifted half.  Velocities follow seed_velocities
(system.py:149-157).
"""

import numpy as np

from .state import MASSES, SimulationBox, SimulationState, seed_velocities  # noqa: F401

_DIAMOND_BASIS = np.array([
    [0.00, 0.00, 0.00], [0.00, 0.50, 0.50],
    [0.50, 0.00, 0.50], [0.50, 0.50, 0.00],
    [0.25, 0.25, 0.25], [0.25, 0.75, 0.75],
    [0.75, 0.25, 0.75], [0.75, 0.75, 0.25],
])



def _lattice(cells, a):
    """cells: int (cubic) or (nx, ny, nz) conventional cells."""
    nc = (int(cells),) * 3 if np.isscalar(cells) else tuple(int(c) for c in cells)
    if min(nc) < 1:
        raise ValueError(f"need at least 1 cell, got {cells}")
    origins = np.stack(np.meshgrid(*[np.arange(c) for c in nc], indexing="ij"),
                       -1).reshape(-1, 3)
    frac = (origins[:, None, :] + _DIAMOND_BASIS[None, :, :]).reshape(-1, 3)
    return frac * a, np.array(nc, dtype=np.float64) * a


def gen_diamond(cells, a=5.431, symbol="Si"):
    """Periodic diamond-cubic crystal, 8 atoms per conventional cell; cells is
    an int (cubic box) or (nx, ny, nz) (slabs stacked along x for weak scaling)."""
    pos, L = _lattice(cells, a)
    box = SimulationBox(L, periodic=(True, True, True))
    return SimulationState(pos, box, species=np.zeros(len(pos), np.int64),
                           masses=np.array([MASSES[symbol]]), symbols=(symbol,))


def gen_zincblende(cells, a=4.359, symbols=("Si", "C")):
    """3C-SiC: species 0 on fcc sites, species 1 on fcc + (1/4,1/4,1/4) a."""
    pos, L = _lattice(cells, a)
    sp = np.tile(np.array([0, 0, 0, 0, 1, 1, 1, 1], np.int64), len(pos) // 8)
    box = SimulationBox(L, periodic=(True, True, True))
    return SimulationState(pos, box, species=sp,
                           masses=np.array([MASSES[s] for s in symbols]),
                           symbols=tuple(symbols))


def displace(state, sigma, seed):
    """Seeded isotropic Gaussian displacement, then wrap into the box."""
    rng = np.random.default_rng(seed)
    state.positions += rng.normal(scale=sigma, size=state.positions.shape)
    state.box.wrap(state.positions)
    return state


def gen_disordered(n, density=0.05, d_min=2.0, seed=1004, symbol="Si",
                   batch=None):
    """Uniform random points in a periodic cube, rejection-sampled so that no
    two atoms are closer than d_min (minimum image).  Candidates are drawn in
    seeded batches; a candidate is kept unless it lies within d_min of an
    accepted atom or of an earlier candidate of its own batch."""
    from scipy.spatial import cKDTree

    n = int(n)
    L = (n / density) ** (1.0 / 3.0)
    rng = np.random.default_rng(seed)
    acc = np.empty((0, 3))
    batch = batch or max(1024, n // 8)
    while acc.shape[0] < n:
        cand = rng.uniform(0.0, L, size=(batch, 3))
        keep = np.ones(batch, bool)
        if acc.shape[0]:
            tree = cKDTree(acc, boxsize=L)
            dist, _ = tree.query(cand, k=1, distance_upper_bound=d_min)
            keep &= ~(dist < d_min)
        pairs = cKDTree(cand, boxsize=L).query_pairs(d_min, output_type="ndarray")
        if pairs.size:
            keep[np.max(pairs, axis=1)] = False
        acc = np.concatenate([acc, cand[keep]])
    pos = acc[:n].copy()
    box = SimulationBox([L, L, L], periodic=(True, True, True))
    return SimulationState(pos, box, species=np.zeros(n, np.int64),
                           masses=np.array([MASSES[symbol]]), symbols=(symbol,))


# name -> (builder, parameter set, velocity temperature/seed)
def config(index, small=False):
    """Build BASELINE configuration `index` (1-5) as a SimulationState.

    small=True shrinks the cell count (same density, same seeds) for parity
    tests at oracle-friendly sizes."""
    if index == 1:
        st = displace(gen_diamond(4, 5.431), 0.1, 1001)
        return seed_velocities(st, 1000.0, 2001), "Si"
    if index == 2:
        st = displace(gen_diamond(8 if small else 20, 5.431), 0.1, 1002)
        return seed_velocities(st, 1000.0, 2002), "Si"
    if index == 3:
        st = displace(gen_zincblende(6 if small else 40, 4.359), 0.08, 1003)
        return seed_velocities(st, 1500.0, 2003), "SiC"
    if index == 4:
        st = gen_disordered(8000 if small else 1_000_000, 0.05, 2.0, 1004)
        return seed_velocities(st, 1000.0, 2004), "Si"
    if index == 5:
        st = displace(gen_diamond(10 if small else 128, 5.431), 0.1, 1005)
        return seed_velocities(st, 1000.0, 2005), "Si"
    raise ValueError(f"unknown configuration {index}")


def config5_weak(n_gpus):
    """BASELINE config 5 weak scaling: 64^3 cells (2,097,152 atoms) per GPU,
    stacked along x (the slab axis); same sigma / temperature / seeds."""
    st = displace(gen_diamond((64 * int(n_gpus), 64, 64), 5.431), 0.1, 1005)
    return seed_velocities(st, 1000.0, 2005), "Si"
