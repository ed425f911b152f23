"""Tersoff parameter entries and the flattened kernel tables.

Host-side mirror of reference pkg/src/tersoffmd/potential.py:40-160.  The
potential *math* lives only in the CUDA kernels (csrc/tersoff_math.cuh);
this module validates entries and flattens a complete table into the two
matrices the C ABI uploads to constant memory, in the reference column order:

    pair_matrix  (S*S, 8)   [R, D, A, lam1, B, lam2, beta, eta]   entry (i,j,j)
    trip_matrix  (S^3, 8)   [R, D, gamma, c, d, h, lam3, m]       entry (i,j,k)

(potential.py:37-38, :127-155).  r_cut = max over entries of R + D
(potential.py:82-84, :106).
"""

from dataclasses import dataclass

import numpy as np

PAIR_FIELDS = ("R", "D", "A", "lam1", "B", "lam2", "beta", "eta")
TRIP_FIELDS = ("R", "D", "gamma", "c", "d", "h", "lam3", "m")
ZETA_TINY = 1e-30  # potential.py:34


@dataclass(frozen=True)
class TersoffParams:
    """One entry (element triple); field semantics as potential.py:40-84."""

    m: int
    gamma: float
    lam3: float
    c: float
    d: float
    h: float
    eta: float
    beta: float
    lam2: float
    B: float
    R: float
    D: float
    lam1: float
    A: float

    def __post_init__(self):
        # validation rules and messages follow potential.py:66-80
        if self.m not in (1, 3):
            raise ValueError(f"m must be 1 or 3, got {self.m}")
        checks = ((self.A > 0, "A must be positive"),
                  (self.B > 0, "B must be positive"),
                  (self.D > 0, "D must be positive"),
                  (self.R > self.D, "R must exceed D"),
                  (self.eta > 0, "eta must be positive"),
                  (self.d != 0, "d must be nonzero"),
                  (self.gamma > 0, "gamma must be positive"))
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def r_cut(self):
        return self.R + self.D


class ParamTable:
    """One TersoffParams per ordered species triple (potential.py:87-160)."""

    def __init__(self, species, entries):
        self.species = tuple(species)
        s = len(self.species)
        if s == 0:
            raise ValueError("no species")
        missing = [(a, b, c) for a in range(s) for b in range(s)
                   for c in range(s) if (a, b, c) not in entries]
        if missing:
            names = ", ".join("-".join(self.species[x] for x in t)
                              for t in missing[:4])
            raise ValueError(f"incomplete table, missing triples: {names}")
        self.entries = dict(entries)
        self.r_cut = max(p.r_cut for p in self.entries.values())
        self._views = {}

    @property
    def nspecies(self):
        return len(self.species)

    def entry(self, ti, tj, tk):
        return self.entries[(ti, tj, tk)]

    def pair_entry(self, ti, tj):
        return self.entries[(ti, tj, tj)]

    def species_index(self, name):
        if name not in self.species:
            raise KeyError(f"species {name!r} not in parameter table")
        return self.species.index(name)

    def views(self, precision="double"):
        """pair_matrix / trip_matrix as float64 (the C ABI casts to fp32 for
        the mixed mode itself, like kernels.py:154-165 casts per precision)."""
        if precision not in ("double", "single"):
            raise ValueError(f"unknown precision {precision!r}")
        if precision not in self._views:
            s = self.nspecies
            pair = np.empty((s * s, 8))
            trip = np.empty((s ** 3, 8))
            for ti in range(s):
                for tj in range(s):
                    p = self.pair_entry(ti, tj)
                    pair[ti * s + tj] = [getattr(p, f) for f in PAIR_FIELDS]
                    for tk in range(s):
                        q = self.entry(ti, tj, tk)
                        trip[(ti * s + tj) * s + tk] = [
                            float(getattr(q, f)) for f in TRIP_FIELDS]
            dt = np.float64 if precision == "double" else np.float32
            self._views[precision] = {
                "pair_matrix": np.ascontiguousarray(pair, dtype=dt),
                "trip_matrix": np.ascontiguousarray(trip, dtype=dt),
            }
        return self._views[precision]
