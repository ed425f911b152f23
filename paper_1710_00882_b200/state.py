"""Atoms, box and units for the B200 drivers.

Any object with `.positions` (n,3), `.species` (n,) and `.box.lengths` /
`.box.periodic` is accepted by compute() and the drivers -- including the
reference's own SimulationState (pkg/src/tersoffmd/system.py:56-122), so a
reference caller keeps its state objects.  This module only provides the
containers the package's own generators (structures.py) and drivers return,
with the reference's field names and units:

  ACCEL  (eV/A)/amu -> A/fs^2, KB_EV eV/K         system.py:18-22
  MASSES amu per element                          system.py:24
  kinetic_energy 0.5 sum m v^2 / ACCEL            system.py:129-134
  seed_velocities N(0, sqrt(kT ACCEL/m)) per component, net momentum removed,
      same generator calls as system.py:149-157 (identical draws per seed)

Positions may be numpy arrays or CUDA float64 tensors (device-resident
states: the drivers then never copy them to the host).
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigurationError

# CODATA 2018 eV and amu: (eV/A)/amu in A/fs^2
ACCEL = 1.602176634e-19 / 1.66053906660e-27 * 1e-10
KB_EV = 8.617333262e-5
MASSES = {"C": 12.011, "Si": 28.0855, "Ge": 72.63}
ELEMENT_MASSES = MASSES


class SimulationBox:
    """Orthorhombic box: edge lengths (A) and per-axis periodic flags."""

    __slots__ = ("lengths", "periodic")

    def __init__(self, lengths, periodic=(False, False, False)):
        lengths = np.asarray(lengths, dtype=np.float64).reshape(-1)
        if lengths.shape != (3,) or len(periodic) != 3:
            raise ConfigurationError("a box needs three edge lengths and three periodic flags")
        if not (lengths > 0).all():
            raise ConfigurationError(f"box edge lengths must be positive, got {lengths}")
        self.lengths = lengths
        self.periodic = tuple(bool(p) for p in periodic)

    def wrap(self, positions):
        """Periodic coordinates into [0, L) in place (numpy remainder)."""
        per = [ax for ax in range(3) if self.periodic[ax]]
        if per:
            positions[:, per] %= self.lengths[per]
        return positions

    @property
    def volume(self):
        return float(self.lengths.prod())

    def __repr__(self):
        return f"SimulationBox({self.lengths.tolist()}, {self.periodic})"


@dataclass
class SimulationState:
    """positions (n,3) A, species (n,) int, masses per species (amu),
    velocities A/fs, box; `symbols[s]` names species s."""

    positions: np.ndarray
    box: SimulationBox
    species: np.ndarray = None
    masses: np.ndarray = None
    symbols: tuple = ("Si",)
    velocities: np.ndarray = None
    forces: np.ndarray = None
    time: float = 0.0
    extra: dict = field(default_factory=dict)

    def __post_init__(self):
        self.positions = np.array(self.positions, dtype=np.float64)
        n = self.positions.shape[0]
        if self.positions.shape != (n, 3):
            raise ConfigurationError(f"positions must be (n, 3), got {self.positions.shape}")
        self.species = (np.zeros(n, np.int64) if self.species is None
                        else np.asarray(self.species, dtype=np.int64))
        if self.masses is None:
            self.masses = np.array([MASSES.get(s, MASSES["Si"]) for s in self.symbols])
        self.masses = np.asarray(self.masses, dtype=np.float64)
        if n and (self.species.min() < 0 or self.species.max() >= len(self.masses)):
            raise ConfigurationError("species index without a mass")
        self.velocities = (np.zeros((n, 3)) if self.velocities is None
                           else np.array(self.velocities, dtype=np.float64))
        self.forces = np.zeros((n, 3)) if self.forces is None else self.forces

    @property
    def natoms(self):
        return self.positions.shape[0]

    @property
    def atom_masses(self):
        return self.masses[self.species]

    def copy(self):
        return SimulationState(self.positions.copy(),
                               SimulationBox(self.box.lengths.copy(), self.box.periodic),
                               self.species.copy(), self.masses.copy(), self.symbols,
                               self.velocities.copy(), np.array(self.forces, copy=True),
                               self.time, dict(self.extra))


def kinetic_energy(state):
    """0.5 sum m v^2 in eV."""
    if state.natoms == 0:
        return 0.0
    # (same association as the reference, so host records agree bit for bit)
    return 0.5 * float((state.atom_masses * (state.velocities ** 2).sum(axis=1)).sum()) / ACCEL


def total_momentum(state):
    return (state.atom_masses[:, None] * state.velocities).sum(axis=0)


def seed_velocities(state, temperature, rng=0):
    """Maxwell-Boltzmann velocities at `temperature` K with zero net momentum
    (no rescaling to T): the same draws as the reference for the same seed."""
    gen = np.random.default_rng(rng)
    m = state.atom_masses
    width = np.sqrt(KB_EV * temperature * ACCEL / m)
    state.velocities = gen.normal(size=(state.natoms, 3)) * width[:, None]
    state.velocities -= total_momentum(state) / m.sum()
    return state
