"""Shared fixtures.  `gpu` tests need a B200 (run with -m gpu); everything
else runs on the CPU.  The oracle (../oracle) is test infrastructure only."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False))


class Frame:
    """Duck-typed state: positions, species, box.lengths/.periodic
    (the reference's own test stub shape, helpers.py:78-97)."""

    def __init__(self, positions, lengths, periodic, species=None):
        from paper_1710_00882_b200.state import SimulationBox
        self.positions = np.ascontiguousarray(positions, dtype=np.float64)
        self.box = SimulationBox(lengths, tuple(bool(p) for p in periodic))
        n = self.positions.shape[0]
        self.species = (np.zeros(n, np.int64) if species is None
                        else np.asarray(species, dtype=np.int64))


def golden_frame(g, prefix=""):
    return Frame(g[prefix + "positions"], g[prefix + "lengths"],
                 g.get(prefix + "periodic", np.zeros(3, bool)), g[prefix + "species"])


def golden_clusters():
    from paper_1710_00882_b200.paramfile import parse_params
    g = load_golden("clusters")
    tables = {False: parse_params(str(g["table_carbon"])),
              True: parse_params(str(g["table_mixed"]))}
    out = []
    for k in range(int(g["count"])):
        p = f"c{k}_"
        mixed = bool(g[p + "mixed"])
        fr = Frame(g[p + "positions"], g[p + "lengths"], (False, False, False),
                   g[p + "species"])
        row = {key[len(p):]: g[key] for key in g if key.startswith(p)}
        out.append((fr, tables[mixed], row))
    return out


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import oracle as O
    O.lib()
    return O
