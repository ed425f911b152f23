"""State containers, XYZ frames and MD run configuration (host logic, CPU).

XYZ text written by the reference's write_xyz (golden harness.npz, produced by
tests/golden/make_golden.py from the reference itself) must survive a
read -> write round trip through this package byte for byte, so trajectory
files are interchangeable with the reference's (system.py:233-307)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1710_00882_b200 import structures
from paper_1710_00882_b200.errors import ConfigurationError, InputError
from paper_1710_00882_b200.md import RunConfig
from paper_1710_00882_b200.state import (ACCEL, SimulationBox, SimulationState, kinetic_energy,
                                         seed_velocities, total_momentum)
from paper_1710_00882_b200.xyz import read_xyz, state_from_xyz, write_xyz


def test_xyz_text_round_trips_reference_file(tmp_path):
    g = load_golden("harness")
    src = tmp_path / "ref.xyz"
    src.write_text(str(g["xyz_text"]))
    frames = read_xyz(src)
    assert len(frames) == 2
    out = tmp_path / "out.xyz"
    for k in range(len(frames)):
        st = state_from_xyz(src, frame=k)
        comment = frames[k][2]
        st.time = float(comment.split("time")[1]) if "time" in comment else 0.0
        write_xyz(out, st, append=k > 0)
    assert out.read_text() == str(g["xyz_text"])


def test_xyz_round_trip(tmp_path):
    st = structures.gen_diamond(2, 3.566, "C")
    st.positions += 0.0123
    path = tmp_path / "d.xyz"
    write_xyz(path, st)
    frames = read_xyz(path)
    assert len(frames) == 1 and len(frames[0][0]) == st.natoms
    back = state_from_xyz(path)
    assert np.abs(back.positions - st.positions).max() < 1e-10
    assert np.array_equal(back.box.lengths, st.box.lengths)
    assert back.box.periodic == st.box.periodic
    assert back.symbols == ("C",)
    path2 = tmp_path / "free.xyz"
    write_xyz(path2, st, comment="no box here")
    free = state_from_xyz(path2)
    assert free.box.periodic == (False, False, False)
    assert np.allclose(free.positions.min(axis=0), 6.0)


def test_xyz_errors(tmp_path):
    bad = tmp_path / "bad.xyz"
    bad.write_text("three\ncomment\n")
    with pytest.raises(InputError):
        read_xyz(bad)
    trunc = tmp_path / "trunc.xyz"
    trunc.write_text("2\nc\nC 0 0 0\n")
    with pytest.raises(InputError):
        read_xyz(trunc)
    empty = tmp_path / "empty.xyz"
    empty.write_text("")
    with pytest.raises(InputError):
        state_from_xyz(empty)


def test_box_and_state_validation():
    with pytest.raises(ConfigurationError):
        SimulationBox([1.0, 0.0, 1.0])
    with pytest.raises(ConfigurationError):
        SimulationBox([1.0, 1.0])
    b = SimulationBox([2.0, 3.0, 4.0], (True, False, True))
    x = np.array([[-0.5, -0.5, 4.5]])
    b.wrap(x)
    assert np.array_equal(x, [[1.5, -0.5, 0.5]])
    with pytest.raises(ConfigurationError):
        SimulationState(np.zeros((2, 3)), b, species=[0, 1], masses=[12.0])
    with pytest.raises(ConfigurationError):
        SimulationState(np.zeros((2, 2)), b)


def test_seed_velocities_and_kinetic_energy():
    st = structures.gen_diamond(6)
    seed_velocities(st, 1000.0, 7)
    assert np.abs(total_momentum(st)).max() < 1e-12
    ke = kinetic_energy(st)
    m = st.atom_masses
    assert ke == pytest.approx(0.5 * float((m[:, None] * st.velocities ** 2).sum()) / ACCEL,
                               rel=1e-14)
    # equipartition within sampling noise: 3/2 N k T
    assert ke / (1.5 * st.natoms * 8.617333262e-5 * 1000.0) == pytest.approx(1.0, abs=0.1)
    again = seed_velocities(structures.gen_diamond(6), 1000.0, 7)
    assert np.array_equal(again.velocities, st.velocities)


def test_run_config_validation():
    with pytest.raises(ConfigurationError):
        RunConfig(dt=0.0)
    with pytest.raises(ConfigurationError):
        RunConfig(steps=-1)
    with pytest.raises(ConfigurationError):
        RunConfig(dump_every=5)
    with pytest.raises(ConfigurationError):
        RunConfig(dump_every=-1, dump_path="x")
    with pytest.raises(ConfigurationError):
        RunConfig(record_every=0)


def test_generators_are_seeded():
    a, _ = structures.config(2, small=True)
    b, _ = structures.config(2, small=True)
    assert np.array_equal(a.positions, b.positions)
    assert np.array_equal(a.velocities, b.velocities)
    c, tname = structures.config(3, small=True)
    assert tname == "SiC" and set(np.unique(c.species)) == {0, 1}
    assert c.natoms == 8 * 6 ** 3
