"""Callers and data formats either side of the path, on
the CPU: structure generators and XYZ text against the reference's own
output (golden harness.npz), the generator-spec parser and CLI error paths,
run-configuration validation, the benchmark report schema."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_1710_00882_b200 import cli
from paper_1710_00882_b200.errors import ConfigurationError, InputError
from paper_1710_00882_b200.harness import CSV_FIELDS, BenchReport, BenchRow
from paper_1710_00882_b200.system import (RunConfig, StretchSpec, gen_diamond, gen_nanotube,
                                          read_xyz, state_from_xyz, write_xyz)
from paper_1710_00882_b200.verify import CheckResult


@pytest.fixture(scope="module")
def g():
    return load_golden("harness")


@pytest.mark.parametrize("n,cells", [(3, 1), (5, 10), (8, 4)])
def test_nanotube_matches_reference(g, n, cells):
    st = gen_nanotube(n, cells)
    assert np.array_equal(st.positions, g[f"tube_{n}_{cells}_positions"])
    assert np.array_equal(st.box.lengths, g[f"tube_{n}_{cells}_lengths"])
    assert st.box.periodic == (False, False, False)
    assert st.symbols == ("C",)


def test_diamond_matches_reference(g):
    st = gen_diamond(3)
    assert np.array_equal(st.positions, g["diamond3_positions"])
    assert np.array_equal(st.box.lengths, g["diamond3_lengths"])
    assert st.box.periodic == (True, True, True)


def test_generator_errors():
    with pytest.raises(ConfigurationError):
        gen_nanotube(2, 4)
    with pytest.raises(ConfigurationError):
        gen_nanotube(5, 0)
    with pytest.raises(ConfigurationError):
        gen_diamond(0)
    with pytest.raises(ConfigurationError):
        gen_diamond(2, lattice_constant=-1.0)


def test_xyz_text_matches_reference(g, tmp_path):
    st = gen_nanotube(5, 2)
    st.time = 12.5
    path = tmp_path / "t.xyz"
    write_xyz(path, st)
    write_xyz(path, gen_diamond(1), append=True)
    assert path.read_text() == str(g["xyz_text"])


def test_xyz_round_trip(tmp_path):
    st = gen_diamond(2)
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
    # no box comment: centred in a free box with 6 A vacuum
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


def test_genspec():
    st = cli.parse_genspec("nanotube:n=6,cells=3")
    assert st.natoms == 2 * 6 * 2 * 3
    assert cli.parse_genspec("diamond", ("2",)).natoms == 64
    assert np.array_equal(cli.parse_genspec("diamond:cells=2,lattice_constant=3.6").box.lengths,
                          [7.2, 7.2, 7.2])
    for bad in ("graphene", "nanotube:q=3", "nanotube:n"):
        with pytest.raises(ConfigurationError):
            cli.parse_genspec(bad)
    with pytest.raises(ConfigurationError):
        cli.parse_genspec("diamond", ("1", "2", "3"))


def test_cli_gen_and_error_codes(tmp_path, capsys):
    out = tmp_path / "tube.xyz"
    assert cli.main(["gen", "nanotube", "5", "2", "-o", str(out)]) == 0
    st = state_from_xyz(out)
    assert np.abs(st.positions - gen_nanotube(5, 2).positions).max() < 1e-9
    assert cli.main(["gen", "bogus"]) == 2
    assert cli.main(["run", "--structure", str(tmp_path / "missing.xyz")]) == 2
    assert cli.main(["run", "--structure", "diamond:cells=2", "--variant", "nope"]) == 2
    assert cli.main(["--help"]) == 0
    assert "error:" in capsys.readouterr().err


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
        StretchSpec(axis=3)
    with pytest.raises(ConfigurationError):
        StretchSpec(grip_fraction=0.5)


def test_bench_report_schema(g):
    assert ",".join(CSV_FIELDS) == str(g["csv_fields"])
    rows = [BenchRow("B200", "sm_100a", 32, "double", 512, 20, 1.234567891234e-3,
                     lane_util=0.78125),
            BenchRow("B200", "sm_100a", 32, "single", 512, 20, 9.87654321e-4)]
    rep = BenchReport(rows, {"repeats": 5, "median_s": {"a": 1.0e-3}, "neighbor_build_s": 0.01})
    csv = rep.render("csv").splitlines()
    assert csv[0] == ",".join(CSV_FIELDS)
    assert csv[1].split(",")[6] == "0.00123456789"
    js = json.loads(rep.render("json"))
    assert js["rows"][0]["time_s"] == 0.00123456789
    table = rep.render("table")
    assert "0.00123456789" in table and "# neighbor build" in table
    with pytest.raises(ValueError):
        rep.render("xml")


def test_check_result():
    c = CheckResult("x", True, 1e-12, 1e-10)
    assert c.margin == pytest.approx(100.0)
    d = CheckResult("y", True, 0.0, 1e-10).as_dict()
    assert d["margin"] is None and d["passed"]
    assert CheckResult("z", False, None, None).margin is None
