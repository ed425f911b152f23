"""The reference's callers running on the B200 kernel: the stretch driver
against the reference's own run (golden harness.npz), XYZ dumps from the NVE
driver, the verify suites, the benchmark harness and the CLI subcommands."""

import json

import numpy as np
import pytest

from conftest import load_golden
from paper_1710_00882_b200 import cli
from paper_1710_00882_b200.harness import run_benchmark
from paper_1710_00882_b200.kernels import make_variant
from paper_1710_00882_b200.paramfile import builtin_params
from paper_1710_00882_b200.system import (RunConfig, StretchSpec, gen_diamond, gen_nanotube,
                                          read_xyz, run_nve, run_stretch, seed_velocities)
from paper_1710_00882_b200.verify import run_verification

pytestmark = pytest.mark.gpu


def test_run_stretch_matches_reference():
    g = load_golden("harness")
    st = gen_nanotube(5, 4)
    st.positions[:] = g["stretch_positions0"]
    st.velocities = g["stretch_velocities0"].copy()
    cfg = RunConfig(dt=0.5, steps=40, variant=make_variant("B200"), skin=0.3,
                    stretch=StretchSpec(axis=2, speed=0.02))
    rec = run_stretch(st, builtin_params("C"), cfg)
    scale = abs(g["stretch_total"][0])
    for k in ("potential", "kinetic", "total"):
        assert np.max(np.abs(rec[k] - g[f"stretch_{k}"])) <= 1e-9 * scale, k
    assert np.max(np.abs(rec["strain"] - g["stretch_strain"])) <= 1e-10
    assert tuple(rec["grip_atoms"]) == tuple(g["stretch_grip_atoms"])
    assert rec["rebuilds"] == int(g["stretch_rebuilds"])
    assert np.abs(st.positions - g["stretch_final_positions"]).max() <= 1e-8


def test_run_nve_dumps_frames(tmp_path):
    st = gen_diamond(2)
    seed_velocities(st, 300.0, 3)
    path = tmp_path / "traj.xyz"
    cfg = RunConfig(dt=0.5, steps=20, dump_every=5, dump_path=str(path))
    run_nve(st, builtin_params("C"), cfg)
    frames = read_xyz(path)
    assert len(frames) == 5
    assert np.abs(frames[-1][1] - st.positions).max() < 1e-9
    assert "time 10" in frames[-1][2]


def test_verify_suite_passes_and_zero_scale_fails():
    st = gen_nanotube(5, 3)
    rep = run_verification(st, builtin_params("C"), conservation_steps=60)
    assert rep["passed"], [c for c in rep["checks"] if not c["passed"]]
    names = [c["name"] for c in rep["checks"]]
    assert names == ["gradient_fd", "cross_variant_energy", "cross_variant_forces",
                     "gather_bitwise_repeat", "atomic_energy_spread", "nve_energy_drift",
                     "nve_force_sum", "nve_momentum"]
    zero = run_verification(st, builtin_params("C"), tol_scale=0.0, conservation_steps=20)
    assert not zero["passed"]


def test_harness_run_benchmark():
    st = gen_diamond(4)
    variants = [make_variant("B200"), make_variant("B200", precision="single"),
                make_variant("B200", scatter="gather")]
    rep = run_benchmark(st, builtin_params("C"), variants, steps=5, warmup=1, repeats=2)
    assert [r.precision for r in rep.rows] == ["double", "single", "double"]
    for r in rep.rows:
        assert r.backend == "sm_100a" and r.width == 32 and r.time_s > 0
        assert 0.0 < r.lane_util <= 1.0
    e = list(rep.meta["energy"].values())
    assert abs(e[0] - e[2]) <= 1e-10 * abs(e[0])


def test_cli_run_bench_verify(capsys, tmp_path):
    assert cli.main(["run", "--structure", "diamond:cells=2", "--steps", "10",
                     "--temperature", "300", "--dt", "0.5"]) == 0
    host = json.loads(capsys.readouterr().out)
    assert host["steps"] == 10 and host["variant"].startswith("B200")
    assert cli.main(["run", "--structure", "diamond:cells=2", "--steps", "10",
                     "--temperature", "300", "--dt", "0.5", "--device-loop"]) == 0
    dev = json.loads(capsys.readouterr().out)
    assert abs(dev["final"]["total"] - host["final"]["total"]) <= 1e-9 * abs(host["initial"]["total"])
    assert cli.main(["run", "--structure", "nanotube:n=5,cells=3", "--steps", "10",
                     "--pull-speed", "0.02"]) == 0
    assert "strain" in json.loads(capsys.readouterr().out)["series"]
    assert cli.main(["bench", "--structure", "diamond:cells=3", "--steps", "3",
                     "--repeats", "2", "--format", "csv", "--variant", "b200,scalar"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0].startswith("variant,backend,width") and len(lines) == 3
    assert cli.main(["verify", "--structure", "nanotube:n=5,cells=3", "--steps", "40",
                     "--format", "table"]) == 0
    assert "PASS  overall" in capsys.readouterr().out
    assert cli.main(["verify", "--structure", "nanotube:n=5,cells=3", "--steps", "10",
                     "--tol-scale", "0"]) == 1
