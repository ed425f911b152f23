"""Pin the CPU oracle (oracle/tersoff_oracle.c) to the reference.

Every vector here was produced by running the reference implementation
(tests/golden/make_golden.py).  The fp64 oracle must reproduce the
reference ScalarOpt BIT FOR BIT (same expression trees, same libm, no FMA);
the neighbour lists must be identical; the mixed-precision mode is compared
with the reference's own "single" mode within the fp32 tolerance.
"""

import numpy as np
import pytest

from conftest import golden_clusters, load_golden
from paper_1710_00882_b200.paramfile import parse_params

SYSTEMS = ["dimer", "si512", "sic216", "disordered"]


def _run(O, g, precision="double"):
    t = parse_params(str(g["table"]))
    off, nb = O.build_neighbor_list(g["positions"], g["lengths"], g["periodic"], t.r_cut, 0.3)
    r = O.compute(g["positions"], g["species"], g["lengths"], g["periodic"], off, nb, t,
                  precision=precision)
    return off, nb, r


@pytest.mark.parametrize("name", SYSTEMS)
def test_oracle_neighbor_list_identical_to_reference(oracle_mod, name):
    g = load_golden(name)
    off, nb, _ = _run(oracle_mod, g)
    assert np.array_equal(off, g["offsets"])
    assert np.array_equal(nb, g["neighbors"])


@pytest.mark.parametrize("name", SYSTEMS)
def test_oracle_fp64_bit_identical_to_reference_scalar_opt(oracle_mod, name):
    g = load_golden(name)
    _, _, r = _run(oracle_mod, g)
    assert r["forces"].tobytes() == g["forces"].tobytes()
    assert np.float64(r["energy"]).tobytes() == np.float64(g["energy"]).tobytes()
    assert r["per_atom"].tobytes() == g["per_atom"].tobytes()
    assert r["zeta_visits"] == int(g["zeta_visits"])


@pytest.mark.parametrize("name", SYSTEMS)
def test_oracle_single_close_to_reference_single(oracle_mod, name):
    # numpy's float32 transcendentals are not glibc's: agree to fp32 noise
    g = load_golden(name)
    _, _, r = _run(oracle_mod, g, "single")
    fscale = max(1.0, np.abs(g["forces"]).max())
    assert abs(r["energy"] - float(g["energy_single"])) <= 1e-5 * abs(float(g["energy_single"]))
    assert np.abs(r["forces"] - g["forces_single"]).max() <= 1e-5 * fscale


def test_oracle_dimer_matches_frozen_50_digit_goldens(oracle_mod):
    # reference test_kernels.py:21-22, test_oracle.py:13-14
    g = load_golden("dimer")
    _, _, r = _run(oracle_mod, g)
    assert r["energy"] == pytest.approx(float(g["frozen_energy"]), rel=5e-14)
    assert r["forces"][0, 0] == pytest.approx(float(g["frozen_f0x"]), rel=5e-13)
    assert r["forces"][0, 0] == -r["forces"][1, 0]


def test_oracle_clusters_match_reference_and_longdouble(oracle_mod):
    for fr, table, row in golden_clusters():
        off, nb = oracle_mod.build_neighbor_list(fr.positions, fr.box.lengths, fr.box.periodic,
                                                 table.r_cut, 0.3)
        assert np.array_equal(off, row["offsets"]) and np.array_equal(nb, row["neighbors"])
        r = oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic, off,
                               nb, table)
        assert r["forces"].tobytes() == row["forces"].tobytes()
        assert r["energy"] == float(row["energy"])
        assert r["zeta_visits"] == int(row["zeta_visits"])
        e_ld = float(row["energy_ld"])
        if np.isfinite(e_ld):  # reference longdouble brute force (tests/oracle.py)
            assert r["energy"] == pytest.approx(e_ld, rel=1e-12)


def test_oracle_virial_matches_strain_finite_difference(oracle_mod):
    # virial diagonal W_aa = -L_a dE/dL_a of the REFERENCE energy (golden)
    g = load_golden("si512")
    _, _, r = _run(oracle_mod, g)
    fd = g["virial_fd_diag"]
    assert np.allclose(r["virial"][:3], fd, rtol=1e-7, atol=1e-6)


def test_oracle_virial_free_cluster_is_sum_x_f(oracle_mod):
    # for a free cluster W_ab = sum_i x_ia F_ib exactly (translation invariant)
    for fr, table, row in golden_clusters()[:8]:
        off, nb = oracle_mod.build_neighbor_list(fr.positions, fr.box.lengths, fr.box.periodic,
                                                 table.r_cut, 0.3)
        r = oracle_mod.compute(fr.positions, fr.species, fr.box.lengths, fr.box.periodic, off,
                               nb, table)
        x, f = fr.positions, r["forces"]
        w = [(x[:, 0] * f[:, 0]).sum(), (x[:, 1] * f[:, 1]).sum(), (x[:, 2] * f[:, 2]).sum(),
             (x[:, 0] * f[:, 1]).sum(), (x[:, 0] * f[:, 2]).sum(), (x[:, 1] * f[:, 2]).sum()]
        scale = max(1.0, np.abs(w).max())
        assert np.abs(r["virial"] - np.array(w)).max() <= 1e-10 * scale


def test_oracle_nve_matches_reference_run(oracle_mod):
    g = load_golden("si512")
    t = parse_params(str(g["table"]))
    res = oracle_mod.run_nve(g["positions"], g["velocities"], g["species"], g["masses"],
                             g["lengths"], g["periodic"], t, dt=1.0, steps=100, skin=0.3)
    assert res["rebuilds"] == int(g["nve_rebuilds"]) + 0  # same trigger sequence
    assert np.allclose(res["total"], g["nve_total"], rtol=0, atol=1e-9 * abs(g["nve_total"][0]))
    assert np.abs(res["positions"] - g["nve_final_positions"]).max() < 1e-9


@pytest.mark.parametrize("frame", [0, 1, 2])
def test_oracle_neighbor_edge_frames(oracle_mod, frame):
    g = load_golden("nl_frames")
    p = f"f{frame}_"
    off, nb = oracle_mod.build_neighbor_list(g[p + "positions"], (9.0, 9.0, 9.0),
                                             g[p + "periodic"], 2.1, 0.3)
    assert np.array_equal(off, g[p + "offsets"])
    assert np.array_equal(nb, g[p + "neighbors"])


def test_oracle_threads_deterministic(oracle_mod):
    g = load_golden("disordered")
    t = parse_params(str(g["table"]))
    off, nb = g["offsets"], g["neighbors"]
    a = oracle_mod.compute(g["positions"], g["species"], g["lengths"], g["periodic"], off, nb, t,
                           threads=4)
    b = oracle_mod.compute(g["positions"], g["species"], g["lengths"], g["periodic"], off, nb, t,
                           threads=4)
    assert a["forces"].tobytes() == b["forces"].tobytes()
    assert np.abs(a["forces"] - g["forces"]).max() < 1e-12
