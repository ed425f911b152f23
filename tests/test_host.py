"""Host-side logic (no GPU): parameter files, tables, generators, and the C
ABI library surface (loads, exports every symbol include/tersoff_b200.h
declares, signatures bound) -- no compute calls."""

import ctypes
import os
import sys
import re

import numpy as np
import pytest

import paper_1710_00882_b200 as B
from conftest import load_golden
from paper_1710_00882_b200 import _native, structures
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
from paper_1710_00882_b200.paramfile import (ParamFileError, builtin_params, parse_params,
                                             serialize_params)


def header_symbols():
    text = open(_native.HEADER_PATH).read()
    return re.findall(r"^(?:int|void|const char \*)\s*\*?(tb_\w+)\(", text, re.M)


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.SIGNATURES)
    assert "sm_100a" in _native.version()


def test_library_built_for_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_builtin_tables():
    c = builtin_params("C")
    assert c.species == ("C",) and c.r_cut == pytest.approx(2.1)
    si = builtin_params("Si")
    p = si.entry(0, 0, 0)
    assert (p.A, p.B, p.lam1, p.lam2, p.lam3, p.beta, p.eta) == (
        1830.8, 471.18, 2.4799, 1.7322, 0.0, 1.1e-6, 0.78734)
    assert (p.c, p.d, p.h, p.R, p.D) == (100390.0, 16.217, -0.59825, 2.85, 0.15)
    assert si.r_cut == pytest.approx(3.0)
    sic = builtin_params("SiC")
    assert sic.species == ("Si", "C") and sic.r_cut == pytest.approx(3.0)
    # Si-C pair: chi * sqrt(B_Si B_C); cutoff from the geometric mixing
    pc = sic.pair_entry(0, 1)
    assert pc.B == pytest.approx(0.9776 * np.sqrt(471.18 * 346.74))
    assert pc.R == pytest.approx(2.357, abs=1e-3)


def test_views_column_order_matches_reference():
    # ParamTable.views layout (potential.py:127-155)
    g = load_golden("clusters")
    t = parse_params(str(g["table_mixed"]))
    v = t.views("double")
    assert v["pair_matrix"].shape == (4, 8) and v["trip_matrix"].shape == (8, 8)
    p = t.pair_entry(1, 0)
    assert list(v["pair_matrix"][1 * 2 + 0]) == [p.R, p.D, p.A, p.lam1, p.B, p.lam2, p.beta,
                                                 p.eta]
    q = t.entry(0, 1, 1)
    assert list(v["trip_matrix"][(0 * 2 + 1) * 2 + 1]) == [q.R, q.D, q.gamma, q.c, q.d, q.h,
                                                           q.lam3, float(q.m)]
    assert v["pair_matrix"].dtype == np.float64
    assert t.views("single")["trip_matrix"].dtype == np.float32


def test_param_round_trip_and_errors():
    t = builtin_params("SiC")
    t2 = parse_params(serialize_params(t))
    assert t2.entries == t.entries and t2.species == t.species
    with pytest.raises(ParamFileError, match=r"<string>:1: expected 17 tokens"):
        parse_params("C C C 1 2 3")
    with pytest.raises(ParamFileError, match=r":2: bad numeric token"):
        parse_params("# c\nC C C 3 1 0 x 4 -0.5 0.7 1e-7 2.2 346 1.95 0.15 3.4 1393\n")
    with pytest.raises(ParamFileError, match="m must be integral"):
        parse_params("C C C 2.5 1 0 1 4 -0.5 0.7 1e-7 2.2 346 1.95 0.15 3.4 1393\n")
    with pytest.raises(ParamFileError, match="m must be 1 or 3"):
        parse_params("C C C 2 1 0 1 4 -0.5 0.7 1e-7 2.2 346 1.95 0.15 3.4 1393\n")
    line = "C C C 3 1 0 1 4 -0.5 0.7 1e-7 2.2 346 1.95 0.15 3.4 1393\n"
    with pytest.raises(ParamFileError, match="duplicate entry"):
        parse_params(line + line)
    with pytest.raises(ParamFileError, match="incomplete table"):
        parse_params("C X C 3 1 0 1 4 -0.5 0.7 1e-7 2.2 346 1.95 0.15 3.4 1393\n")
    with pytest.raises(ParamFileError, match="no parameter entries"):
        parse_params("# nothing\n")


def test_variant_selection():
    v = B.make_variant("VecI", "native", precision="single")
    assert v.precision == "single" and v.tag == "VecI"
    with pytest.raises(B.ConfigurationError, match="kernel tag"):
        B.make_variant("Fastest")
    with pytest.raises(B.ConfigurationError, match="scatter"):
        B.make_variant("B200", scatter="magic")


def test_reference_variant_objects_resolve():
    # the reference's KernelVariant(tag, backend) (kernels.py:46-77), duck-typed
    from paper_1710_00882_b200.kernels import resolve_variant

    class Backend:
        name, width, precision, strict = "native", 8, "single", False

    class RefVariant:
        tag, backend, precision = "VecI", Backend(), "single"

    v = resolve_variant(RefVariant())
    assert (v.tag, v.precision, v.scatter) == ("VecI", "single", "atomic")
    kv = B.KernelVariant("ScalarOpt", Backend())  # positional (tag, backend) like the reference
    assert kv.precision == "single" and kv.backend.width == 8
    assert B.make_variant("Reference", Backend()).precision == "single"
    assert resolve_variant(None).tag == "B200"


def test_stats_contract():
    # pkg/tests/test_kernels.py:218-249: Reference walks k twice, scalar tags
    # have no lanes (lane_utilization None) and no gathers
    from paper_1710_00882_b200.kernels import ForceEnergyResult, _stats
    counts = [10, 4, 4, 6, 1, 2]
    ref = _stats("Reference", counts, 3, 70)
    opt = _stats("ScalarOpt", counts, 3, 70)
    vec = _stats("VecI", counts, 3, 70)
    assert ref["zeta_visits"] == 20 and opt["zeta_visits"] == 10 == vec["zeta_visits"]
    for s in (ref, opt):
        assert s["lane_total"] == 0 and s["gathers"] == 0
        assert ForceEnergyResult(None, 0.0, None, s).lane_utilization is None
    assert vec["lane_total"] == 96 and vec["lane_active"] == 70 == vec["gathers"]
    assert ForceEnergyResult(None, 0.0, None, vec).lane_utilization == pytest.approx(70 / 96)


def _reference_package():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "tersoffmd")):
        pytest.skip("reference not installed in baseline/_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import tersoffmd
    return tersoffmd


def test_integration_install_registers_variant():
    tersoffmd = _reference_package()
    from paper_1710_00882_b200 import integration
    import tersoffmd.cli
    import tersoffmd.kernels as K
    import tersoffmd.system as S
    orig = K.compute
    integration.install(tersoffmd)
    try:
        integration.install(tersoffmd)  # idempotent
        assert K.KERNEL_TAGS.count("B200") == 1
        v = K.make_variant("B200", precision="single")
        assert v.tag == "B200" and v.precision == "single"
        assert S.compute is K.compute and K.compute._b200_orig is orig
        assert tersoffmd.cli._VARIANT_NAMES["b200"] == "B200"
    finally:
        integration.uninstall(tersoffmd)
    assert K.compute is orig and S.compute is orig and "B200" not in K.KERNEL_TAGS
    with pytest.raises(tersoffmd.errors.ConfigurationError):
        K.make_variant("B200")


def test_generators_deterministic_and_sized():
    st, name = structures.config(1)
    assert st.natoms == 512 and name == "Si"
    assert np.allclose(st.box.lengths, 4 * 5.431)
    st2, _ = structures.config(1)
    assert np.array_equal(st.positions, st2.positions)
    assert np.array_equal(st.velocities, st2.velocities)
    p = (st.atom_masses[:, None] * st.velocities).sum(0)
    assert np.abs(p).max() < 1e-10
    sic = structures.gen_zincblende(2, 4.359)
    assert sic.natoms == 64 and (sic.species == 1).sum() == 32
    dis = structures.gen_disordered(500, 0.05, 2.0, 7)
    from scipy.spatial import cKDTree
    pairs = cKDTree(dis.positions, boxsize=dis.box.lengths[0]).query_pairs(2.0)
    assert dis.natoms == 500 and not pairs


def test_unbuilt_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setattr(_native, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_native.NativeUnavailable):
        _native.load_library()


def test_option_and_status_codes_match_the_header():
    """The Python mirror of tb_set_option's options, the precision / scatter
    selectors and the status codes are the header's #defines."""
    import re
    from paper_1710_00882_b200 import _native
    text = open(os.path.join(ROOT, "include", "tersoff_b200.h")).read()
    defs = {m.group(1): int(m.group(2))
            for m in re.finditer(r"^#define\s+(TB_[A-Z0-9_]+)\s+(-?\d+)\b", text, re.M)}
    opts = {k: v for k, v in defs.items() if k.startswith("TB_OPT_")}
    assert len(opts) >= 7 and len(set(opts.values())) == len(opts)
    for name, value in opts.items():
        assert getattr(_native, name[3:]) == value, name
    assert _native.TB_ERR_UNSUPPORTED == defs["TB_ERR_UNSUPPORTED"]
    assert _native.NSTATS == defs["TB_NSTATS"]
    assert _native.PRECISION == {"double": defs["TB_PREC_DOUBLE"], "single": defs["TB_PREC_MIXED"],
                                 "mixed": defs["TB_PREC_MIXED"]}
    for k, name in enumerate(("TB_OK", "TB_ERR_CONFIG", "TB_ERR_INPUT", "TB_ERR_CUDA",
                              "TB_ERR_ARG", "TB_ERR_UNSUPPORTED")):
        assert defs[name] == k == getattr(_native, name)
    assert _native.SCATTER == {"atomic": defs["TB_SCATTER_ATOMIC"],
                               "gather": defs["TB_SCATTER_GATHER"]}
