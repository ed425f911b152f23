"""Accuracy of the branch-free fp64 exp/log/log1p/rcp used by the pair term
(csrc/tb_fastmath.h), checked on the host against glibc libm over their
documented domains (the same source compiles for the device)."""

import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fastmath_ulp_bounds(tmp_path):
    exe = tmp_path / "fmc"
    subprocess.run(["/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc", "-O2",
                    "-std=c11", "-o", str(exe),
                    os.path.join(ROOT, "tests", "native", "fastmath_check.c"), "-lm"],
                   check=True)
    out = json.loads(subprocess.run([str(exe), "400000"], check=True, capture_output=True,
                                    text=True).stdout)
    assert out["ood_ok"] == 1  # libm fallback outside the fast domains
    assert out["exp_ulp"] <= 4
    assert out["log_ulp"] <= 2
    assert out["log1p_ulp"] <= 2
    assert out["rcp_ulp"] <= 1
    assert out["sqrt_ulp"] <= 1
    assert out["rsqrt_ulp"] <= 4
