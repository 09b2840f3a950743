"""ddiv_k (point.cuh; DESIGN reading A47): division by a per-launch constant through RN(1/d) and two
residual steps must equal the IEEE division __ddiv_rn bit for bit -- the exact high-order path (A40)
relies on it for PPM's and WENO-Z's /6 and for p/(gamma-1).  tools/ddiv_check.cu draws 2^26 dividends per
divisor (random over exponents -950..950, exact multiples, near-midpoint quotients, powers of two,
range edges / zeros / subnormals / non-finite) for d = 6 and gamma - 1 of eight gammas."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ddiv_k_matches_ieee_division(tmp_path):
    exe = str(tmp_path / "ddiv_check")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_2202_12309_b200", "csrc"), os.path.join(ROOT, "tools", "ddiv_check.cu"),
                    "-o", exe], check=True, capture_output=True)
    r = subprocess.run([exe, "26"], capture_output=True, text=True, timeout=600)
    rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(rows) == 9, r.stdout + r.stderr
    for row in rows:
        assert row["mismatches"] == 0, row
    assert r.returncode == 0
