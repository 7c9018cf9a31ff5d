"""The device log1p/expm1 (csrc/pmh_math.cuh) restate glibc's FMA builds:
compile the header with g++ on the host and compare with the host libm
bit-for-bit on millions of inputs (the GPU tests check the device build)."""
import os
import subprocess
import tempfile

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _fma_host():
    flags = open("/proc/cpuinfo").read()
    return " fma " in flags and " avx2 " in flags


@pytest.mark.skipif(not _fma_host(), reason="glibc selects its non-FMA builds on this CPU")
def test_glibc_log1p_expm1_restatement_bit_exact():
    src = os.path.join(ROOT, "tests", "native", "math_check.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "mc")
        subprocess.run(["g++", "-O2", "-ffp-contract=off", "-o", exe, src, "-lm"], check=True)
        out = subprocess.run([exe, "3000000"], capture_output=True, text=True, check=True).stdout
    vals = dict(zip(out.split()[0::2], map(int, out.split()[1::2])))
    assert vals["total"] == 3000000
    assert vals["log1p_dom"] == 0
    assert vals["log1p_negu"] == 0   # the x = -U specialisation the kernels call
    assert vals["log1p_wide"] == 0
    assert vals["expm1"] == 0
    assert vals["expm1_outofrange"] == 0
