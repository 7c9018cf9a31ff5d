"""Device transcendental parity: the DEVICE build of the
glibc log1p / expm1 restatements (csrc/pmh_math.cuh, evaluated by the
pmh_math_eval kernel) against the host glibc, bit for bit, on >= 10^6 inputs
of the sampled domain -- E = -log1p(-U), U = k 2^-53 (K:120-122) -- and of
TruncExp's expm1 argument lam (1 - x) (K:146).  north_star allows a mismatch
fraction < 1e-6; the restatement is exact, so the fraction must be 0.  (A
rare 1-ulp flip seldom changes a signature, so signature parity alone would
not pin this.)"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

from paper_1911_00675_b200 import _lib, datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
N = 1 << 21


@pytest.fixture(scope="module")
def glibc():
    d = tempfile.mkdtemp()
    so = os.path.join(d, "glibc_eval.so")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                    os.path.join(ROOT, "tests", "native", "glibc_eval.c"), "-lm"], check=True)
    L = ctypes.CDLL(so)
    for f in (L.glibc_log1p, L.glibc_expm1):
        f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
    return L


def _host(fn, x):
    y = np.empty_like(x)
    fn(x.ctypes.data, y.ctypes.data, x.size)
    return y


def _device(fn_id, x):
    import torch
    dx = torch.from_numpy(x).cuda()
    out = torch.empty_like(dx)
    _lib.check(_lib.load().pmh_math_eval(fn_id, dx.data_ptr(), x.size, out.data_ptr(),
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out.cpu().numpy()


def _log1p_inputs():
    st = datagen.CounterStream(0xC0FFEE)
    w = st.words(N)
    w2 = st.words(N)
    k = w >> np.uint64(11)
    i = np.arange(N)
    sh = (w2 & np.uint64(63))
    k = np.where(i % 8 == 1, k >> sh, k)                                # small U
    k = np.where(i % 8 == 2, np.uint64((1 << 53) - 1) - (k >> sh), k)   # U near 1
    return -(k.astype(np.float64) * 2.0 ** -53)


def _expm1_inputs():
    st = datagen.CounterStream(0xE4A1)
    t = st.uniform01(N)
    w = st.words(N)
    i = np.arange(N)
    arg = np.where(i % 2 == 1, t * 0.6931471805599453, (t - 0.5) * 2.0 * 1.0397)
    tiny = t * np.exp2(-(w & np.uint64(63)).astype(np.float64))
    return np.where(i % 16 == 3, tiny, arg)


def test_device_log1p_bit_exact_vs_glibc(glibc):
    x = _log1p_inputs()
    got = _device(0, x).view(np.uint64)
    ref = _host(glibc.glibc_log1p, x).view(np.uint64)
    frac = float((got != ref).mean())
    print(f"device log1p vs glibc: {int((got != ref).sum())} mismatches in {x.size} "
          f"(fraction {frac:.3g})")
    assert frac == 0.0


def test_device_log1p_sampled_domain_specialisation_bit_exact(glibc):
    """g_log1p_negu -- the log1p every kernel calls (E = -log1p(-U)) -- on the
    device, against the host glibc, bit for bit."""
    x = _log1p_inputs()
    got = _device(2, x).view(np.uint64)
    ref = _host(glibc.glibc_log1p, x).view(np.uint64)
    frac = float((got != ref).mean())
    print(f"device log1p (x = -U specialisation) vs glibc: {int((got != ref).sum())} "
          f"mismatches in {x.size} (fraction {frac:.3g})")
    assert frac == 0.0


def test_device_expm1_bit_exact_vs_glibc(glibc):
    x = _expm1_inputs()
    got = _device(1, x)
    ok = ~np.isnan(got)
    assert ok.mean() > 0.99
    ref = _host(glibc.glibc_expm1, x)
    mism = (got.view(np.uint64) != ref.view(np.uint64)) & ok
    print(f"device expm1 vs glibc: {int(mism.sum())} mismatches in {int(ok.sum())} "
          f"(fraction {float(mism.sum()) / ok.sum():.3g})")
    assert not mism.any()
