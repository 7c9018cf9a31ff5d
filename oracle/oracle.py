"""ctypes wrapper of the CPU ORACLE (oracle/pmh_oracle.c) -- test infrastructure.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg import this module, as the checker and the CPU baseline.  The
product package (paper_1911_00675_b200) never imports it.

The oracle restates /root/reference/pkg/src/probminhash/_kernels.py (K) in C;
its parity with the live numba reference is pinned by the committed fixtures
in tests/golden/ (generator: tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None
_lock = threading.Lock()

# K:866-881
ALG = {
    "pminhash": 0, "probminhash1": 1, "probminhash1a": 2, "probminhash2": 3,
    "probminhash3": 4, "probminhash3a": 5, "probminhash4": 6,
    "minhash": 10, "superminhash": 11, "oph": 12,
    "unweighted1": 13, "unweighted1a": 14, "unweighted2": 15,
    "unweighted3": 16, "unweighted3a": 17, "unweighted4": 18,
}
RANDOMNESS_FAILURE = 3

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    """Compile liborc.so with the committed Makefile (gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "pmh_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.run(["make", "-s", "-C", _HERE, "liborc.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                build()
            L = ctypes.CDLL(_LIB_PATH)
            L.orc_sketch.argtypes = [ctypes.c_int, _u64p, _f64p, ctypes.c_int64,
                                     ctypes.c_int64, _u64p, _i64p, _f64p,
                                     ctypes.c_double]
            L.orc_sketch.restype = ctypes.c_int
            L.orc_sketch_csr.argtypes = [ctypes.c_int, ctypes.c_int64, _u64p, _f64p,
                                         _i64p, ctypes.c_int64, ctypes.c_int64,
                                         _u64p, _i64p]
            L.orc_sketch_csr.restype = ctypes.c_int
            L.orc_pminhash_part.argtypes = [_u64p, _f64p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, _f64p, _i64p]
            L.orc_pminhash_part.restype = None
            L.orc_bbit.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int, _i64p]
            L.orc_count_equal.argtypes = [_u64p, _u64p, ctypes.c_int64,
                                          ctypes.c_int64, _i32p]
            L.orc_allpairs.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.c_int64, _i32p]
            L.orc_stream_words.argtypes = [ctypes.c_uint64, ctypes.c_int64, _u64p]
            L.orc_stream_uniform01.argtypes = [ctypes.c_uint64, ctypes.c_int64, _f64p]
            L.orc_stream_exp1.argtypes = [ctypes.c_uint64, ctypes.c_int64, _f64p]
            L.orc_stream_trunc_exp.argtypes = [ctypes.c_uint64, ctypes.c_double,
                                               ctypes.c_int64, _f64p]
            L.orc_trunc_exp_consts.argtypes = [ctypes.c_double, _f64p]
            _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _algo_id(algo):
    return ALG[algo] if isinstance(algo, str) else int(algo)


class OracleError(RuntimeError):
    pass


def sketch(algo, ids, weights=None, m=64, pin=float("nan"), want_h=False):
    """One set -> (sig u64[m], stats i64[3]) [, hfinal]."""
    ids = np.ascontiguousarray(ids, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    sig = np.zeros(m, np.uint64)
    stats = np.zeros(3, np.int64)
    h = np.zeros(1, np.float64)
    rc = lib().orc_sketch(_algo_id(algo), _p(ids, _u64p),
                          None if w is None else _p(w, _f64p), ids.size, m,
                          _p(sig, _u64p), _p(stats, _i64p), _p(h, _f64p),
                          float(pin))
    if rc:
        raise OracleError(f"oracle error {rc}")
    return (sig, stats, float(h[0])) if want_h else (sig, stats)


def sketch_csr(algo, m, ids, weights, offsets, set_range=None, threads=1):
    """CSR batch -> (sig u64[nsets, m], stats i64[nsets, 3]).

    threads > 1 splits the set range into contiguous chunks run by Python
    threads (ctypes releases the GIL, so they run on separate cores)."""
    ids = np.ascontiguousarray(ids, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    s0, s1 = (0, offsets.size - 1) if set_range is None else set_range
    ns = s1 - s0
    sig = np.zeros((ns, m), np.uint64)
    stats = np.zeros((ns, 3), np.int64)
    L = lib()
    aid = _algo_id(algo)

    def run(a, b):
        return L.orc_sketch_csr(aid, m, _p(ids, _u64p),
                                None if w is None else _p(w, _f64p),
                                _p(offsets, _i64p), a, b,
                                _p(sig[a - s0:], _u64p), _p(stats[a - s0:], _i64p))

    if threads <= 1 or ns <= 1:
        rcs = [run(s0, s1)]
    else:
        # interleaved fine-grained chunks balance the log-uniform set sizes
        chunk = max(1, ns // (threads * 16))
        bounds = [(a, min(a + chunk, s1)) for a in range(s0, s1, chunk)]
        with ThreadPoolExecutor(threads) as ex:
            rcs = list(ex.map(lambda ab: run(*ab), bounds))
    for rc in rcs:
        if rc:
            raise OracleError(f"oracle error {rc}")
    return sig, stats


def sketch_csr_balanced(algo, m, ids, weights, offsets, threads=1, part=2048):
    """sketch_csr with equal-cost work items for a multi-core CPU baseline:
    P-MinHash sets are cut into element parts of <= `part` elements (merged on
    (h, index): order-independent, so the signature is exactly the sequential
    one), every other algorithm runs whole sets; items go to the thread pool
    largest-cost first (LPT).  Returns sig u64[nsets, m]."""
    ids = np.ascontiguousarray(ids, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    ns = offsets.size - 1
    sig = np.zeros((ns, m), np.uint64)
    L = lib()
    aid = _algo_id(algo)
    sizes = np.diff(offsets)
    if aid == ALG["pminhash"]:
        items = [(s, a, min(a + part, int(sizes[s]))) for s in range(ns)
                 for a in range(0, int(sizes[s]), part)]
        hmin = [np.full((len(range(0, int(sizes[s]), part)), m), np.inf) for s in range(ns)]
        idx = [np.full((len(range(0, int(sizes[s]), part)), m), -1, np.int64) for s in range(ns)]

        def run(it):
            s, a, b = it
            o = int(offsets[s])
            L.orc_pminhash_part(_p(ids[o + a:], _u64p), _p(w[o + a:], _f64p), b - a, m, a,
                                _p(hmin[s][a // part], _f64p), _p(idx[s][a // part], _i64p))
            return 0
        order = sorted(items, key=lambda it: -(it[2] - it[1]))
    else:
        def run(s):
            return L.orc_sketch_csr(aid, m, _p(ids, _u64p), None if w is None else _p(w, _f64p),
                                    _p(offsets, _i64p), s, s + 1, _p(sig[s:], _u64p), None)
        order = sorted(range(ns), key=lambda s: -(int(sizes[s]) + 7 * m))
    with ThreadPoolExecutor(max(1, threads)) as ex:
        rcs = list(ex.map(run, order))
    if any(rcs):
        raise OracleError(f"oracle error {max(rcs)}")
    if aid == ALG["pminhash"]:
        for s in range(ns):
            h, ix = hmin[s], idx[s]
            # lexicographic (h, index) minimum over the parts of each component
            best = np.lexsort((ix, h), axis=0)[0]
            sel = ix[best, np.arange(m)]
            sig[s] = ids[int(offsets[s]) + sel]
    return sig


def bbit(sig, b):
    sig = np.ascontiguousarray(sig, np.uint64)
    out = np.empty(sig.size, np.int64)
    lib().orc_bbit(_p(sig, _u64p), sig.size, b, _p(out, _i64p))
    return out


def count_equal(a, b):
    a = np.ascontiguousarray(a, np.uint64)
    b = np.ascontiguousarray(b, np.uint64)
    npairs, m = a.shape
    out = np.empty(npairs, np.int32)
    lib().orc_count_equal(_p(a, _u64p), _p(b, _u64p), npairs, m, _p(out, _i32p))
    return out


def allpairs(sigs, r0=0, r1=None):
    sigs = np.ascontiguousarray(sigs, np.uint64)
    n, m = sigs.shape
    r1 = n if r1 is None else r1
    out = np.zeros((r1 - r0, n), np.int32)
    lib().orc_allpairs(_p(sigs, _u64p), n, m, r0, r1, _p(out, _i32p))
    return out


def stream_words(seed, count):
    out = np.empty(count, np.uint64)
    lib().orc_stream_words(seed & 0xFFFFFFFFFFFFFFFF, count, _p(out, _u64p))
    return out


def stream_uniform01(seed, count):
    out = np.empty(count, np.float64)
    lib().orc_stream_uniform01(seed & 0xFFFFFFFFFFFFFFFF, count, _p(out, _f64p))
    return out


def stream_exp1(seed, count):
    out = np.empty(count, np.float64)
    lib().orc_stream_exp1(seed & 0xFFFFFFFFFFFFFFFF, count, _p(out, _f64p))
    return out


def stream_trunc_exp(seed, lam, count):
    out = np.empty(count, np.float64)
    rc = lib().orc_stream_trunc_exp(seed & 0xFFFFFFFFFFFFFFFF, lam, count,
                                    _p(out, _f64p))
    if rc:
        raise OracleError(f"oracle error {rc}")
    return out


def trunc_exp_consts(lam):
    out = np.empty(3, np.float64)
    lib().orc_trunc_exp_consts(lam, _p(out, _f64p))
    return tuple(float(v) for v in out)


def mse_cell(algo, m, wa, wb, seed, s, threads=8):
    """K._k_mse_cell (K:920-963) restated: pair t, weight pair q takes stream
    word t*npairs + q of RandomStream(seed) as its id; side A keeps the q with
    wa[q] > 0, side B those with wb[q] > 0 (q order); both sides are sketched
    and equal components counted -> int64[s]."""
    wa = np.asarray(wa, np.float64)
    wb = np.asarray(wb, np.float64)
    P = wa.size
    words = stream_words(seed, s * P).reshape(s, P)
    ma, mb = wa > 0, wb > 0
    na, nb = int(ma.sum()), int(mb.sum())
    ids = np.concatenate([words[:, ma].ravel(), words[:, mb].ravel()])
    w = np.concatenate([np.tile(wa[ma], s), np.tile(wb[mb], s)])
    off = np.concatenate([np.arange(s + 1, dtype=np.int64) * na,
                          s * na + np.arange(1, s + 1, dtype=np.int64) * nb])
    sig, _ = sketch_csr(algo, m, ids, w, off, threads=threads)
    return (sig[:s] == sig[s:]).sum(axis=1).astype(np.int64)
