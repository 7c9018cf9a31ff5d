"""Loader and thin typed wrapper of the native library libpmh.so (C ABI in
include/pmh.h).  The library is built in-tree by __graft_entry__.build()
(or `python -m paper_1911_00675_b200.build`).  There is no fallback: if the
library or a CUDA device is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import EmptyInputError, InvalidParamsError, RandomnessFailureError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PMH_LIB_PATH") or os.path.join(_HERE, "libpmh.so")

PMH_OK = 0
PMH_ERR_EMPTY = -1
PMH_ERR_INVALID = -2
PMH_ERR_RANDOMNESS = -3
PMH_ERR_CUDA = -4
PMH_ERR_NOMEM = -5

# reference algorithm ids, K:866-881
ALG = {
    "pminhash": 0, "probminhash1": 1, "probminhash1a": 2, "probminhash2": 3,
    "probminhash3": 4, "probminhash3a": 5, "probminhash4": 6,
    "minhash": 10, "superminhash": 11, "oph": 12,
    "unweighted1": 13, "unweighted1a": 14, "unweighted2": 15,
    "unweighted3": 16, "unweighted3a": 17, "unweighted4": 18,
}
UNWEIGHTED_IDS = {10, 11, 12, 13, 14, 15, 16, 17, 18}

# every symbol include/pmh.h declares
EXPORTS = ("pmh_version", "pmh_last_error", "pmh_sketch_csr", "pmh_sketch_csr_async",
           "pmh_sketch_csr_multi_async",
           "pmh_status_reset", "pmh_status_check", "pmh_sketch_csr_host", "pmh_sketch_csr_host_multi",
           "pmh_sketch_csr_host_multi_async",
           "pmh_count_equal", "pmh_allpairs_tile", "pmh_allpairs_hist", "pmh_bbit",
           "pmh_bbit_words", "pmh_bbit_pack", "pmh_allpairs_bbit_hist",
           "pmh_mse_cell", "pmh_parse_weighted_text", "pmh_probe_alu_peak",
           "pmh_probe_pipe_peak", "pmh_probe_point_rate", "pmh_math_eval",
           "pmh_sketch_csr_w_async", "pmh_set_weights", "pmh_allpairs_join_hist")

_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)


class NativeLibraryMissing(RuntimeError):
    pass


def load():
    """Load libpmh.so (no CUDA context is created)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run __graft_entry__.build() "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        L.pmh_version.restype = ctypes.c_int
        L.pmh_last_error.restype = ctypes.c_char_p
        L.pmh_sketch_csr.argtypes = [ctypes.c_int, _i64, _vp, _vp, _vp, _i64, _vp, _vp,
                                     _i64p, _vp]
        L.pmh_sketch_csr.restype = ctypes.c_int
        L.pmh_sketch_csr_async.argtypes = [ctypes.c_int, _i64, _vp, _vp, _vp, _i64, _vp, _vp,
                                           _vp, _vp]
        L.pmh_sketch_csr_async.restype = ctypes.c_int
        L.pmh_sketch_csr_multi_async.argtypes = [_vp, ctypes.c_int, _i64, _vp, _vp, _vp, _i64,
                                                 _vp, _vp, _vp, _vp]
        L.pmh_sketch_csr_multi_async.restype = ctypes.c_int
        L.pmh_status_reset.argtypes = [_vp, _vp]
        L.pmh_status_reset.restype = ctypes.c_int
        L.pmh_status_check.argtypes = [_vp, _i64p, _vp]
        L.pmh_status_check.restype = ctypes.c_int
        L.pmh_sketch_csr_host.argtypes = [ctypes.c_int, _i64, _vp, _vp, _vp, _i64, _i64,
                                          _vp, _vp, _i64p]
        L.pmh_sketch_csr_host.restype = ctypes.c_int
        L.pmh_sketch_csr_host_multi.argtypes = [_vp, ctypes.c_int, _i64, _vp, _vp, _vp, _i64,
                                                _i64, _vp, _vp, _i64p]
        L.pmh_sketch_csr_host_multi.restype = ctypes.c_int
        L.pmh_sketch_csr_host_multi_async.argtypes = [_vp, ctypes.c_int, _i64, _vp, _vp, _vp, _i64,
                                                      _i64, _vp, _vp, _vp, _vp]
        L.pmh_sketch_csr_host_multi_async.restype = ctypes.c_int
        L.pmh_count_equal.argtypes = [_vp, _vp, _i64, _i64, _vp, _vp]
        L.pmh_count_equal.restype = ctypes.c_int
        L.pmh_allpairs_tile.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _i64, _vp, _i64,
                                        _vp]
        L.pmh_allpairs_tile.restype = ctypes.c_int
        L.pmh_allpairs_hist.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _i64, ctypes.c_int32,
                                         _vp, _vp, _i64, _vp, _vp]
        L.pmh_allpairs_hist.restype = ctypes.c_int
        L.pmh_bbit.argtypes = [_vp, _i64, _i64, ctypes.c_int, _vp, _vp]
        L.pmh_bbit.restype = ctypes.c_int
        L.pmh_bbit_words.argtypes = [_i64, ctypes.c_int]
        L.pmh_bbit_words.restype = _i64
        L.pmh_bbit_pack.argtypes = [_vp, _i64, _i64, ctypes.c_int, _vp, _vp]
        L.pmh_bbit_pack.restype = ctypes.c_int
        L.pmh_allpairs_bbit_hist.argtypes = [_vp, _i64, _i64, ctypes.c_int, _i64, _i64, _i64, _i64,
                                             ctypes.c_int32, _vp, _vp, _i64, _vp, _vp]
        L.pmh_allpairs_bbit_hist.restype = ctypes.c_int
        L.pmh_parse_weighted_text.argtypes = [ctypes.c_char_p, _i64, _vp, _vp, _i64]
        L.pmh_parse_weighted_text.restype = _i64
        L.pmh_mse_cell.argtypes = [ctypes.c_int, _i64, _vp, _vp, _i64, ctypes.c_uint64, _i64,
                                   _vp, _vp]
        L.pmh_mse_cell.restype = ctypes.c_int
        L.pmh_probe_alu_peak.argtypes = [ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
        L.pmh_probe_alu_peak.restype = ctypes.c_int
        L.pmh_probe_pipe_peak.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
        L.pmh_probe_pipe_peak.restype = ctypes.c_int
        L.pmh_probe_point_rate.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                           ctypes.POINTER(ctypes.c_double)]
        L.pmh_probe_point_rate.restype = ctypes.c_int
        L.pmh_sketch_csr_w_async.argtypes = [ctypes.c_int, _i64, _vp, _vp, _vp, _i64, _vp, _vp,
                                             _vp, _vp, _vp]
        L.pmh_sketch_csr_w_async.restype = ctypes.c_int
        L.pmh_set_weights.argtypes = [_vp, _vp, _i64, _vp, _vp]
        L.pmh_set_weights.restype = ctypes.c_int
        L.pmh_allpairs_join_hist.argtypes = [_vp, _i64, _i64, _i64, _i64, _i64, _i64,
                                             ctypes.c_int32, _vp, _vp, _i64, _vp, _i64, _vp]
        L.pmh_allpairs_join_hist.restype = ctypes.c_int
        L.pmh_math_eval.argtypes = [ctypes.c_int, _vp, _i64, _vp, _vp]
        L.pmh_math_eval.restype = ctypes.c_int
        _lib = L
        return L


def check(rc: int, err_set: int = -1):
    """Map a C status to the reference's exception types (errors.py)."""
    if rc == PMH_OK:
        return
    msg = load().pmh_last_error().decode(errors="replace")
    if rc == PMH_ERR_EMPTY:
        raise EmptyInputError(msg)
    if rc == PMH_ERR_INVALID:
        raise InvalidParamsError(msg)
    if rc == PMH_ERR_RANDOMNESS:
        raise RandomnessFailureError(msg)
    raise RuntimeError(f"libpmh error {rc}: {msg}")
