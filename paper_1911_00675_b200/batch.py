"""Batch (CSR) API on the GPU: the engine's native calling convention.

A batch is (ids u64[N], weights f64[N] or None, offsets i64[S+1]).  Inputs may
be numpy arrays (host; copied to the device) or torch CUDA tensors (device
resident; int64 tensors carry the u64 ids bit-for-bit).  Signatures come back
as int64 CUDA tensors (bit-identical to the u64 ids) or numpy uint64 arrays.

Every call goes through libpmh.so (include/pmh.h); there is no CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import EmptyInputError, InvalidParamsError


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1911_00675_b200 needs a CUDA device (no CPU fallback)")
    return torch


def algo_id(algo) -> int:
    if isinstance(algo, str):
        if algo not in _lib.ALG:
            raise InvalidParamsError(f"unknown algorithm {algo!r}")
        return _lib.ALG[algo]
    return int(algo)


def to_device_u64(x, device=None):
    """numpy uint64 / int64 array or torch tensor -> contiguous int64 CUDA tensor."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x if x.dtype == torch.int64 else x.view(torch.int64) if x.dtype == torch.uint64 \
            else x.to(torch.int64)
        return t.to(device or "cuda").contiguous()
    a = np.ascontiguousarray(x)
    if a.dtype != np.uint64:
        a = a.astype(np.uint64)
    return torch.from_numpy(a.view(np.int64)).to(device or "cuda")


def to_device_f64(x, device=None):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device or "cuda", torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, np.float64)).to(device or "cuda")


def to_device_i64(x, device=None):
    torch = _torch()
    if isinstance(x, torch.Tensor):
        return x.to(device or "cuda", torch.int64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x, np.int64)).to(device or "cuda")


def _check_host_csr(ids, weights, offsets):
    """Host CSR bounds: offsets[0] == 0 and offsets[-1] == ids.size (== weights.size
    when weighted), so the C ABI's copies stay inside the caller's arrays."""
    if offsets.ndim != 1 or offsets.size < 1:
        raise InvalidParamsError("offsets must be a 1-d array of nsets + 1 entries")
    if offsets.size > 1:
        if int(offsets[0]) != 0:
            raise InvalidParamsError("offsets[0] must be 0")
        if int(offsets[-1]) != ids.size:
            raise InvalidParamsError(f"offsets[-1] = {int(offsets[-1])} != len(ids) = {ids.size}")
        if weights is not None and weights.size != ids.size:
            raise InvalidParamsError(f"len(weights) = {weights.size} != len(ids) = {ids.size}")


def _check_device_csr(torch, ids, weights, offsets):
    """Device CSR: dtypes, contiguity, one device, and the offsets' ends against
    the array lengths (one 16-byte read of offsets; the call syncs anyway)."""
    if ids.dtype not in (torch.int64, torch.uint64):
        raise InvalidParamsError(f"ids must be int64/uint64, got {ids.dtype}")
    if offsets.dtype != torch.int64:
        raise InvalidParamsError(f"offsets must be int64, got {offsets.dtype}")
    if weights is not None and weights.dtype != torch.float64:
        raise InvalidParamsError(f"weights must be float64, got {weights.dtype}")
    for name, t in (("ids", ids), ("offsets", offsets), ("weights", weights)):
        if t is None:
            continue
        if not t.is_cuda or t.device != ids.device:
            raise InvalidParamsError(f"{name} must be a CUDA tensor on {ids.device}")
        if t.dim() != 1 or not t.is_contiguous():
            raise InvalidParamsError(f"{name} must be a contiguous 1-d tensor")
    if offsets.numel() > 1:
        o0, o1 = (int(v) for v in offsets[[0, -1]].tolist())
        if o0 != 0:
            raise InvalidParamsError("offsets[0] must be 0")
        if o1 != ids.numel():
            raise InvalidParamsError(f"offsets[-1] = {o1} != len(ids) = {ids.numel()}")
        if weights is not None and weights.numel() != ids.numel():
            raise InvalidParamsError(f"len(weights) = {weights.numel()} != len(ids) = {ids.numel()}")


def _stream_ptr(torch, dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def sketch_csr_device(algo, m: int, ids, weights, offsets, want_stats=True, set_weights=None):
    """Device-resident batch sketch.

    ids: int64 CUDA tensor [N]; weights: float64 CUDA tensor [N] or None;
    offsets: int64 CUDA tensor [S+1].  set_weights: optional float64 CUDA
    tensor [S] of the sets' total weights known in advance (the non-streaming
    form, pmh_sketch_csr_w_async; any positive values give the same
    signatures).  Returns (sig int64 [S, m] CUDA tensor, stats int64 [S, 3]
    CUDA tensor or None)."""
    torch = _torch()
    aid = algo_id(algo)
    nsets = offsets.numel() - 1
    dev = ids.device
    sig = torch.empty((max(nsets, 0), m), dtype=torch.int64, device=dev)
    stats = torch.empty((max(nsets, 0), 3), dtype=torch.int64, device=dev) if want_stats else None
    if aid in _lib.UNWEIGHTED_IDS:
        weights = None
    _check_device_csr(torch, ids, weights, offsets)
    if set_weights is not None:
        if (not isinstance(set_weights, torch.Tensor) or set_weights.dtype != torch.float64
                or set_weights.device != dev or set_weights.numel() != max(nsets, 0)):
            raise InvalidParamsError("set_weights must be a float64 tensor of nsets entries on "
                                     "the batch's device")
        L = _lib.load()
        sp = _stream_ptr(torch, dev)
        status = torch.empty(2, dtype=torch.int64, device=dev)
        _lib.check(L.pmh_status_reset(status.data_ptr(), sp))
        _lib.check(L.pmh_sketch_csr_w_async(
            aid, m, ids.data_ptr(), weights.data_ptr() if weights is not None else None,
            offsets.data_ptr(), nsets, set_weights.contiguous().data_ptr(), sig.data_ptr(),
            stats.data_ptr() if stats is not None else None, status.data_ptr(), sp))
        err = ctypes.c_int64(-1)
        _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
        return sig, stats
    err = ctypes.c_int64(-1)
    rc = _lib.load().pmh_sketch_csr(
        aid, m, ids.data_ptr(), weights.data_ptr() if weights is not None else None,
        offsets.data_ptr(), nsets, sig.data_ptr(),
        stats.data_ptr() if stats is not None else None, ctypes.byref(err),
        _stream_ptr(torch, dev))
    _lib.check(rc, err.value)
    return sig, stats


def sketch_csr_multi_device(algos, m: int, ids, weights, offsets, want_stats=False):
    """Device-resident batch sketched by several algorithms concurrently
    (pmh_sketch_csr_multi_async + one status check) -> list of (sig, stats)."""
    torch = _torch()
    aids = [algo_id(a) for a in algos]
    nsets = offsets.numel() - 1
    dev = ids.device
    if all(a in _lib.UNWEIGHTED_IDS for a in aids):
        weights = None
    _check_device_csr(torch, ids, weights, offsets)
    sigs = [torch.empty((max(nsets, 0), m), dtype=torch.int64, device=dev) for _ in aids]
    stats = [torch.empty((max(nsets, 0), 3), dtype=torch.int64, device=dev) if want_stats
             else None for _ in aids]
    L = _lib.load()
    sp = _stream_ptr(torch, dev)
    status = torch.empty(2, dtype=torch.int64, device=dev)
    _lib.check(L.pmh_status_reset(status.data_ptr(), sp))
    arr_a = (ctypes.c_int * len(aids))(*aids)
    arr_s = (ctypes.c_void_p * len(aids))(*[t.data_ptr() for t in sigs])
    arr_t = (ctypes.c_void_p * len(aids))(*[t.data_ptr() if t is not None else None for t in stats])
    rc = L.pmh_sketch_csr_multi_async(arr_a, len(aids), m, ids.data_ptr(),
                                      weights.data_ptr() if weights is not None else None,
                                      offsets.data_ptr(), nsets, arr_s, arr_t,
                                      status.data_ptr(), sp)
    _lib.check(rc)
    err = ctypes.c_int64(-1)
    _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
    return list(zip(sigs, stats))


def sketch_csr(algo, m: int, ids, weights, offsets, want_stats=True, set_weights=None):
    """Host-array batch sketch -> (sig uint64[S, m], stats int64[S, 3]).

    Goes through the C ABI's host entry point (H2D, kernels, D2H inside); with
    set_weights (float64 [S], the sets' total weights known in advance)
    through the device entry pmh_sketch_csr_w_async."""
    aid = algo_id(algo)
    torch = _torch()  # a CUDA device is required
    if set_weights is not None:
        ids_h = np.ascontiguousarray(ids, np.uint64)
        off_h = np.ascontiguousarray(offsets, np.int64)
        w_h = None if (aid in _lib.UNWEIGHTED_IDS or weights is None) else \
            np.ascontiguousarray(weights, np.float64)
        _check_host_csr(ids_h, w_h, off_h)
        sw = np.ascontiguousarray(set_weights, np.float64)
        sig, st = sketch_csr_device(aid, m, to_device_u64(ids_h),
                                    to_device_f64(w_h) if w_h is not None else None,
                                    to_device_i64(off_h), want_stats,
                                    torch.from_numpy(sw).cuda())
        return sigs_to_numpy(sig), (st.cpu().numpy() if st is not None else None)
    ids = np.ascontiguousarray(ids, np.uint64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    nsets = offsets.size - 1
    if aid in _lib.UNWEIGHTED_IDS or weights is None:
        w = None
    else:
        w = np.ascontiguousarray(weights, np.float64)
    _check_host_csr(ids, w, offsets)
    sig = np.empty((max(nsets, 0), m), np.uint64)
    stats = np.empty((max(nsets, 0), 3), np.int64) if want_stats else None
    err = ctypes.c_int64(-1)
    rc = _lib.load().pmh_sketch_csr_host(
        aid, m, ids.ctypes.data, w.ctypes.data if w is not None else None,
        offsets.ctypes.data, nsets, int(offsets[-1]) if nsets > 0 else 0,
        sig.ctypes.data, stats.ctypes.data if stats is not None else None,
        ctypes.byref(err))
    _lib.check(rc, err.value)
    return sig, stats


def sketch_csr_multi(algos, m: int, ids, weights, offsets, sig_outs=None, want_stats=False):
    """Several algorithms over one host batch through pmh_sketch_csr_host_multi
    (inputs cross PCIe once; D2H overlaps the next algorithm's compute).
    sig_outs: optional preallocated host uint64 [S, m] arrays (pinned for
    full overlap).  Returns (list of sig arrays, list of stats or None)."""
    _torch()
    aids = (ctypes.c_int * len(algos))(*[algo_id(a) for a in algos])
    ids = np.ascontiguousarray(ids, np.uint64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    nsets = offsets.size - 1
    _check_host_csr(ids, w, offsets)
    if sig_outs is None:
        sig_outs = [np.empty((nsets, m), np.uint64) for _ in algos]
    stats = [np.empty((nsets, 3), np.int64) for _ in algos] if want_stats else None
    sp = (ctypes.c_void_p * len(algos))(*[o.ctypes.data for o in sig_outs])
    stp = (ctypes.c_void_p * len(algos))(*[o.ctypes.data for o in stats]) if stats else None
    err = ctypes.c_int64(-1)
    rc = _lib.load().pmh_sketch_csr_host_multi(
        aids, len(algos), m, ids.ctypes.data, w.ctypes.data if w is not None else None,
        offsets.ctypes.data, nsets, int(offsets[-1]) if nsets > 0 else 0, sp, stp,
        ctypes.byref(err))
    _lib.check(rc, err.value)
    return sig_outs, stats


def count_equal_device(a, b):
    """a, b: int64 CUDA tensors [P, m] -> int32 CUDA tensor [P] of equal counts."""
    torch = _torch()
    if a.shape != b.shape:
        raise InvalidParamsError("signature sizes differ")
    P, m = a.shape
    out = torch.empty(P, dtype=torch.int32, device=a.device)
    rc = _lib.load().pmh_count_equal(a.contiguous().data_ptr(), b.contiguous().data_ptr(),
                                     P, m, out.data_ptr(), _stream_ptr(torch, a.device))
    _lib.check(rc)
    return out


def allpairs_tile_device(sigs, r0, r1, c0, c1, out=None):
    """Equal-component counts for rows [r0,r1) x cols [c0,c1), upper triangle
    (j > i); uint16 counts in a (r1-r0, c1-c0) int16 CUDA tensor (zeros
    elsewhere)."""
    torch = _torch()
    n, m = sigs.shape
    if out is None:
        out = torch.zeros((r1 - r0, c1 - c0), dtype=torch.int16, device=sigs.device)
    rc = _lib.load().pmh_allpairs_tile(sigs.contiguous().data_ptr(), n, m, r0, r1, c0, c1,
                                       out.data_ptr(), out.stride(0),
                                       _stream_ptr(torch, sigs.device))
    _lib.check(rc)
    return out


def allpairs_hist_device(sigs, r0=0, r1=None, c0=0, c1=None, threshold=1, cap=1 << 22,
                         hist=None, method="dense", max_visits=0):
    """Histogram (int64 [m+1], CUDA) of equal-component counts over the pairs
    (i, j), j > i, of rows [r0,r1) x cols [c0,c1), plus the pairs with count >=
    threshold: returns (hist, pairs int64 [K, 3] numpy (i, j, count), total K).

    method: "dense" compares every pair (pmh_allpairs_hist); "join" visits only
    the pairs sharing a (component, value) key (pmh_allpairs_join_hist; raises
    if it declines); "auto" tries the join and falls back to dense when the
    key lists are too long.  All give the same histogram and pair set."""
    torch = _torch()
    n, m = sigs.shape
    r1 = n if r1 is None else r1
    c1 = n if c1 is None else c1
    if hist is None:
        hist = torch.zeros(m + 1, dtype=torch.int64, device=sigs.device)
    pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=sigs.device)
    cursor = torch.zeros(1, dtype=torch.int64, device=sigs.device)
    L = _lib.load()
    sp = _stream_ptr(torch, sigs.device)
    sg = sigs.contiguous()
    rc = 1
    if method in ("join", "auto") and int(threshold) >= 1:
        rc = L.pmh_allpairs_join_hist(sg.data_ptr(), n, m, r0, r1, c0, c1, int(threshold),
                                      hist.data_ptr(), pairs.data_ptr(), cap, cursor.data_ptr(),
                                      int(max_visits), sp)
        if rc == 1 and method == "join":
            raise InvalidParamsError("join declined: too many pairs share a component")
    elif method not in ("dense", "auto"):
        raise InvalidParamsError(f"unknown all-pairs method {method!r}")
    if rc == 1:
        rc = L.pmh_allpairs_hist(sg.data_ptr(), n, m, r0, r1, c0, c1, int(threshold),
                                 hist.data_ptr(), pairs.data_ptr(), cap, cursor.data_ptr(), sp)
    _lib.check(rc)
    k = int(cursor.item())
    return hist, _pairs_out(pairs, k, cap), k


def bbit_device(sig, b: int):
    torch = _torch()
    S, m = sig.shape
    out = torch.empty((S, m), dtype=torch.int64, device=sig.device)
    rc = _lib.load().pmh_bbit(sig.contiguous().data_ptr(), S, m, b, out.data_ptr(),
                              _stream_ptr(torch, sig.device))
    _lib.check(rc)
    return out


def _pairs_out(pairs, k, cap):
    got = pairs[: min(k, cap)].cpu().numpy()
    ij = got[:, 0].view(np.uint64)
    return np.stack([(ij >> np.uint64(32)).astype(np.int64),
                     (ij & np.uint64(0xFFFFFFFF)).astype(np.int64), got[:, 1]], axis=1)


def bbit_words(m: int, b: int) -> int:
    """Packed words per row: floor(64/b) b-bit fields per word."""
    return -(-m // (64 // b))


def bbit_pack_device(sig, b: int):
    """Fused b-bit reduction (estimate.py:105-114, K:851-861) + packing of a
    [S, m] signature batch -> int64 [S, bbit_words(m, b)] CUDA tensor."""
    torch = _torch()
    S, m = sig.shape
    if not 1 <= b <= 16:
        raise InvalidParamsError("b must be in 1..16")
    out = torch.empty((S, bbit_words(m, b)), dtype=torch.int64, device=sig.device)
    rc = _lib.load().pmh_bbit_pack(sig.contiguous().data_ptr(), S, m, b, out.data_ptr(),
                                   _stream_ptr(torch, sig.device))
    _lib.check(rc)
    return out


def bbit_unpack(packed: np.ndarray, m: int, b: int) -> np.ndarray:
    """Host helper: packed words -> int64 [S, m] b-bit components."""
    fpw = 64 // b
    p = np.ascontiguousarray(packed).view(np.uint64)
    k = np.arange(m)
    words = p[:, k // fpw]
    return ((words >> (np.uint64(b) * (k % fpw).astype(np.uint64))) &
            np.uint64((1 << b) - 1)).astype(np.int64)


def allpairs_bbit_hist_device(packed, m: int, b: int, r0=0, r1=None, c0=0, c1=None,
                              threshold=1, cap=1 << 22, hist=None):
    """As allpairs_hist_device for packed b-bit rows (bbit_pack_device):
    histogram of equal b-bit component counts C (int64 [m+1]) and the pairs
    with C >= threshold.  The collision-corrected estimate of a pair is
    bbit_estimate(C, m, b) (estimate.py:117-123)."""
    torch = _torch()
    n = packed.shape[0]
    r1 = n if r1 is None else r1
    c1 = n if c1 is None else c1
    if hist is None:
        hist = torch.zeros(m + 1, dtype=torch.int64, device=packed.device)
    pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=packed.device)
    cursor = torch.zeros(1, dtype=torch.int64, device=packed.device)
    rc = _lib.load().pmh_allpairs_bbit_hist(packed.contiguous().data_ptr(), n, m, b, r0, r1, c0,
                                            c1, int(threshold), hist.data_ptr(), pairs.data_ptr(),
                                            cap, cursor.data_ptr(), _stream_ptr(torch, packed.device))
    _lib.check(rc)
    k = int(cursor.item())
    return hist, _pairs_out(pairs, k, cap), k


def bbit_estimate(count, m: int, b: int):
    """(C/m - 2^-b) / (1 - 2^-b) clamped to [0, 1] (estimate.py:117-123),
    vectorised over equal-component counts C."""
    c = np.asarray(count, np.float64) / m
    p = 2.0 ** -b
    return np.minimum(1.0, np.maximum(0.0, (c - p) / (1.0 - p)))


def sigs_to_numpy(sig) -> np.ndarray:
    return sig.cpu().numpy().view(np.uint64)


def check_nonempty(offsets):
    sizes = np.diff(np.asarray(offsets, np.int64))
    if sizes.size and (sizes <= 0).any():
        raise EmptyInputError("cannot sketch an empty set")
