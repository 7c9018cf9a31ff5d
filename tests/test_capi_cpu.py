"""CPU-side checks of the C ABI library: it loads without a GPU, exports every
symbol include/pmh.h declares, validates arguments with the reference's error
domain, and the host-side package mirrors the reference API surface."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1911_00675_b200 import _lib

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _header_symbols():
    src = open(os.path.join(ROOT, "include", "pmh.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(pmh_\w+)\s*\(", src, re.M)))


def test_library_loads_and_exports_header_symbols():
    L = _lib.load()
    syms = _header_symbols()
    assert len(syms) >= 10
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_lib.EXPORTS)
    assert L.pmh_version() >= 100


def test_invalid_params_rejected_without_gpu():
    """Host-side validation happens before any CUDA call (sketch.py:96-114)."""
    L = _lib.load()
    err = ctypes.c_int64(0)
    # PMH3 needs m >= 2
    rc = L.pmh_sketch_csr(_lib.ALG["probminhash3"], 1, None, None, None, 1, None, None,
                          ctypes.byref(err), None)
    assert rc == _lib.PMH_ERR_INVALID
    # unknown algorithm
    rc = L.pmh_sketch_csr(99, 16, None, None, None, 1, None, None, ctypes.byref(err), None)
    assert rc == _lib.PMH_ERR_INVALID
    # b out of range
    assert L.pmh_bbit(None, 1, 16, 0, None, None) == _lib.PMH_ERR_INVALID
    assert L.pmh_bbit(None, 1, 16, 17, None, None) == _lib.PMH_ERR_INVALID
    # empty batch is a no-op
    assert L.pmh_sketch_csr(_lib.ALG["probminhash1"], 16, None, None, None, 0, None, None,
                            ctypes.byref(err), None) == _lib.PMH_OK


def test_error_mapping_to_reference_exceptions():
    from paper_1911_00675_b200 import (EmptyInputError, InvalidParamsError,
                                       RandomnessFailureError)
    with pytest.raises(InvalidParamsError):
        _lib.check(_lib.PMH_ERR_INVALID)
    with pytest.raises(EmptyInputError):
        _lib.check(_lib.PMH_ERR_EMPTY)
    with pytest.raises(RandomnessFailureError):
        _lib.check(_lib.PMH_ERR_RANDOMNESS)
    assert issubclass(EmptyInputError, ValueError)
    assert issubclass(RandomnessFailureError, RuntimeError)


def test_public_names_match_reference_surface():
    import paper_1911_00675_b200 as pkg
    # the reference's __all__ (/root/reference/pkg/src/probminhash/__init__.py:50-89)
    ref_all = {
        "BBitSignature", "EmptyInputError", "InvalidParamsError", "LazyPermutation",
        "RandomStream", "RandomnessFailureError", "Signature", "SketchParams", "SketchStats",
        "StopLimitTree", "TruncExpParams", "WEIGHTED_ALGORITHMS", "WeightPairMultiset",
        "WeightedSet", "bbit_reduce", "estimate_similarity", "estimate_similarity_bbit",
        "estimator_variance", "improvement_factor", "jaccard_exact", "jaccard_n_exact",
        "jaccard_p_exact", "jaccard_w_exact", "minhash", "new_stream", "oph_densified",
        "perm_new", "pminhash", "probminhash1", "probminhash1a", "probminhash2",
        "probminhash3", "probminhash3a", "probminhash4", "sketch_unweighted", "superminhash",
        "superminhash_variance", "tree_new"}
    assert ref_all <= set(pkg.__all__)
    for n in ref_all:
        assert hasattr(pkg, n), n


def test_host_validation_mirrors_reference():
    from paper_1911_00675_b200 import InvalidParamsError, SketchParams, WeightedSet
    import math
    with pytest.raises(InvalidParamsError):
        WeightedSet([(1, 0.0)])
    with pytest.raises(InvalidParamsError):
        WeightedSet([(1, -2.0)])
    with pytest.raises(InvalidParamsError):
        WeightedSet([(1, math.inf)])
    with pytest.raises(InvalidParamsError):
        WeightedSet([(1, 1.0), (1, 2.0)])
    with pytest.raises(InvalidParamsError):
        WeightedSet.from_arrays([1, 2], [1.0])
    with pytest.raises(InvalidParamsError):
        SketchParams(0)
    ws = WeightedSet([(5, 1.5), (7, 2.0)])
    assert len(ws) == 2 and ws.ids.dtype == np.uint64


def test_compute_fails_loudly_without_cuda(monkeypatch):
    """No CPU fallback: without a CUDA device the product path raises."""
    import torch
    from paper_1911_00675_b200 import WeightedSet, probminhash1
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        probminhash1(WeightedSet([(1, 1.0)]), 8)


def test_multi_async_validates_before_device_work():
    import ctypes
    L = _lib.load()
    arr = (ctypes.c_int * 2)(1, 99)
    outs = (ctypes.c_void_p * 2)(None, None)
    rc = L.pmh_sketch_csr_multi_async(arr, 2, 64, None, None, None, 3, outs, None, None, None)
    assert rc == _lib.PMH_ERR_INVALID
    rc = L.pmh_sketch_csr_multi_async(arr, 0, 64, None, None, None, 3, outs, None, None, None)
    assert rc == _lib.PMH_ERR_INVALID
    one = (ctypes.c_int * 1)(4)
    rc = L.pmh_sketch_csr_multi_async(one, 1, 1, None, None, None, 3, outs, None, None, None)
    assert rc == _lib.PMH_ERR_INVALID   # PMH3 needs m >= 2


def test_bbit_words_and_validation():
    L = _lib.load()
    for m, b in [(256, 1), (256, 3), (100, 7), (1024, 16), (1, 13)]:
        assert L.pmh_bbit_words(m, b) == -(-m // (64 // b))
    assert L.pmh_bbit_words(0, 4) == -1 and L.pmh_bbit_words(8, 17) == -1
    assert L.pmh_bbit_pack(None, 1, 8, 0, None, None) == _lib.PMH_ERR_INVALID
    assert L.pmh_allpairs_bbit_hist(None, 4, 8, 17, 0, 4, 0, 4, 1, None, None, 0, None,
                                    None) == _lib.PMH_ERR_INVALID
    assert L.pmh_allpairs_bbit_hist(None, 4, 8, 4, 0, 5, 0, 4, 1, None, None, 0, None,
                                    None) == _lib.PMH_ERR_INVALID


def test_bbit_host_helpers():
    from paper_1911_00675_b200.batch import bbit_estimate, bbit_unpack
    b, m = 3, 50
    rng = np.random.default_rng(0)
    comp = rng.integers(0, 1 << b, size=(4, m))
    fpw = 64 // b
    words = np.zeros((4, -(-m // fpw)), np.uint64)
    for k in range(m):
        words[:, k // fpw] |= comp[:, k].astype(np.uint64) << np.uint64(b * (k % fpw))
    assert np.array_equal(bbit_unpack(words.view(np.int64), m, b), comp)
    # estimate.py:117-123 on a few counts
    for c in (0, 10, 25, 50):
        p = 2.0 ** -b
        assert bbit_estimate(c, m, b) == min(1.0, max(0.0, (c / m - p) / (1 - p)))


def test_nonstreaming_api_validation():
    """Non-streaming PMH2/PMH4 (configs[3]): argument checks run on the host
    before any CUDA call, with the reference's exception types."""
    import math
    from paper_1911_00675_b200 import (EmptyInputError, InvalidParamsError,
                                       NONSTREAMING_ALGORITHMS, WeightedSet,
                                       probminhash2_nonstreaming, probminhash4_nonstreaming)
    assert set(NONSTREAMING_ALGORITHMS) == {"nonstreaming2", "nonstreaming4"}
    ws = WeightedSet([(1, 1.0), (2, 0.5)])
    for bad in (0.0, -1.0, math.inf, math.nan):
        with pytest.raises(InvalidParamsError):
            probminhash2_nonstreaming(ws, 16, total_weight=bad)
        with pytest.raises(InvalidParamsError):
            probminhash4_nonstreaming(ws, 16, total_weight=bad)
    with pytest.raises(InvalidParamsError):
        probminhash4_nonstreaming(ws, 1)           # m >= 2 like probminhash4
    with pytest.raises(EmptyInputError):
        probminhash2_nonstreaming(WeightedSet([]), 16)


@pytest.mark.parametrize("algo,m_bad", [("pminhash", 16385), ("minhash", 16385),
                                        ("probminhash1", 13841), ("probminhash3a", 13841),
                                        ("unweighted3", 13841), ("probminhash2", 6776),
                                        ("probminhash4", 6776), ("unweighted4", 6776),
                                        ("superminhash", 65536)])
def test_signature_size_limits_rejected_before_cuda(algo, m_bad):
    """m beyond the shared-memory limits is refused with
    PMH_ERR_INVALID by host validation -- no CUDA call is made, so this runs
    without a GPU."""
    import ctypes
    from paper_1911_00675_b200 import _lib
    L = _lib.load()
    err = ctypes.c_int64(-1)
    p = ctypes.c_void_p(4096)      # never dereferenced: validation fails first
    rc = L.pmh_sketch_csr(_lib.ALG[algo], m_bad, p, p, p, 1, p, None, ctypes.byref(err), None)
    assert rc == _lib.PMH_ERR_INVALID
