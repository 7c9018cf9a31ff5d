"""GPU tests of the drop-in API, mirroring the reference's own tests
(/root/reference/pkg/tests/test_sketch.py, test_estimate.py) through the
CUDA path, plus estimator kernels and size-independent properties at the
BASELINE.json sizes."""
import math

import ctypes

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import _lib
from paper_1911_00675_b200 import (
    WEIGHTED_ALGORITHMS, EmptyInputError, InvalidParamsError, TruncExpParams, WeightedSet,
    bbit_reduce, datagen, estimate_pairs, estimate_similarity, estimate_similarity_bbit,
    minhash, new_stream, oph_densified, pminhash, probminhash1, probminhash1a, probminhash2,
    probminhash3, probminhash3a, probminhash4, sketch_batch, sketch_unweighted, superminhash)
from paper_1911_00675_b200.batch import (allpairs_tile_device, count_equal_device, sigs_to_numpy,
                                         to_device_f64, to_device_i64, to_device_u64)

pytestmark = pytest.mark.gpu
ALL_WEIGHTED = list(WEIGHTED_ALGORITHMS.items())


def _random_set(seed, n, weighted=True):
    b = datagen.random_sets(seed, [n], "pareto2" if weighted else "unit")
    return WeightedSet.from_arrays(b.ids, b.weights, validate=False)


@pytest.mark.parametrize("name,fn", ALL_WEIGHTED)
def test_single_element_all_components_equal(name, fn):
    sig, _ = fn(WeightedSet([(12345, 5.0)]), 8)
    assert np.all(sig.components == 12345)


@pytest.mark.parametrize("name,fn", ALL_WEIGHTED)
def test_deterministic_on_repeat(name, fn):
    ws = _random_set(1, 50)
    assert fn(ws, 16)[0] == fn(ws, 16)[0]


@pytest.mark.parametrize("name,fn", ALL_WEIGHTED)
def test_empty_set_rejected(name, fn):
    with pytest.raises(EmptyInputError):
        fn(WeightedSet.from_arrays([], [], validate=False), 16)


@pytest.mark.parametrize("fn", [probminhash3, probminhash3a, probminhash4])
def test_correlated_variants_require_m2(fn):
    with pytest.raises(InvalidParamsError):
        fn(WeightedSet([(1, 1.0)]), 1)


def test_signature_components_come_from_input():
    ws = _random_set(2, 20)
    members = set(int(i) for i in ws.ids)
    for _, fn in ALL_WEIGHTED:
        sig, _ = fn(ws, 32)
        assert set(int(c) for c in sig.components) <= members


@pytest.mark.parametrize("n", [1, 3, 100])
def test_interleaved_equivalence_pairs(n):
    ws = _random_set(n, n)
    assert probminhash1(ws, 16)[0] == probminhash1a(ws, 16)[0]
    assert probminhash3(ws, 16)[0] == probminhash3a(ws, 16)[0]


def test_power_of_two_scale_invariance():
    ws = _random_set(4, 30)
    for k in (-8, -3, 1, 8):
        scaled = WeightedSet.from_arrays(ws.ids, ws.weights * 2.0 ** k, validate=False)
        for _, fn in ALL_WEIGHTED:
            assert fn(ws, 16)[0] == fn(scaled, 16)[0]


def test_point_budget_without_replacement():
    ws = _random_set(5, 40)
    m = 8
    for fn in (probminhash2, probminhash4):
        _, stats = fn(ws, m)
        assert stats.points_generated <= m * len(ws)


def test_coupon_collector_single_element():
    m = 64
    hm = sum(1.0 / i for i in range(1, m + 1))
    # batch the 300 single-element sets in one call
    ids = np.arange(300, dtype=np.uint64)
    off = np.arange(301, dtype=np.int64)
    _, stats = sketch_batch("probminhash1", ids, np.ones(300), off, m)
    assert np.mean(stats[:, 0]) == pytest.approx(m * hm, rel=0.1)


def test_buffer_stats_only_for_interleaved():
    ws = _random_set(6, 200)
    for name, fn in ALL_WEIGHTED:
        _, stats = fn(ws, 16)
        if name in ("probminhash1a", "probminhash3a"):
            assert stats.max_buffer_size > 0
        else:
            assert stats.max_buffer_size == 0


def test_unit_weights_match_minhash():
    ws = _random_set(7, 25, weighted=False)
    sig, _ = pminhash(ws, 32)
    assert sig == minhash(ws.ids, 32)


def test_correlated_points_stay_in_their_intervals():
    m = 16
    p = TruncExpParams.from_rate(math.log(1.0 + 1.0 / (m - 1)))
    s = new_stream(123)
    w = 0.7
    for i in range(1, m + 1):
        x = ((i - 1) + s.next_trunc_exp(p)) / w
        assert (i - 1) / w <= x < i / w


def test_baselines_single_id():
    for fn in (minhash, superminhash, oph_densified):
        sig = fn(np.array([99], np.uint64), 16)
        assert np.all(sig.components == 99)


def test_superminhash_requires_m2():
    with pytest.raises(InvalidParamsError):
        superminhash(np.array([1], np.uint64), 1)


def test_oph_all_bins_filled():
    ids = new_stream(8).u64_batch(4)
    sig = oph_densified(ids, 256)
    assert set(int(c) for c in sig.components) <= set(int(i) for i in ids)


def test_sketch_unweighted_variants():
    ids = new_stream(9).u64_batch(30)
    for variant in ("1", "1a", "2", "3", "3a", "4"):
        sig, _ = sketch_unweighted(variant, ids, 16)
        assert set(int(c) for c in sig.components) <= set(int(i) for i in ids)
    with pytest.raises(InvalidParamsError):
        sketch_unweighted("5", ids, 16)


def test_unweighted_1_matches_unit_weight_run():
    ids = new_stream(10).u64_batch(12)
    ws = WeightedSet.from_arrays(ids, np.ones(12), validate=False)
    assert sketch_unweighted("1", ids, 16)[0] == probminhash1(ws, 16)[0]


def test_unweighted_3a_first_pass_only_when_n_large():
    m = 16
    n = 100 * m
    for seed in range(10):
        ids = new_stream(seed).u64_batch(n)
        _, stats = sketch_unweighted("3a", ids, m)
        assert stats.points_generated == n


# ---- estimator family -----------------------------------------------------

def test_estimate_similarity_counts_equal_components():
    from paper_1911_00675_b200 import Signature
    a = Signature(np.array([1, 2, 3, 4], np.uint64), 4)
    b = Signature(np.array([1, 9, 3, 8], np.uint64), 4)
    assert estimate_similarity(a, b) == 0.5
    with pytest.raises(InvalidParamsError):
        estimate_similarity(a, Signature(np.array([1, 2], np.uint64), 2))


def test_count_equal_and_allpairs_vs_oracle():
    rng = np.random.default_rng(0)
    # signatures with planted collisions (few distinct ids per column)
    sigs = rng.integers(0, 6, size=(300, 64)).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    A, B = sigs[:150], sigs[150:]
    got = estimate_pairs(A, B)
    ref = orc.count_equal(A, B) / 64.0
    np.testing.assert_array_equal(got, ref)
    import torch
    t = torch.from_numpy(sigs.view(np.int64)).cuda()
    out = allpairs_tile_device(t, 0, 300, 0, 300).cpu().numpy().view(np.uint16)
    full = orc.allpairs(sigs)
    iu = np.triu_indices(300, 1)
    np.testing.assert_array_equal(out[iu], full[iu])
    # tile offsets
    out2 = allpairs_tile_device(t, 64, 200, 100, 300).cpu().numpy().view(np.uint16)
    for i in range(64, 200):
        for j in range(max(100, i + 1), 300):
            assert out2[i - 64, j - 100] == full[i, j]
    c = count_equal_device(t[:150], t[150:]).cpu().numpy()
    np.testing.assert_array_equal(c, orc.count_equal(A, B))


def test_bbit_golden_and_estimator():
    from golden_io import load
    from paper_1911_00675_b200 import Signature
    z = load("bbit")
    sig = Signature(z["sig"], z["sig"].size)
    for b in (1, 2, 4, 8, 16):
        np.testing.assert_array_equal(bbit_reduce(sig, b).components, z[f"bbit_{b}"])
    with pytest.raises(InvalidParamsError):
        bbit_reduce(sig, 0)
    sa, sb = bbit_reduce(sig, 4), bbit_reduce(sig, 4)
    assert estimate_similarity_bbit(sa, sb) == 1.0


# ---- BASELINE-size parity and properties ----------------------------------

def _dev(batch):
    ids = to_device_u64(batch.ids)
    w = to_device_f64(batch.weights) if batch.weights is not None else None
    return ids, w, to_device_i64(batch.offsets)


def test_config1_full_bit_exact():
    """configs[0]: PMH3, m=256, 1000 sets x 1000 elements (the PR1 oracle)."""
    b = datagen.config1()
    sig, _ = sketch_batch("probminhash3", *_dev(b), 256)
    ref, _ = orc.sketch_csr("probminhash3", 256, b.ids, b.weights, b.offsets, threads=16)
    assert (sigs_to_numpy(sig) != ref).sum() == 0


def test_config2_subset_all_variants_bit_exact():
    """configs[1]: the 7 weighted variants at m=1024 on a stratified subset."""
    full = datagen.config2()
    sizes = np.diff(full.offsets)
    order = np.argsort(sizes, kind="stable")
    sub = full.subset(np.sort(order[::50]))           # 200 sets, all sizes
    d = _dev(sub)
    for algo in ("probminhash1", "probminhash1a", "probminhash2", "probminhash3",
                 "probminhash3a", "probminhash4"):
        sig, _ = sketch_batch(algo, *d, 1024)
        ref, _ = orc.sketch_csr(algo, 1024, sub.ids, sub.weights, sub.offsets, threads=16)
        assert (sigs_to_numpy(sig) != ref).sum() == 0, algo
    small = full.subset(np.sort(order[::500]))        # P-MinHash: 20 sets
    sig, _ = sketch_batch("pminhash", *_dev(small), 1024)
    ref, _ = orc.sketch_csr("pminhash", 1024, small.ids, small.weights, small.offsets, threads=16)
    assert (sigs_to_numpy(sig) != ref).sum() == 0


def test_config2_pminhash_reference_sample_bit_exact():
    """configs[1] P-MinHash at m=1024 on the reference arm's 137-set stratified
    sample (1.14M elements, sizes 1..10^5, the largest sets split across CTAs
    on the GPU) against the oracle's equal-cost parallel run."""
    import os
    full = datagen.config2()
    sizes = np.diff(full.offsets)
    order = np.argsort(sizes, kind="stable")
    k = int(np.ceil(sizes.sum() / 1_200_000))
    sub = full.subset(np.sort(order[::k]))
    assert sub.nelems > 1_000_000
    sig, _ = sketch_batch("pminhash", *_dev(sub), 1024)
    ref = orc.sketch_csr_balanced("pminhash", 1024, sub.ids, sub.weights, sub.offsets,
                                  threads=os.cpu_count() or 8)
    assert (sigs_to_numpy(sig) != ref).sum() == 0


def test_config2_full_properties():
    """Full configs[1] batch: permutation invariance within sets, power-of-two
    scale invariance and determinism (size-independent properties)."""
    full = datagen.config2()
    ids, w, off = _dev(full)
    rng = np.random.default_rng(1)
    perm = np.concatenate([rng.permutation(np.arange(a, b))
                           for a, b in zip(full.offsets[:-1], full.offsets[1:])])
    for algo in ("probminhash1", "probminhash2", "probminhash3", "probminhash4", "pminhash"):
        s1, _ = sketch_batch(algo, ids, w, off, 1024)
        s2, _ = sketch_batch(algo, ids[perm], w[perm], off, 1024)
        s3, _ = sketch_batch(algo, ids, w * 8.0, off, 1024)
        s4, _ = sketch_batch(algo, ids, w, off, 1024)
        a1 = sigs_to_numpy(s1)
        assert np.array_equal(a1, sigs_to_numpy(s2)), algo
        assert np.array_equal(a1, sigs_to_numpy(s3)), algo
        assert np.array_equal(a1, sigs_to_numpy(s4)), algo


def test_config3_unweighted_m4096_subset():
    """configs[2]: unweighted variants at m=4096 (1000 ids per set)."""
    b = datagen.config3(nsets=64)
    d = _dev(b)
    for algo in ("unweighted1", "unweighted1a", "unweighted2", "unweighted3", "unweighted3a",
                 "unweighted4"):
        sig, _ = sketch_batch(algo, d[0], None, d[2], 4096)
        ref, _ = orc.sketch_csr(algo, 4096, b.ids, None, b.offsets, threads=16)
        assert (sigs_to_numpy(sig) != ref).sum() == 0, algo


def test_config4_pareto_m64_subset():
    """configs[3]: PMH2/PMH4 at m=64, Pareto(1.5) weights (non-streaming ==
    streaming signatures)."""
    b = datagen.config4(nsets=20000)
    d = _dev(b)
    for algo in ("probminhash2", "probminhash4"):
        sig, _ = sketch_batch(algo, *d, 64)
        ref, _ = orc.sketch_csr(algo, 64, b.ids, b.weights, b.offsets, threads=16)
        assert (sigs_to_numpy(sig) != ref).sum() == 0, algo


@pytest.mark.parametrize("m", [64, 1024])
def test_nonstreaming_batch_with_set_weights(m):
    """sketch_batch("nonstreaming2/4", set_weights=...) through
    pmh_sketch_csr_w_async: the kernels take the caller's W_s and skip their
    weight pre-pass; exact W, W off by 10^-3..10^3 (scheduling only: too
    large costs points, too small forces the verified retry) and the device
    sums all give the oracle's signatures, on the device and host paths."""
    import torch
    b = datagen.config4(nsets=3000, seed=5)
    W = np.add.reduceat(b.weights, b.offsets[:-1])
    rng = np.random.default_rng(1)
    wrong = W * np.exp(rng.uniform(np.log(1e-3), np.log(1e3), W.size))
    d = _dev(b)
    L = _lib.load()
    dev_w = torch.empty(b.nsets, dtype=torch.float64, device="cuda")
    _lib.check(L.pmh_set_weights(d[1].data_ptr(), d[2].data_ptr(), b.nsets, dev_w.data_ptr(),
                                 ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    np.testing.assert_allclose(dev_w.cpu().numpy(), W, rtol=1e-12)
    for algo in ("nonstreaming2", "nonstreaming4"):
        ref, _ = orc.sketch_csr("probminhash" + algo[-1], m, b.ids, b.weights, b.offsets, threads=16)
        for sw in (W, wrong, dev_w):
            sig, _ = sketch_batch(algo, *d, m, set_weights=sw)
            assert np.array_equal(sigs_to_numpy(sig), ref), (algo, m)
        sig, _ = sketch_batch(algo, b.ids, b.weights, b.offsets, m, set_weights=wrong)
        assert np.array_equal(sig, ref), (algo, m, "host")


@pytest.mark.parametrize("m", [2, 64, 1024])
def test_nonstreaming_single_set_api(m):
    """probminhash2/4_nonstreaming == streaming signatures == oracle, with and
    without a total weight (also a wrong one: it is scheduling-only)."""
    from paper_1911_00675_b200 import (WeightedSet, probminhash2_nonstreaming,
                                       probminhash4_nonstreaming)
    b = datagen.config4(nsets=12, seed=3)
    for i in range(b.nsets):
        lo, hi = b.offsets[i], b.offsets[i + 1]
        ws = WeightedSet.from_arrays(b.ids[lo:hi], b.weights[lo:hi])
        W = float(b.weights[lo:hi].sum())
        for algo, fn in (("probminhash2", probminhash2_nonstreaming),
                         ("probminhash4", probminhash4_nonstreaming)):
            ref, _ = orc.sketch_csr(algo, m, b.ids[lo:hi], b.weights[lo:hi],
                                    np.array([0, hi - lo], np.int64))
            for tw in (None, W, 1e-3 * W, 1e3 * W):
                sig, _ = fn(ws, m, total_weight=tw)
                assert np.array_equal(sig.components, ref[0]), (algo, i, tw)


def test_empty_set_in_batch_reports_index():
    ids = np.arange(10, dtype=np.uint64)
    off = np.array([0, 4, 4, 10], np.int64)
    import ctypes
    from paper_1911_00675_b200 import _lib
    L = _lib.load()
    t_ids, t_w, t_off = to_device_u64(ids), to_device_f64(np.ones(10)), to_device_i64(off)
    import torch
    sig = torch.empty((3, 16), dtype=torch.int64, device="cuda")
    err = ctypes.c_int64(-1)
    rc = L.pmh_sketch_csr(_lib.ALG["probminhash3"], 16, t_ids.data_ptr(), t_w.data_ptr(),
                          t_off.data_ptr(), 3, sig.data_ptr(), None, ctypes.byref(err), None)
    assert rc == _lib.PMH_ERR_EMPTY and err.value == 1


def test_host_multi_matches_single_calls():
    """pmh_sketch_csr_host_multi (chunked H2D, overlapped D2H) == per-algorithm
    device calls, including the chunked first algorithm."""
    from paper_1911_00675_b200.batch import sketch_csr_multi
    b = datagen.random_sets(31, list(np.exp(np.linspace(0, 9.5, 40)).astype(int) + 1), "uniform")
    algos = ["probminhash3", "pminhash", "probminhash2", "probminhash4", "probminhash1"]
    sigs, stats = sketch_csr_multi(algos, 256, b.ids, b.weights, b.offsets, want_stats=True)
    for a, sg in zip(algos, sigs):
        ref, _ = orc.sketch_csr(a, 256, b.ids, b.weights, b.offsets, threads=16)
        assert np.array_equal(sg, ref), a
    with pytest.raises(EmptyInputError):
        sketch_csr_multi(["probminhash1"], 16, np.arange(3, dtype=np.uint64), np.ones(3),
                         np.array([0, 3, 3]))


def test_multi_async_matches_single_calls():
    """pmh_sketch_csr_multi_async (variants on concurrent internal streams)
    == the oracle for every algorithm, weighted and unweighted, with stats."""
    from paper_1911_00675_b200.batch import sketch_csr_multi_device, to_device_f64, to_device_i64, to_device_u64
    b = datagen.random_sets(33, list(np.exp(np.linspace(0, 9.0, 48)).astype(int) + 1), "pareto1.5")
    algos = ["probminhash1", "probminhash1a", "probminhash2", "probminhash3", "probminhash3a",
             "probminhash4", "pminhash", "unweighted3", "unweighted4", "minhash"]
    outs = sketch_csr_multi_device(algos, 256, to_device_u64(b.ids), to_device_f64(b.weights),
                                   to_device_i64(b.offsets), want_stats=True)
    for a, (sg, st) in zip(algos, outs):
        w = None if a in ("unweighted3", "unweighted4", "minhash") else b.weights
        ref, _ = orc.sketch_csr(a, 256, b.ids, w, b.offsets, threads=16)
        assert np.array_equal(sg.cpu().numpy().view(np.uint64), ref), a
        assert st is not None and (st.cpu().numpy()[:, 0] > 0).all()


def test_text_ingestion_to_signatures(tmp_path):
    """CLI-format text files -> CSR (native parser) -> GPU sketch == oracle."""
    from paper_1911_00675_b200.ingest import read_sets_csr
    rng = np.random.default_rng(8)
    srcs = []
    for s in range(6):
        n = int(rng.integers(1, 400))
        ids = rng.choice(2**40, size=n, replace=False)
        w = rng.exponential(size=n) + 1e-3
        lines = ["# set %d" % s] + [f"{hex(int(i)) if k % 3 == 0 else int(i)} {float(x)!r}"
                                    for k, (i, x) in enumerate(zip(ids, w))]
        p = tmp_path / f"s{s}.txt"
        p.write_text("\n".join(lines) + "\n")
        srcs.append(str(p))
    b = read_sets_csr(srcs)
    for algo in ("probminhash4", "pminhash"):
        sig, _ = sketch_batch(algo, to_device_u64(b.ids), to_device_f64(b.weights),
                              to_device_i64(b.offsets), 128)
        ref, _ = orc.sketch_csr(algo, 128, b.ids, b.weights, b.offsets)
        assert np.array_equal(sig.cpu().numpy().view(np.uint64), ref)


def test_host_multi_async_pipelined_batches():
    """Several pmh_sketch_csr_host_multi_async batches in flight (pinned host
    buffers, one stream) == the synchronous call, batch by batch."""
    import ctypes
    import torch
    from paper_1911_00675_b200 import _lib
    from paper_1911_00675_b200.batch import sketch_csr_multi
    L = _lib.load()
    algos = ["probminhash3", "pminhash", "probminhash2"]
    aids = (ctypes.c_int * len(algos))(*[_lib.ALG[a] for a in algos])
    batches = [datagen.random_sets(70 + k, list(np.exp(np.linspace(0, 8.5, 30)).astype(int) + 1),
                                   "uniform") for k in range(3)]
    keep, outs = [], []
    status = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    sp = ctypes.c_void_p(s.cuda_stream)
    _lib.check(L.pmh_status_reset(status.data_ptr(), sp))
    s.synchronize()
    for b in batches:
        h_ids = torch.from_numpy(b.ids.view(np.int64)).pin_memory()
        h_w = torch.from_numpy(b.weights).pin_memory()
        h_off = torch.from_numpy(b.offsets).pin_memory()
        o = [torch.empty((b.nsets, 128), dtype=torch.int64).pin_memory() for _ in algos]
        ptrs = (ctypes.c_void_p * len(algos))(*[t.data_ptr() for t in o])
        _lib.check(L.pmh_sketch_csr_host_multi_async(aids, len(algos), 128, h_ids.data_ptr(),
                                                     h_w.data_ptr(), h_off.data_ptr(), b.nsets,
                                                     b.nelems, ptrs, None, status.data_ptr(), sp))
        keep.append((h_ids, h_w, h_off, ptrs))
        outs.append(o)
    s.synchronize()
    err = ctypes.c_int64(-1)
    _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
    for b, o in zip(batches, outs):
        ref, _ = sketch_csr_multi(algos, 128, b.ids, b.weights, b.offsets)
        for got, r in zip(o, ref):
            assert np.array_equal(got.numpy().view(np.uint64), r)


def test_config2_shards_equal_full_batch():
    """The strong-scaling split (dist.shard_ranges_multi, what bench.py --gpus 8
    gives each rank) is exact: every shard computed alone equals its rows of
    the full configs[1] batch.  A shard is a small batch, so this also runs
    the small-batch split rule (sets cut at a quarter of the fair share) and
    the singleton-only warp-per-set path against the whole-batch schedule."""
    from paper_1911_00675_b200.dist import local_batch, shard_ranges_multi
    full = datagen.config2()
    variants = ["pminhash", "probminhash1", "probminhash2", "probminhash3", "probminhash4"]
    shards = shard_ranges_multi(full.offsets, 8, 1024, variants)
    ids, w, off = _dev(full)
    for algo in variants:
        whole = sigs_to_numpy(sketch_batch(algo, ids, w, off, 1024)[0])
        for s0, s1 in shards:
            b = local_batch(full, (s0, s1))
            part = sigs_to_numpy(sketch_batch(algo, *_dev(b), 1024)[0])
            assert np.array_equal(part, whole[s0:s1]), (algo, s0, s1)
