"""Statistical check of the estimator on the GPU (BASELINE.json configs[4]):
synthetic set pairs with known probability Jaccard J_P in {0.1, ..., 0.9},
ProbMinHash4 signatures at m = 256, equal-component estimates; the mean error
per J bucket must be ~0 (z-test with the reference's 4.9-sigma band,
test_acceptance.py:32) and the MSE must not exceed the independent-component
binomial variance J(1-J)/m by more than the band of harness.mse_sampling_sd
(harness.py:230-235).  All-pairs over the same signatures must find exactly
the designated pairs with their exact counts."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import datagen, jaccard_p_exact, sketch_batch
from paper_1911_00675_b200.batch import (allpairs_hist_device, count_equal_device, to_device_f64,
                                         to_device_i64, to_device_u64)

pytestmark = pytest.mark.gpu
Z_BAND = 4.9
M = 256


def _mse_sampling_sd(jp, m, s):
    var = (jp ** 2 * (1.0 - jp) ** 2 / (m * m * s) * (2.0 - 6.0 / m)
           + jp * (1.0 - jp) / (m ** 3 * s))
    return math.sqrt(max(var, 0.0))


@pytest.fixture(scope="module")
def pairs_run():
    npairs = 9 * 700
    b, jt, jx = datagen.config5_pairs(npairs=npairs, n=500, seed=55)
    sig, _ = sketch_batch("probminhash4", to_device_u64(b.ids), to_device_f64(b.weights),
                          to_device_i64(b.offsets), M)
    cnt = count_equal_device(sig[0::2].contiguous(), sig[1::2].contiguous()).cpu().numpy()
    return b, jt, jx, sig, cnt


def test_designed_jp_matches_definition(pairs_run):
    b, jt, jx, _, _ = pairs_run
    for p in (0, 4, 8, 13):
        ia, wa = b.set(2 * p)
        ib, wb = b.set(2 * p + 1)
        da = dict(zip(ia.tolist(), wa.tolist()))
        db = dict(zip(ib.tolist(), wb.tolist()))
        keys = sorted(set(da) | set(db))
        V = [(da.get(k, 0.0), db.get(k, 0.0)) for k in keys]
        assert jaccard_p_exact(V) == pytest.approx(jx[p], rel=1e-9)
        assert jx[p] == pytest.approx(jt[p], abs=0.01)


def test_estimator_mean_and_variance_per_bucket(pairs_run):
    _, jt, jx, _, cnt = pairs_run
    est = cnt / M
    for j in np.unique(np.round(jt, 1)):
        sel = np.isclose(jt, j)
        err = est[sel] - jx[sel]
        s = int(sel.sum())
        z = err.mean() / (err.std(ddof=1) / math.sqrt(s))
        assert abs(z) < Z_BAND, (j, z)
        jp = float(jx[sel].mean())
        mse = float((err ** 2).mean())
        ref = jp * (1 - jp) / M
        assert mse <= ref + Z_BAND * _mse_sampling_sd(jp, M, s), (j, mse, ref)


def test_gpu_signatures_equal_oracle_on_subset(pairs_run):
    b, _, _, sig, _ = pairs_run
    sub = b.subset(np.arange(0, 360))
    ref, _ = orc.sketch_csr("probminhash4", M, sub.ids, sub.weights, sub.offsets, threads=16)
    got = sig[:360].cpu().numpy().view(np.uint64)
    assert np.array_equal(got, ref)


def test_allpairs_finds_exactly_the_designed_pairs(pairs_run):
    _, _, _, sig, cnt = pairs_run
    n = sig.shape[0]
    hist, pairs, k = allpairs_hist_device(sig, threshold=1, cap=1 << 16)
    hist = hist.cpu().numpy()
    assert hist.sum() == n * (n - 1) // 2
    assert k == pairs.shape[0]
    got = {(int(i), int(j)): int(c) for i, j, c in pairs}
    exp = {(2 * p, 2 * p + 1): int(c) for p, c in enumerate(cnt) if c >= 1}
    assert got == exp
    assert hist[0] == n * (n - 1) // 2 - len(exp)


def test_allpairs_hist_vs_oracle_dense():
    rng = np.random.default_rng(3)
    sigs = rng.integers(0, 4, size=(333, 48)).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    import torch
    t = torch.from_numpy(sigs.view(np.int64)).cuda()
    hist, pairs, k = allpairs_hist_device(t, threshold=20, cap=1 << 20)
    full = orc.allpairs(sigs)
    iu = np.triu_indices(333, 1)
    np.testing.assert_array_equal(hist.cpu().numpy(), np.bincount(full[iu], minlength=49))
    exp = {(int(i), int(j)) for i, j in zip(*iu) if full[i, j] >= 20}
    assert {(int(i), int(j)) for i, j, _ in pairs} == exp
    # block-row split of the same matrix sums to the same histogram
    h2 = None
    for r0 in range(0, 333, 64):
        h2, _, _ = allpairs_hist_device(t, r0, min(333, r0 + 64), r0, 333, threshold=1000,
                                        hist=h2)
    np.testing.assert_array_equal(h2.cpu().numpy(), hist.cpu().numpy())


def _orc_hist(sigs):
    full = orc.allpairs(sigs)
    n, m = sigs.shape
    iu = np.triu_indices(n, 1)
    return full, iu, np.bincount(full[iu], minlength=m + 1)


def test_allpairs_low_word_collisions_are_recounted_exactly():
    """Two-stage exact all-pairs: components whose LOW 32 bits collide but
    whose high words differ must not count (stage 2 recounts candidates with
    64-bit compares)."""
    import torch
    rng = np.random.default_rng(11)
    n, m = 300, 40
    lo = rng.integers(0, 3, size=(n, m)).astype(np.uint64)          # heavy low-word collisions
    hi = rng.integers(0, 2, size=(n, m)).astype(np.uint64)          # ~half of them differ above
    sigs = (hi << np.uint64(32)) | lo
    t = torch.from_numpy(sigs.view(np.int64)).cuda()
    hist, pairs, k = allpairs_hist_device(t, threshold=15, cap=1 << 20)
    full, iu, exp_hist = _orc_hist(sigs)
    np.testing.assert_array_equal(hist.cpu().numpy(), exp_hist)
    exp = {(int(i), int(j)) for i, j in zip(*iu) if full[i, j] >= 15}
    assert {(int(i), int(j)) for i, j, _ in pairs} == exp and k == len(exp)


@pytest.mark.parametrize("ccap", ["1", "100"])
def test_allpairs_candidate_overflow_falls_back_exactly(monkeypatch, ccap):
    """A candidate list smaller than the candidates switches, on the device,
    to the single-stage exact reduction: same histogram and pairs."""
    import torch
    rng = np.random.default_rng(5)
    sigs = rng.integers(0, 4, size=(200, 32)).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15)
    t = torch.from_numpy(sigs.view(np.int64)).cuda()
    monkeypatch.setenv("PMH_ALLPAIRS_CCAP", ccap)
    hist, pairs, k = allpairs_hist_device(t, threshold=12, cap=1 << 20)
    full, iu, exp_hist = _orc_hist(sigs)
    np.testing.assert_array_equal(hist.cpu().numpy(), exp_hist)
    exp = {(int(i), int(j)) for i, j in zip(*iu) if full[i, j] >= 12}
    assert {(int(i), int(j)) for i, j, _ in pairs} == exp and k == len(exp)


def test_allpairs_threshold_zero_lists_every_pair():
    """thr <= 0 lists every pair, zero counts included (single-stage path)."""
    import torch
    rng = np.random.default_rng(6)
    sigs = rng.integers(0, 1 << 62, size=(90, 16)).astype(np.uint64)
    sigs[7] = sigs[3]
    t = torch.from_numpy(sigs.view(np.int64)).cuda()
    hist, pairs, k = allpairs_hist_device(t, threshold=0, cap=1 << 20)
    assert k == 90 * 89 // 2 and len(pairs) == k
    full, iu, exp_hist = _orc_hist(sigs)
    np.testing.assert_array_equal(hist.cpu().numpy(), exp_hist)
    assert {(int(i), int(j), int(c)) for i, j, c in pairs} == \
        {(int(i), int(j), int(full[i, j])) for i, j in zip(*iu)}
