"""The hash-join all-pairs path (pmh_allpairs_join_hist, csrc/pmh_join.cuh)
against the dense path (pmh_allpairs_hist) and the CPU oracle: same
histogram and same pair set, on random batches, designed pairs, duplicate-
heavy batches (long key lists), tile ranges, and the decline/fallback rule."""
import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import datagen, sketch_batch
from paper_1911_00675_b200.batch import (allpairs_hist_device, sigs_to_numpy, to_device_f64,
                                         to_device_i64, to_device_u64)

pytestmark = pytest.mark.gpu


def _sigs(batch, algo, m):
    sig, _ = sketch_batch(algo, to_device_u64(batch.ids), to_device_f64(batch.weights),
                          to_device_i64(batch.offsets), m, want_stats=False)
    return sig


def _both(sig, **kw):
    hd, pd, kd = allpairs_hist_device(sig, method="dense", **kw)
    hj, pj, kj = allpairs_hist_device(sig, method="join", **kw)
    return (hd.cpu().numpy(), {tuple(p) for p in pd.tolist()}, kd), \
           (hj.cpu().numpy(), {tuple(p) for p in pj.tolist()}, kj)


@pytest.mark.parametrize("thr", [1, 2, 40])
def test_join_equals_dense_and_oracle_designed_pairs(thr):
    b, _, _ = datagen.config5_pairs(npairs=900, n=120, seed=77)
    sig = _sigs(b, "probminhash4", 64)
    (hd, pd, kd), (hj, pj, kj) = _both(sig, threshold=thr)
    np.testing.assert_array_equal(hj, hd)
    assert pj == pd and kj == kd
    ref = orc.allpairs(sigs_to_numpy(sig))
    iu = np.triu_indices(ref.shape[0], 1)
    np.testing.assert_array_equal(hj, np.bincount(ref[iu], minlength=65))


def test_join_with_duplicates_and_ranges():
    b = datagen.random_sets(41, [30] * 60, "exp")
    # every set three times: keys shared by 3 sets, pairs with count m
    ids = np.concatenate([b.ids] * 3)
    w = np.concatenate([b.weights] * 3)
    off = np.concatenate([b.offsets[:-1] + k * b.offsets[-1] for k in range(3)] + [[3 * b.offsets[-1]]])
    big = datagen.CSRBatch(ids, w, off, "dup3")
    sig = _sigs(big, "probminhash2", 32)
    n = sig.shape[0]
    for rng in ((0, n, 0, n), (10, 70, 0, n), (0, 50, 60, 180), (33, 34, 0, n)):
        r0, r1, c0, c1 = rng
        (hd, pd, kd), (hj, pj, kj) = _both(sig, r0=r0, r1=r1, c0=c0, c1=c1, threshold=1)
        np.testing.assert_array_equal(hj, hd)
        assert pj == pd and kj == kd, rng


def test_join_declines_and_auto_falls_back():
    b = datagen.random_sets(42, [20] * 40, "uniform")
    ids = np.concatenate([b.ids] * 8)
    w = np.concatenate([b.weights] * 8)
    off = np.concatenate([b.offsets[:-1] + k * b.offsets[-1] for k in range(8)] + [[8 * b.offsets[-1]]])
    sig = _sigs(datagen.CSRBatch(ids, w, off, "dup8"), "probminhash1", 16)
    with pytest.raises(Exception):
        allpairs_hist_device(sig, method="join", max_visits=10)
    ha, pa, ka = allpairs_hist_device(sig, method="auto", max_visits=10)
    hd, pd, kd = allpairs_hist_device(sig, method="dense")
    np.testing.assert_array_equal(ha.cpu().numpy(), hd.cpu().numpy())
    assert ka == kd and {tuple(p) for p in pa.tolist()} == {tuple(p) for p in pd.tolist()}


def test_join_random_batch_many_components():
    b = datagen.random_sets(43, list(np.exp(np.linspace(0, 7, 300)).astype(int) + 1), "pareto1.5")
    sig = _sigs(b, "probminhash3", 256)
    (hd, pd, kd), (hj, pj, kj) = _both(sig, threshold=1)
    np.testing.assert_array_equal(hj, hd)
    assert pj == pd and kj == kd
