"""configs[4] end to end on the GPU through the multi-GPU code path
(dist.sketch_sharded / dist.allpairs_distributed / similarity.run_pairs with
their GPU defaults) under a real NCCL process group of world_size 1:

* the full-size workload: 50,000 designed pairs (100,000 sets of 500
  elements, Exp(1) weights), ProbMinHash4 at m = 256, NCCL all-gather,
  exact all-pairs histogram, per-J-bucket mean z-test and MSE band
  (harness.py:230-245, test_acceptance.py:32's 4.9 sigma);
* the GPU defaults of sketch_sharded / allpairs_distributed against the CPU
  oracle on a small batch;
* a two-sample test of the GPU estimator's per-bucket MSE against the CPU
  oracle's (K._k_probminhash4 restated) on an independent 2,000-pair sample
  (SURVEY.md §8d's second variance check)."""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import datagen
from paper_1911_00675_b200 import dist as pdist
from paper_1911_00675_b200 import similarity as psim

pytestmark = pytest.mark.gpu
M = 256


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    if not dist.is_initialized():
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                rank=0, world_size=1)
        own = True
    else:
        own = False
    assert dist.get_backend() == "nccl"
    yield
    if own:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def full_run(nccl_world1):
    b, jt, jx = datagen.config5_pairs(npairs=50_000, n=500, seed=5)
    res = psim.run_pairs(b, jt, jx, M, rank=0, world=1)
    return b, jt, jx, res


def test_config5_full_size_bucket_statistics(full_run):
    _, jt, _, res = full_run
    assert res.npairs == 50_000
    assert [b.pairs for b in res.buckets] == [int(np.isclose(jt, 0.1 * (k + 1)).sum())
                                              for k in range(9)]
    for b in res.buckets:
        assert abs(b.z_mean) < psim.Z_BAND, (b.j, b.z_mean)
        assert b.mse <= b.mse_binomial + b.mse_band, (b.j, b.mse, b.mse_binomial)
    assert res.ok
    n = 100_000
    assert int(res.hist.sum()) == n * (n - 1) // 2          # every pair counted once
    # unrelated sets share no ids, so a non-designed pair can only match by an
    # id collision: essentially none
    assert res.extra_pairs <= 10
    for k in ("h2d", "sketch", "allpairs", "allpairs.allgather", "allpairs.block_rows"):
        assert res.ms[k] >= 0.0


def test_gpu_defaults_of_sketch_sharded_and_allpairs_distributed(nccl_world1):
    batch = datagen.random_sets(21, [5, 40, 1, 300, 17, 2, 90, 12, 7, 33, 500, 64], "exp")
    m = 64
    rng, sig = pdist.sketch_sharded("probminhash4", m, batch, 0, 1)
    assert rng == (0, batch.nsets)
    ref, _ = orc.sketch_csr("probminhash4", m, batch.ids, batch.weights, batch.offsets)
    np.testing.assert_array_equal(sig.cpu().numpy().view(np.uint64), ref)
    res = pdist.allpairs_distributed(sig, 0, 1, tile=5, threshold=1)
    full = orc.allpairs(ref)
    iu = np.triu_indices(ref.shape[0], 1)
    np.testing.assert_array_equal(res.hist, np.bincount(full[iu], minlength=m + 1))
    exp_pairs = {(int(i), int(j), int(full[i, j])) for i, j in zip(*iu) if full[i, j] >= 1}
    assert {tuple(map(int, p)) for p in res.pairs} == exp_pairs
    assert res.total == len(exp_pairs)


def test_allpairs_pair_list_never_truncated(nccl_world1):
    """A block row with more listed pairs than the cap is recomputed
    (the list was silently cut at the cap)."""
    batch = datagen.random_sets(22, [30] * 40, "exp")
    # half the sets duplicated: many pairs with count >= 1
    ids = np.concatenate([batch.ids, batch.ids])
    w = np.concatenate([batch.weights, batch.weights])
    off = np.concatenate([batch.offsets, batch.offsets[1:] + batch.offsets[-1]])
    big = datagen.CSRBatch(ids, w, off, "dup")
    _, sig = pdist.sketch_sharded("probminhash3", 32, big, 0, 1)
    res_small = pdist.allpairs_distributed(sig, 0, 1, tile=16, threshold=1, cap=3)
    res_big = pdist.allpairs_distributed(sig, 0, 1, tile=16, threshold=1)
    assert res_small.total == res_big.total == len(res_small.pairs) >= 40
    np.testing.assert_array_equal(res_small.hist, res_big.hist)
    assert {tuple(p) for p in res_small.pairs.tolist()} == {tuple(p) for p in res_big.pairs.tolist()}


def test_two_sample_mse_gpu_vs_cpu_oracle(full_run):
    """GPU estimator MSE per bucket (50,000 pairs) vs the CPU oracle's
    ProbMinHash4 MSE on an independent 2,000-pair sample: two-sample z of the
    squared errors within the 4.9-sigma band."""
    from paper_1911_00675_b200 import sketch_batch
    from paper_1911_00675_b200.batch import count_equal_device, to_device_f64, to_device_i64, \
        to_device_u64
    b, jt, jx, _ = full_run
    sig, _ = sketch_batch("probminhash4", to_device_u64(b.ids), to_device_f64(b.weights),
                          to_device_i64(b.offsets), M, want_stats=False)
    cnt_gpu = count_equal_device(sig[0::2].contiguous(), sig[1::2].contiguous()).cpu().numpy()
    b2, jt2, jx2 = datagen.config5_pairs(npairs=2_000, n=500, seed=5005)
    ref, _ = orc.sketch_csr("probminhash4", M, b2.ids, b2.weights, b2.offsets,
                            threads=os.cpu_count() or 8)
    cnt_cpu = orc.count_equal(ref[0::2], ref[1::2])
    for k in range(9):
        j = 0.1 * (k + 1)
        sa = np.isclose(jt, j)
        sb = np.isclose(jt2, j)
        ea = cnt_gpu[sa] / M - jx[sa]
        eb = cnt_cpu[sb] / M - jx2[sb]
        z = psim.two_sample_mse_z(ea, eb)
        assert abs(z) < psim.Z_BAND, (j, z, (ea ** 2).mean(), (eb ** 2).mean())
