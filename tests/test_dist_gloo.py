"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU driver's
host logic: cost-balanced sharding, sharded sketch reassembly, and the
all-gather + block-row all-pairs with an all_reduce'd histogram.  The GPU
compute steps are replaced by the CPU oracle (test infrastructure)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_1911_00675_b200 import datagen
from paper_1911_00675_b200 import dist as pdist
from paper_1911_00675_b200 import similarity as psim


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_sketch(algo, m, b):
    sig, _ = orc.sketch_csr(algo, m, b.ids, b.weights, b.offsets)
    return torch.from_numpy(sig.view(np.int64))


def _oracle_tile(sigs_all, r0, r1, c0, c1):
    s = sigs_all.numpy().view(np.uint64)
    a = s[r0:r1][:, None, :]
    b = s[c0:c1][None, :, :]
    return (a == b).sum(axis=2)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch = datagen.random_sets(3, [5, 40, 1, 300, 17, 2, 90, 12, 7, 33], "exp")
        m = 32
        rng, sig = pdist.sketch_sharded("probminhash4", m, batch, rank, world,
                                        sketch_fn=_oracle_sketch)
        res = pdist.allpairs_distributed(sig, rank, world, tile=3, threshold=1,
                                         count_tile_fn=_oracle_tile)
        q.put((rank, rng, sig.numpy().copy(), res.hist.copy(), res.pairs.copy(), res.tiles))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_balanced_and_complete():
    b = datagen.config2(nsets=2000)
    for world in (1, 2, 4, 8):
        rngs = pdist.shard_ranges(b.offsets, world, 1024, "probminhash3")
        assert rngs[0][0] == 0 and rngs[-1][1] == b.nsets
        assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
        c = pdist.set_costs(b.offsets, 1024, "probminhash3")
        loads = [c[a:z].sum() for a, z in rngs]
        assert max(loads) <= 1.15 * c.sum() / world + c.max()


def test_shard_ranges_multi_strong_scaling_split():
    """bench.py --scaling strong: one config-2 batch split for the 7-variant
    step; shards tile the batch and balance the summed per-variant cost."""
    b = datagen.config2(nsets=3000)
    algos = ["pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3",
             "probminhash3a", "probminhash4"]
    c = sum(pdist.set_costs(b.offsets, 1024, a) for a in algos)
    for world in (1, 2, 4, 8):
        rngs = pdist.shard_ranges_multi(b.offsets, world, 1024, algos)
        assert rngs[0][0] == 0 and rngs[-1][1] == b.nsets
        assert all(rngs[i][1] == rngs[i + 1][0] for i in range(world - 1))
        loads = [c[a:z].sum() for a, z in rngs]
        assert max(loads) <= c.sum() / world + c.max()
        parts = [pdist.local_batch(b, r) for r in rngs]
        assert sum(p.nelems for p in parts) == b.nelems
        assert np.array_equal(np.concatenate([p.ids for p in parts]), b.ids)


def test_block_rows_cover_triangle_balanced():
    for n, tile, world in ((1000, 64, 3), (100000, 4096, 8), (10, 3, 2)):
        rows = pdist.block_rows(n, tile, world)
        nb = (n + tile - 1) // tile
        assert sorted(sum(rows, [])) == list(range(nb))
        loads = [sum(nb - b for b in r) for r in rows]
        assert max(loads) - min(loads) <= nb


def test_gloo_world2_sharded_sketch_and_allpairs():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    batch = datagen.random_sets(3, [5, 40, 1, 300, 17, 2, 90, 12, 7, 33], "exp")
    m = 32
    ref, _ = orc.sketch_csr("probminhash4", m, batch.ids, batch.weights, batch.offsets)
    got = np.concatenate([o[2] for o in out]).view(np.uint64)
    np.testing.assert_array_equal(got, ref)
    # all-pairs: reduced histogram and union of pairs match a single-process pass
    full = orc.allpairs(ref)
    n = ref.shape[0]
    iu = np.triu_indices(n, 1)
    exp_hist = np.bincount(full[iu], minlength=m + 1)
    np.testing.assert_array_equal(out[0][3], exp_hist)
    np.testing.assert_array_equal(out[1][3], exp_hist)
    pairs = np.concatenate([o[4] for o in out])
    exp_pairs = {(int(i), int(j), int(full[i, j])) for i, j in zip(*iu) if full[i, j] >= 1}
    assert {tuple(map(int, p)) for p in pairs} == exp_pairs


def _pairs_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, jt, jx = datagen.config5_pairs(npairs=45, n=40, seed=9)
        res = psim.run_pairs(b, jt, jx, 16, rank, world, tile=8, sketch_fn=_oracle_sketch,
                             count_tile_fn=_oracle_tile)
        q.put((rank, res.summary(), res.hist.copy()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_pairs_pipeline_matches_single_process():
    """configs[4] pipeline (similarity.run_pairs): sharded sketch, all-gather,
    block rows, designed-pair statistics reduced over 2 ranks == one process."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pairs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    b, jt, jx = datagen.config5_pairs(npairs=45, n=40, seed=9)
    m = 16
    ref, _ = orc.sketch_csr("probminhash4", m, b.ids, b.weights, b.offsets)
    cnt = orc.count_equal(ref[0::2], ref[1::2])
    stats = psim.bucket_stats(psim.bucket_sums(jt, jx, cnt, m), m)
    full = orc.allpairs(ref)
    iu = np.triu_indices(ref.shape[0], 1)
    exp_hist = np.bincount(full[iu], minlength=m + 1)
    designed = {(2 * p, 2 * p + 1) for p in range(45)}
    extra = sum(1 for i, j in zip(*iu) if full[i, j] >= 1 and (i, j) not in designed)
    for rank, summ, hist in out:
        np.testing.assert_array_equal(hist, exp_hist)
        assert summ["extra_pairs"] == extra
        assert [bk["pairs"] for bk in summ["buckets"]] == [s.pairs for s in stats]
        for bk, s in zip(summ["buckets"], stats):
            assert bk["mean_err"] == pytest.approx(s.mean_err, abs=1e-12)
            assert bk["mse"] == pytest.approx(s.mse, rel=1e-12, abs=1e-15)


def test_bucket_stats_and_designed_counts():
    jt = np.array([0.1, 0.1, 0.5, 0.5, 0.5])
    jx = np.array([0.1, 0.12, 0.5, 0.49, 0.51])
    pairs = np.array([[0, 1, 2], [2, 3, 1], [4, 5, 8], [6, 7, 7], [8, 9, 9], [1, 4, 1]])
    counts, extra = psim.designed_counts(pairs, 0, 5)
    assert counts.tolist() == [2, 1, 8, 7, 9] and extra == 1
    st = psim.bucket_stats(psim.bucket_sums(jt, jx, counts, 16), 16)
    assert [s.pairs for s in st] == [2, 3]
    err = counts / 16 - jx
    assert st[0].mean_err == pytest.approx(err[:2].mean())
    assert st[1].mse == pytest.approx((err[2:] ** 2).mean())
    assert st[1].z_mean == pytest.approx(err[2:].mean() / (err[2:].std(ddof=1) / np.sqrt(3)))
    assert psim.two_sample_mse_z([0.1, -0.1, 0.2], [0.1, -0.1, 0.2]) == 0.0
