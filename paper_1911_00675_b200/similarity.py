"""End-to-end similarity over designed set pairs (BASELINE.json configs[4]).

The pipeline the reference runs one pair at a time -- sketch A and B
(`probminhash4`, sketch.py:161-166), then `estimate_similarity(sa, sb)`
(estimate.py:91-95) -- run over a whole batch on N GPUs:

  1. cost-balanced contiguous set shards, one per rank, sketched with no
     collective (dist.sketch_sharded);
  2. one NCCL all-gather of the [S, m] signature matrix, upper-triangle block
     rows dealt to ranks, the exact equal-component histogram of every pair
     and the list of pairs with count >= 1 (dist.allpairs_distributed; one
     all_reduce of the histogram);
  3. the designed pairs (2p, 2p+1) read out of each rank's pair list, and the
     per-J-bucket statistics reduced with one more all_reduce.

The statistics are the reference harness's (harness.py:230-245): per bucket
the mean error (Ĵ - J_P) with its z-score against 0, and the empirical MSE
against the binomial reference J(1-J)/m with the sampling band of
`mse_sampling_sd` (an upper reference: ProbMinHash4's components are
correlated and its MSE may lie below it).

Every compute step is injectable (sketch_fn / count_tile_fn), so the
orchestration runs under gloo on CPU in the tests with the oracle injected;
the defaults run libpmh.so on the rank's GPU.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import dist as pdist
from .harness import mse_sampling_sd

Z_BAND = 4.9   # the reference's acceptance band (test_acceptance.py:32)


@dataclass
class BucketStats:
    j: float           # target probability Jaccard of the bucket
    pairs: int
    jp_mean: float     # mean exact J_P over the bucket's pairs
    mean_err: float    # mean of (estimate - J_P)
    z_mean: float      # mean_err / (sd / sqrt(pairs))
    mse: float
    mse_binomial: float   # J(1-J)/m at jp_mean
    mse_band: float       # Z_BAND * mse_sampling_sd(jp_mean, m, pairs)

    @property
    def ok(self) -> bool:
        return abs(self.z_mean) < Z_BAND and self.mse <= self.mse_binomial + self.mse_band


@dataclass
class PairsRunResult:
    buckets: list
    m: int
    npairs: int
    extra_pairs: int            # non-designed pairs with >= 1 equal component
    hist: np.ndarray            # all-pairs histogram of equal-component counts
    ms: dict = field(default_factory=dict)   # stage -> max-over-ranks milliseconds

    @property
    def ok(self) -> bool:
        return all(b.ok for b in self.buckets)

    def summary(self) -> dict:
        return {
            "pairs": self.npairs, "m": self.m, "extra_pairs": self.extra_pairs,
            "all_pairs_total": int(self.hist.sum()), "ok": self.ok,
            "max_abs_z_mean": max(abs(b.z_mean) for b in self.buckets),
            "buckets": [{"j": round(b.j, 3), "pairs": b.pairs, "mean_err": b.mean_err,
                         "z_mean": b.z_mean, "mse": b.mse, "mse_binomial": b.mse_binomial,
                         "mse_band": b.mse_band} for b in self.buckets],
            "ms": self.ms,
        }


def bucket_sums(jtarget, jexact, counts, m: int, pair_ids=None):
    """Per-bucket partial sums [9, 4] = (pairs, sum J_P, sum err, sum err^2)
    over the designed pairs `pair_ids` (default: all); buckets are the
    targets 0.1 .. 0.9."""
    jt = np.asarray(jtarget)
    jx = np.asarray(jexact)
    c = np.asarray(counts, np.float64)
    sel = np.arange(jt.size) if pair_ids is None else np.asarray(pair_ids, np.int64)
    b = np.rint(jt[sel] * 10).astype(np.int64) - 1
    err = c[sel] / m - jx[sel]
    out = np.zeros((9, 4))
    np.add.at(out[:, 0], b, 1.0)
    np.add.at(out[:, 1], b, jx[sel])
    np.add.at(out[:, 2], b, err)
    np.add.at(out[:, 3], b, err * err)
    return out


def bucket_stats(sums, m: int):
    """BucketStats per non-empty bucket from reduced `bucket_sums`."""
    res = []
    for b in range(9):
        s, sj, se, se2 = sums[b]
        if s < 2:
            continue
        s_i = int(round(s))
        mean = se / s
        var = max(se2 / s - mean * mean, 0.0) * s / (s - 1)
        sd = math.sqrt(var)
        jp = sj / s
        mse = se2 / s
        res.append(BucketStats(
            j=0.1 * (b + 1), pairs=s_i, jp_mean=jp, mean_err=mean,
            z_mean=(mean / (sd / math.sqrt(s)) if sd > 0 else (0.0 if mean == 0 else math.inf)),
            mse=mse, mse_binomial=jp * (1.0 - jp) / m,
            mse_band=Z_BAND * mse_sampling_sd(jp, m, s_i)))
    return res


def designed_counts(pairs: np.ndarray, p0: int, p1: int):
    """Equal-component counts of the designed pairs p in [p0, p1) (sets 2p,
    2p+1) found in an all-pairs list (i, j, count); absent pairs count 0.
    Returns (counts [p1-p0], number of non-designed pairs in the list)."""
    counts = np.zeros(p1 - p0, np.int64)
    if len(pairs) == 0:
        return counts, 0
    i, j, c = pairs[:, 0], pairs[:, 1], pairs[:, 2]
    designed = (i % 2 == 0) & (j == i + 1)
    p = i // 2
    mine = designed & (p >= p0) & (p < p1)
    counts[p[mine] - p0] = c[mine]
    return counts, int((~designed).sum())


def _sync(device):
    if device is not None and getattr(device, "type", "cpu") == "cuda":
        import torch
        torch.cuda.synchronize(device)


def run_pairs(batch, jtarget, jexact, m: int, rank: int = 0, world: int = 1, group=None,
              algo: str = "probminhash4", tile: int = 4096, sketch_fn=None,
              count_tile_fn=None, method: str = "auto") -> PairsRunResult:
    """The configs[4] pipeline on this rank (every rank calls it with the same
    batch; ranks > 0 may pass world > 1 only inside an initialised process
    group).  Returns the reduced per-bucket statistics (identical on every
    rank) and the stage times (max over ranks, device-synchronised)."""
    import torch
    import torch.distributed as tdist

    npairs = len(jtarget)
    assert batch.nsets == 2 * npairs
    ms = {}

    def stage(name, fn, device=None):
        if world > 1:
            tdist.barrier(group=group)
        _sync(device)
        t0 = time.perf_counter()
        out = fn()
        _sync(device)
        dt = (time.perf_counter() - t0) * 1e3
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64,
                             device=device if device is not None else "cpu")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=group)
            dt = float(t.item())
        ms[name] = dt
        return out

    if sketch_fn is None:
        from . import sketch_batch
        from .batch import to_device_f64, to_device_i64, to_device_u64
        dev = torch.device("cuda", torch.cuda.current_device())
        rng = pdist.shard_ranges(batch.offsets, world, m, algo)[rank]
        lb = pdist.local_batch(batch, rng)
        d = stage("h2d", lambda: (to_device_u64(lb.ids), to_device_f64(lb.weights),
                                  to_device_i64(lb.offsets)), dev)
        local = stage("sketch", lambda: sketch_batch(algo, *d, m, want_stats=False)[0], dev)
    else:
        dev = None
        rng, local = stage("sketch", lambda: pdist.sketch_sharded(
            algo, m, batch, rank, world, sketch_fn=sketch_fn), dev)
    inner = {}
    res = stage("allpairs", lambda: pdist.allpairs_distributed(
        local, rank, world, tile=tile, threshold=1, group=group,
        count_tile_fn=count_tile_fn, ms=inner, method=method), dev)
    ms.update({"allpairs." + k: v for k, v in inner.items()})
    # each designed pair (2p, 2p+1) lies in exactly one block row; pairs of
    # the rows this rank computed are in its list
    counts, extra = designed_counts(res.pairs, 0, npairs)
    # the designed pairs whose first set lies in the rows this rank covered
    first = 2 * np.arange(npairs)
    mine = np.zeros(npairs, bool)
    for r0, r1 in res.rows:
        mine |= (first >= r0) & (first < r1)
    sums = bucket_sums(jtarget, jexact, counts, m, np.nonzero(mine)[0])
    red = np.concatenate([sums.ravel(), [float(extra)]])
    if world > 1:
        t = torch.from_numpy(red).to(local.device)
        tdist.all_reduce(t, group=group)
        red = t.cpu().numpy()
    sums = red[:-1].reshape(9, 4)
    return PairsRunResult(bucket_stats(sums, m), m, npairs, int(round(red[-1])), res.hist, ms)


def two_sample_mse_z(err_a, err_b) -> float:
    """Two-sample z of the mean squared errors of two independent samples:
    (MSE_a - MSE_b) / sqrt(var(e_a^2)/n_a + var(e_b^2)/n_b)."""
    qa = np.asarray(err_a, np.float64) ** 2
    qb = np.asarray(err_b, np.float64) ** 2
    se = math.sqrt(qa.var(ddof=1) / qa.size + qb.var(ddof=1) / qb.size)
    d = qa.mean() - qb.mean()
    return 0.0 if se == 0 and d == 0 else (d / se if se > 0 else math.inf)
