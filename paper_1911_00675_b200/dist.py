"""Multi-GPU driver (one process per GPU, torch.distributed).

Sketching shards: sets are independent, so each rank sketches a contiguous
range of sets chosen to balance ESTIMATED COST (not element count): a
ProbMinHash set costs about n + m (ln m + 4) points (the coupon-collector
phase dominates small sets), a P-MinHash set n * m draws.  No collective is
needed on the sketch path.

All-pairs estimation (configs[4]) has one real exchange step: an all-gather
of the [N, m] signature matrix (NCCL over NVLink/NVSwitch on the GPU box),
then each rank computes a balanced share of upper-triangle block rows with
the tiled equal-component kernel and a histogram/threshold reduction; the
per-rank histograms are summed with one all_reduce.

Every compute step is a callable so the orchestration is testable on CPU
(gloo, world_size 2) with the oracle injected in tests; the defaults call
libpmh.so on the rank's GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def set_costs(offsets, m: int, algo: str) -> np.ndarray:
    sizes = np.diff(np.asarray(offsets, np.int64)).astype(np.float64)
    if algo in ("pminhash", "minhash"):
        return sizes * m
    return sizes + m * (math.log(m) + 4.0)


def shard_ranges(offsets, world: int, m: int = 1024, algo: str = "probminhash3"):
    """Contiguous set ranges [(s0, s1)] per rank with near-equal total cost
    (greedy split of the cumulative cost curve)."""
    return _split_cost(set_costs(offsets, m, algo), world)


def shard_ranges_multi(offsets, world: int, m: int, algos):
    """shard_ranges for a step that runs several algorithms over the same
    batch: the cost of a set is the sum of its per-algorithm costs."""
    costs = sum(set_costs(offsets, m, a) for a in algos)
    return _split_cost(costs, world)


def _split_cost(costs, world: int):
    S = costs.size
    if world <= 1 or S == 0:
        return [(0, S)]
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    total = cum[-1]
    bounds = [0]
    for r in range(1, world):
        b = int(np.searchsorted(cum, total * r / world, side="left"))
        bounds.append(min(max(b, bounds[-1]), S))
    bounds.append(S)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def local_batch(batch, rng):
    """Slice a CSRBatch to sets [s0, s1) with rebased offsets."""
    s0, s1 = rng
    a, b = int(batch.offsets[s0]), int(batch.offsets[s1])
    from .datagen import CSRBatch
    w = None if batch.weights is None else batch.weights[a:b]
    return CSRBatch(batch.ids[a:b], w, batch.offsets[s0:s1 + 1] - a, batch.name + f"[{s0}:{s1}]")


def _gpu_sketch(algo, m, batch):
    import torch
    from . import sketch_batch
    from .batch import to_device_f64, to_device_i64, to_device_u64
    ids = to_device_u64(batch.ids)
    w = to_device_f64(batch.weights) if batch.weights is not None else None
    off = to_device_i64(batch.offsets)
    sig, _ = sketch_batch(algo, ids, w, off, m, want_stats=False)
    torch.cuda.synchronize()
    return sig


def sketch_sharded(algo, m, batch, rank, world, sketch_fn=None):
    """Each rank sketches its cost-balanced range; returns (range, local sigs).
    No collective: signatures stay sharded."""
    rng = shard_ranges(batch.offsets, world, m, algo)[rank]
    fn = sketch_fn or _gpu_sketch
    return rng, fn(algo, m, local_batch(batch, rng))


# ---------------------------------------------------------------------------
# all-pairs
# ---------------------------------------------------------------------------

def block_rows(n: int, tile: int, world: int):
    """Balanced assignment of upper-triangle block rows to ranks: block row b
    has (nb - b) tiles; rows are dealt in a serpentine order so every rank
    gets a near-equal tile count."""
    nb = (n + tile - 1) // tile
    order = sorted(range(nb), key=lambda b: -(nb - b))
    loads = [0] * world
    assign = [[] for _ in range(world)]
    for b in order:
        r = min(range(world), key=lambda q: loads[q])
        assign[r].append(b)
        loads[r] += nb - b
    return [sorted(a) for a in assign]


@dataclass
class AllPairsResult:
    hist: np.ndarray          # int64[m+1]: number of pairs (i<j) with count c
    pairs: np.ndarray         # int64[K, 3]: (i, j, count) with count >= threshold
    tiles: int
    total: int = -1           # pairs with count >= threshold found (== len(pairs))
    rows: list = None         # [(r0, r1)]: the pair rows (smaller index) this rank covered


def allpairs_local(sigs_all, rows, tile, threshold, count_tile_fn):
    """Compute this rank's block rows: histogram + pairs above threshold.

    count_tile_fn(sigs_all, r0, r1, c0, c1) -> int array (r1-r0, c1-c0) of
    equal-component counts (only j > i entries are used)."""
    n, m = sigs_all.shape
    hist = np.zeros(m + 1, np.int64)
    found = []
    tiles = 0
    for b in rows:
        r0, r1 = b * tile, min(n, (b + 1) * tile)
        for c0 in range(r0, n, tile):
            c1 = min(n, c0 + tile)
            cnt = np.asarray(count_tile_fn(sigs_all, r0, r1, c0, c1))
            ii = np.arange(r0, r1)[:, None]
            jj = np.arange(c0, c1)[None, :]
            upper = jj > ii
            vals = cnt[upper].astype(np.int64)
            hist += np.bincount(vals, minlength=m + 1)[: m + 1]
            sel = upper & (cnt >= threshold)
            if sel.any():
                iw, jw = np.nonzero(sel)
                found.append(np.stack([iw + r0, jw + c0, cnt[sel]], axis=1).astype(np.int64))
            tiles += 1
    pairs = np.concatenate(found) if found else np.zeros((0, 3), np.int64)
    return AllPairsResult(hist, pairs, tiles, len(pairs),
                          [(b * tile, min(n, (b + 1) * tile)) for b in rows])


def _gpu_count_tile(sigs_all, r0, r1, c0, c1):
    from .batch import allpairs_tile_device
    out = allpairs_tile_device(sigs_all, r0, r1, c0, c1)
    return out.cpu().numpy().view(np.uint16)


def _gpu_rows_hist(sigs_all, rows, tile, threshold, cap=1 << 22):
    """This rank's block rows on the GPU with the fused histogram kernel.

    The kernel lists at most `cap` pairs per call but always returns the
    exact total k; a block row whose k exceeds the cap is recomputed with
    cap = k (into a fresh histogram, so nothing is counted twice), so the
    pair list is never truncated."""
    import torch
    from .batch import allpairs_hist_device
    n, m = sigs_all.shape
    hist = torch.zeros(m + 1, dtype=torch.int64, device=sigs_all.device)
    found = []
    total = 0
    for b in rows:
        r0, r1 = b * tile, min(n, (b + 1) * tile)
        h_b = torch.zeros(m + 1, dtype=torch.int64, device=sigs_all.device)
        _, pairs, k = allpairs_hist_device(sigs_all, r0, r1, r0, n, threshold, cap=cap, hist=h_b)
        if k > cap:
            h_b.zero_()
            _, pairs, k2 = allpairs_hist_device(sigs_all, r0, r1, r0, n, threshold, cap=k,
                                                hist=h_b)
            if k2 != k or len(pairs) != k:
                raise RuntimeError(f"all-pairs block row {b}: pair list {len(pairs)} != {k}")
        hist += h_b
        total += k
        found.append(pairs)
    pairs = np.concatenate(found) if found else np.zeros((0, 3), np.int64)
    return AllPairsResult(hist.cpu().numpy(), pairs, len(rows), total,
                          [(b * tile, min(n, (b + 1) * tile)) for b in rows])


def triangle_rows(n: int, world: int):
    """Contiguous row ranges [(r0, r1)] per rank with near-equal upper-triangle
    pair counts (row i holds n - 1 - i pairs)."""
    cum = np.concatenate([[0], np.cumsum(np.arange(n - 1, -1, -1, dtype=np.float64))])
    total = cum[-1]
    b = [0] + [int(np.searchsorted(cum, total * r / world, side="left")) for r in range(1, world)] + [n]
    for r in range(1, world + 1):
        b[r] = max(b[r], b[r - 1])
    return [(b[r], b[r + 1]) for r in range(world)]


def _gpu_rows_join(sigs_all, rank, world, threshold, cap=1 << 22):
    """This rank's contiguous triangle rows by the (component, value) hash join
    (pmh_allpairs_join_hist), one call; None if the join declines."""
    import torch
    from . import _lib
    from .batch import _pairs_out, _stream_ptr
    n, m = sigs_all.shape
    r0, r1 = triangle_rows(n, world)[rank]
    hist = torch.zeros(m + 1, dtype=torch.int64, device=sigs_all.device)
    while True:
        pairs = torch.empty((max(cap, 1), 2), dtype=torch.int64, device=sigs_all.device)
        cursor = torch.zeros(1, dtype=torch.int64, device=sigs_all.device)
        rc = _lib.load().pmh_allpairs_join_hist(
            sigs_all.data_ptr(), n, m, r0, r1, 0, n, int(threshold), hist.data_ptr(),
            pairs.data_ptr(), cap, cursor.data_ptr(), 0, _stream_ptr(torch, sigs_all.device))
        if rc == 1:
            return None
        _lib.check(rc)
        k = int(cursor.item())
        if k <= cap:
            break
        hist.zero_()
        cap = k          # the list overflowed: once more with room for all
    return AllPairsResult(hist.cpu().numpy(), _pairs_out(pairs, k, cap), 1, k, [(r0, r1)])


def _stamp(dev):
    import time
    if dev.type == "cuda":
        import torch
        torch.cuda.synchronize(dev)
    return time.perf_counter()


def allpairs_distributed(local_sigs, rank, world, tile=4096, threshold=1, group=None,
                         count_tile_fn=None, cap=1 << 22, ms=None, method="auto"):
    """All-gather the sharded signatures, compute this rank's block rows and
    all_reduce the histogram.  local_sigs: torch tensor [n_r, m] (int64, on
    the rank's device for NCCL; CPU for gloo).  Ranks may hold different row
    counts (padded for the all_gather).  `ms` (a dict), if given, receives
    this rank's device-synchronised milliseconds of the all-gather, the
    block-row compute and the histogram all_reduce."""
    import torch
    import torch.distributed as dist
    dev = local_sigs.device
    t0 = _stamp(dev)
    n_r = torch.tensor([local_sigs.shape[0]], device=local_sigs.device, dtype=torch.int64)
    sizes = [torch.zeros_like(n_r) for _ in range(world)]
    dist.all_gather(sizes, n_r, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    m = local_sigs.shape[1]
    pad = torch.zeros((mx, m), dtype=local_sigs.dtype, device=local_sigs.device)
    pad[: local_sigs.shape[0]] = local_sigs
    gathered = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(gathered, pad, group=group)
    sigs_all = torch.cat([g[:s] for g, s in zip(gathered, sizes)], dim=0)
    t1 = _stamp(dev)
    n = sigs_all.shape[0]
    rows = block_rows(n, tile, world)[rank]
    if count_tile_fn is None:
        res = None
        if method in ("join", "auto") and threshold >= 1:
            # contiguous triangle rows by the hash join (a few ms at configs[4]);
            # the dense block rows when the join declines
            res = _gpu_rows_join(sigs_all.contiguous(), rank, world, threshold, cap)
            if res is None and method == "join":
                raise RuntimeError("all-pairs join declined")
        if res is None:
            res = _gpu_rows_hist(sigs_all, rows, tile, threshold, cap)
    else:
        res = allpairs_local(sigs_all, rows, tile, threshold, count_tile_fn)
    t2 = _stamp(dev)
    h = torch.from_numpy(res.hist).to(local_sigs.device)
    dist.all_reduce(h, group=group)
    res.hist = h.cpu().numpy()
    t3 = _stamp(dev)
    if ms is not None:
        ms.update({"allgather": (t1 - t0) * 1e3, "block_rows": (t2 - t1) * 1e3,
                   "hist_allreduce": (t3 - t2) * 1e3})
    return res
