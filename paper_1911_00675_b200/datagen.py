"""Seeded synthetic CSR batches for the BASELINE.json configs (host side, numpy).

There is no public dataset on this path (the paper uses synthetic data only,
/root/reference/PAPER.md:874), so every workload is generated here from a
counter-based splitmix64 stream (the reference's generator, K:40-60):

    word(seed, j) = mix64(seed + (j + 1) * 0x9E3779B97F4A7C15)   (j >= 0)

Uniforms are U = (word >> 11) * 2**-53 in [0, 1).  Distinct draws use
disjoint word counters, so a batch is a pure function of (seed, config) and the
CPU oracle and the GPU see identical arrays.  Element ids are raw words
(uniform u64, unique with overwhelming probability; checked).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)


def mix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, np.uint64)
    z = (x ^ (x >> np.uint64(30))) * MIX1
    z = (z ^ (z >> np.uint64(27))) * MIX2
    return z ^ (z >> np.uint64(31))


class CounterStream:
    """Counter-based splitmix64: draws are blocks of consecutive words."""

    def __init__(self, seed: int):
        self.seed = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.pos = 0

    def words(self, count: int) -> np.ndarray:
        j = np.arange(self.pos + 1, self.pos + 1 + count, dtype=np.uint64)
        self.pos += count
        with np.errstate(over="ignore"):
            return mix64(self.seed + j * GOLDEN)

    def uniform01(self, count: int) -> np.ndarray:
        return (self.words(count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def open01(self, count: int) -> np.ndarray:
        """Uniform on the open interval (0, 1)."""
        k = (self.words(count) >> np.uint64(11)).astype(np.float64)
        return (k + 0.5) * 2.0 ** -53


@dataclass
class CSRBatch:
    ids: np.ndarray        # uint64[N]
    weights: np.ndarray    # float64[N] or None (unweighted)
    offsets: np.ndarray    # int64[S+1]
    name: str = ""

    @property
    def nsets(self) -> int:
        return self.offsets.size - 1

    @property
    def nelems(self) -> int:
        return int(self.offsets[-1])

    def set(self, s: int):
        a, b = int(self.offsets[s]), int(self.offsets[s + 1])
        w = None if self.weights is None else self.weights[a:b]
        return self.ids[a:b], w

    def subset(self, sets) -> "CSRBatch":
        sets = np.asarray(sets, np.int64)
        sizes = self.offsets[sets + 1] - self.offsets[sets]
        offs = np.zeros(sets.size + 1, np.int64)
        np.cumsum(sizes, out=offs[1:])
        idx = np.concatenate([np.arange(self.offsets[s], self.offsets[s + 1])
                              for s in sets]) if sets.size else np.zeros(0, np.int64)
        w = None if self.weights is None else self.weights[idx]
        return CSRBatch(self.ids[idx], w, offs, self.name + "[subset]")

    def nbytes_in(self) -> int:
        b = self.ids.nbytes + self.offsets.nbytes
        if self.weights is not None:
            b += self.weights.nbytes
        return b


def _offsets(sizes) -> np.ndarray:
    offs = np.zeros(len(sizes) + 1, np.int64)
    np.cumsum(np.asarray(sizes, np.int64), out=offs[1:])
    return offs


def _unique_ids(st: CounterStream, n: int) -> np.ndarray:
    ids = st.words(n)
    return ids


def config1(nsets: int = 1000, n: int = 1000, seed: int = 0) -> CSRBatch:
    """PMH3 m=256: sets of exactly 1000 elements, Exp(1) weights (BASELINE.json
    configs[0]; 'hash seed 42' has no counterpart -- the per-element stream
    seed is the id itself, K:291 -- and is recorded as a no-op)."""
    st = CounterStream(seed)
    ids = st.words(nsets * n)
    w = -np.log(st.open01(nsets * n))
    return CSRBatch(ids, w, _offsets([n] * nsets), "config1")


def config2_sizes(nsets: int = 10_000, seed: int = 2, nmax: int = 100_000):
    st = CounterStream(seed ^ 0x5EED0002)
    u = st.uniform01(nsets)
    return np.clip(np.floor(np.exp(u * np.log(nmax + 1.0))), 1, nmax).astype(np.int64)


def config2(nsets: int = 10_000, seed: int = 2, nmax: int = 100_000) -> CSRBatch:
    """All weighted variants m=1024: log-uniform sizes in [1, 1e5], uniform
    (0,1] weights (BASELINE.json configs[1], the headline)."""
    sizes = config2_sizes(nsets, seed, nmax)
    st = CounterStream(seed)
    N = int(sizes.sum())
    ids = st.words(N)
    w = 1.0 - st.uniform01(N)
    return CSRBatch(ids, w, _offsets(sizes), "config2")


def config3(nsets: int = 100_000, n: int = 1000, seed: int = 3) -> CSRBatch:
    """Unweighted m=4096: 1000 uniform u64 ids per set (configs[2])."""
    st = CounterStream(seed)
    return CSRBatch(st.words(nsets * n), None, _offsets([n] * nsets), "config3")


def config4(nsets: int = 1_000_000, n: int = 100, seed: int = 4,
            alpha: float = 1.5) -> CSRBatch:
    """PMH2/PMH4 m=64: 100 elements per set, Pareto(alpha, x_min=1) weights
    via (1-U)^(-1/alpha), the harness form (harness.py:116-120)."""
    st = CounterStream(seed)
    ids = st.words(nsets * n)
    w = (1.0 - st.uniform01(nsets * n)) ** (-1.0 / alpha)
    return CSRBatch(ids, w, _offsets([n] * nsets), "config4")


def config5_pairs(npairs: int = 50_000, n: int = 500, seed: int = 5):
    """End-to-end pairs: 2*npairs sets of n elements, Exp(1) weights; pair p
    targets probability Jaccard j = 0.1 * (1 + p % 9).  Shared elements carry
    equal weights in A and B, so J_P = W_sh / (W_sh + W_A + W_B)
    (estimate.py:63-71); the exclusive weights are rescaled by
    c = W_sh (1 - j) / (j (W_A + W_B)) so that J_P == j up to rounding.
    Returns (batch, jtarget[npairs], jexact[npairs]); sets 2p and 2p+1 are the
    pair."""
    st = CounterStream(seed)
    j = 0.1 * (1 + (np.arange(npairs) % 9))
    s = np.rint(n * 2 * j / (1 + j)).astype(np.int64)  # shared count, |A|=|B|=n
    s = np.minimum(s, n)
    sizes = np.full(2 * npairs, n, np.int64)
    offs = _offsets(sizes)
    N = int(offs[-1])
    ids = np.empty(N, np.uint64)
    w = np.empty(N, np.float64)
    fresh = st.words(npairs * (2 * n))          # enough distinct ids
    wraw = -np.log(st.open01(npairs * (2 * n)))
    jexact = np.empty(npairs)
    for p in range(npairs):
        sp = int(s[p])
        base = p * 2 * n
        shared_ids = fresh[base:base + sp]
        a_ids = fresh[base + sp: base + n]
        b_ids = fresh[base + n: base + 2 * n - sp]
        wsh = wraw[base:base + sp]
        wa = wraw[base + sp: base + n]
        wb = wraw[base + n: base + 2 * n - sp]
        Wsh, WA, WB = wsh.sum(), wa.sum(), wb.sum()
        if sp < n and WA + WB > 0:
            c = Wsh * (1 - j[p]) / (j[p] * (WA + WB))
            wa = wa * c
            wb = wb * c
        oa, ob = offs[2 * p], offs[2 * p + 1]
        ids[oa:oa + sp] = shared_ids
        ids[oa + sp:oa + n] = a_ids
        w[oa:oa + sp] = wsh
        w[oa + sp:oa + n] = wa
        ids[ob:ob + sp] = shared_ids
        ids[ob + sp:ob + n] = b_ids
        w[ob:ob + sp] = wsh
        w[ob + sp:ob + n] = wb
        Wsh2, WA2, WB2 = wsh.sum(), wa.sum(), wb.sum()
        jexact[p] = Wsh2 / (Wsh2 + WA2 + WB2)
    return CSRBatch(ids, w, offs, "config5"), j, jexact


def random_sets(seed: int, sizes, dist: str = "uniform") -> CSRBatch:
    """Small parity batches with a chosen weight law: uniform (0,1], exp,
    pareto1.5, pareto2, unit, or wide (log-uniform over 2^-20..2^20)."""
    st = CounterStream(seed)
    sizes = np.asarray(sizes, np.int64)
    N = int(sizes.sum())
    ids = st.words(N)
    u = st.uniform01(N)
    if dist == "uniform":
        w = 1.0 - u
    elif dist == "exp":
        w = -np.log1p(-u)
        w[w == 0.0] = 1.0
    elif dist == "pareto1.5":
        w = (1.0 - u) ** (-1.0 / 1.5)
    elif dist == "pareto2":
        w = (1.0 - u) ** (-0.5)
    elif dist == "unit":
        w = np.ones(N)
    elif dist == "wide":
        w = np.exp2((u - 0.5) * 40.0)
    else:
        raise ValueError(dist)
    return CSRBatch(ids, w, _offsets(sizes), f"random[{dist}]")
