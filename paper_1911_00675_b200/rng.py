"""Deterministic seeded 64-bit random stream (API surface of
/root/reference/pkg/src/probminhash/rng.py:20-128).

This is the user-facing stream utility, not the signature path: it restates
the splitmix64 stream with its LSB-first bit buffer (K:40-122) on the host in
exact integer arithmetic; Exp(1) uses the host libm log1p (the same glibc
call the reference reaches through numba).  The GPU kernels implement the
identical stream independently (csrc/pmh_device.cuh).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import InvalidParamsError, RandomnessFailureError

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_REJECT_CAP = 4096


def _mix64(x: int) -> int:
    z = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


@dataclass(frozen=True)
class TruncExpParams:
    """Constants for sampling Exp(lam) conditioned on [0,1) (rng.py:20-40)."""

    lam: float
    c1: float
    c2: float
    c3: float

    @classmethod
    def from_rate(cls, lam: float) -> "TruncExpParams":
        if not lam > 0.0:
            raise InvalidParamsError("rate must be positive")
        c1 = math.expm1(lam) / lam
        c2 = math.log(2.0 / (1.0 + math.exp(-lam))) / lam
        c3 = -math.expm1(-lam) / lam
        return cls(lam, c1, c2, c3)

    @property
    def fast_path_probability(self) -> float:
        return 1.0 / self.c1


class RandomStream:
    """Single-owner deterministic random stream; identical seeds give
    bit-identical sequences."""

    __slots__ = ("_s", "_buf", "_nb", "_words")

    def __init__(self, seed: int):
        self._s = seed & _MASK
        self._buf = 0
        self._nb = 0
        self._words = 0

    def next_u64(self) -> int:
        self._s = (self._s + _GOLDEN) & _MASK
        self._words += 1
        return _mix64(self._s)

    def _next_bits(self, k: int) -> int:
        if self._nb >= k:
            out = self._buf & ((1 << k) - 1)
            self._buf >>= k
            self._nb -= k
            return out
        out = self._buf
        w = self.next_u64()
        need = k - self._nb
        out |= (w & ((1 << need) - 1)) << self._nb
        self._buf = w >> need
        self._nb = 64 - need
        return out

    def next_uniform01(self) -> float:
        return float(self._next_bits(53)) * 1.1102230246251565e-16

    def next_uniform_int(self, n: int) -> int:
        if n < 1:
            raise InvalidParamsError("range size must be >= 1")
        if n <= 1:
            return 0
        k = (n - 1).bit_length()
        for _ in range(_REJECT_CAP + 1):
            r = self._next_bits(k)
            if r < n:
                return r
        raise RandomnessFailureError("uniform integer rejection loop exceeded its cap")

    def next_exp1(self) -> float:
        return -math.log1p(-self.next_uniform01())

    def next_trunc_exp(self, p: TruncExpParams, counters=None) -> float:
        if counters is not None:
            counters[0] += 1
        x = p.c1 * self.next_uniform01()
        if x < 1.0:
            if counters is not None:
                counters[1] += 1
            return x
        rounds = 0
        while True:
            x = self.next_uniform01()
            if x < p.c2:
                if counters is not None:
                    counters[2] += 1
                return x
            y = 0.5 * self.next_uniform01()
            if y > 1.0 - x:
                x = 1.0 - x
                y = 1.0 - y
            if x <= p.c3 * (1.0 - y):
                if counters is not None:
                    counters[3] += 1
                return x
            if y * p.c1 <= 1.0 - x:
                if counters is not None:
                    counters[4] += 1
                return x
            if counters is not None:
                counters[6] += 1
            if y * p.c1 * p.lam <= math.expm1(p.lam * (1.0 - x)):
                if counters is not None:
                    counters[5] += 1
                return x
            if counters is not None:
                counters[7] += 1
            rounds += 1
            if rounds > _REJECT_CAP:
                raise RandomnessFailureError(
                    "truncated exponential rejection loop exceeded its cap")

    def _words_np(self, count: int) -> np.ndarray:
        """The next `count` stream words (vectorised next_u64)."""
        k = np.arange(1, count + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            x = np.uint64(self._s) + k * np.uint64(_GOLDEN)
            z = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self._s = (self._s + count * _GOLDEN) & _MASK
        self._words += count
        return z

    def _bits53_np(self, count: int) -> np.ndarray:
        """`count` consecutive 53-bit draws of _next_bits(53), vectorised:
        draw i is bits [53 i, 53 i + 53) of (buffered bits, then whole words,
        LSB first)."""
        out = np.empty(count, np.uint64)
        if count == 0:
            return out
        i0 = 0
        if self._nb >= 53:           # the first draw fits the buffer
            out[0] = self._next_bits(53)
            i0 = 1
        if i0 == count:
            return out
        nb, buf = self._nb, self._buf
        need = 53 * (count - i0) - nb                 # bits to take from new words
        nw = -(-need // 64)
        w = np.concatenate([self._words_np(nw), np.zeros(1, np.uint64)])
        q = np.arange(count - i0, dtype=np.int64) * 53 - nb   # offset into the words
        first = q < 0                                  # straddles buffer and words
        qq = np.where(first, 0, q)
        wi, sh = qq >> 6, (qq & 63).astype(np.uint64)
        lo = w[wi] >> sh
        hi = np.where(sh > 0, w[wi + 1] << ((np.uint64(64) - sh) & np.uint64(63)), np.uint64(0))
        v = (lo | hi) & np.uint64((1 << 53) - 1)
        if first[0]:                                   # buffer bits + low bits of word 0
            v[0] = np.uint64((buf | ((int(w[0]) << nb) & _MASK)) & ((1 << 53) - 1))
        out[i0:] = v
        used = 53 * (count - i0) - nb                  # bits consumed from the new words
        rem = 64 * nw - used
        last = int(w[nw - 1])
        self._buf = last >> (64 - rem) if rem else 0
        self._nb = rem
        return out

    def uniform01_batch(self, count: int) -> np.ndarray:
        return self._bits53_np(count).astype(np.float64) * 1.1102230246251565e-16

    def uniform_int_batch(self, n: int, count: int) -> np.ndarray:
        return np.array([self.next_uniform_int(n) for _ in range(count)], np.int64)

    def exp1_batch(self, count: int) -> np.ndarray:
        return np.array([self.next_exp1() for _ in range(count)], np.float64)

    def trunc_exp_batch(self, p: TruncExpParams, count: int,
                        counters: np.ndarray | None = None) -> np.ndarray:
        if counters is None:
            counters = np.zeros(8, np.int64)
        return np.array([self.next_trunc_exp(p, counters) for _ in range(count)],
                        np.float64)

    def u64_batch(self, count: int) -> np.ndarray:
        # whole words; the bit buffer is left as it is (K:242-245)
        return self._words_np(count)

    @property
    def words_generated(self) -> int:
        return self._words

    @property
    def bits_buffered(self) -> int:
        return self._nb

    @property
    def bits_consumed(self) -> int:
        return 64 * self._words - self._nb


def new_stream(seed: int) -> RandomStream:
    return RandomStream(seed)
