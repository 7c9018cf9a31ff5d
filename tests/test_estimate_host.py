"""Host-side estimator utilities of the API mirror (estimate.py:20-178):
exact Jaccard oracles, the b-bit estimator, alpha(m, u) and the variance
formulas, checked against exact rational arithmetic and their defining
properties (the reference's test_estimate.py / acceptance criterion 10
cover the same ground)."""
import math
from fractions import Fraction

import numpy as np
import pytest

from paper_1911_00675_b200 import (BBitSignature, Signature, WeightPairMultiset, bbit_reduce,
                                   estimate_similarity, estimate_similarity_bbit,
                                   estimator_variance, improvement_factor, jaccard_exact,
                                   jaccard_n_exact, jaccard_p_exact, jaccard_w_exact,
                                   superminhash_variance)
from paper_1911_00675_b200.errors import InvalidParamsError


def _jp_fraction(pairs):
    """J_P by its definition with exact rationals: sum over shared d of
    1 / sum_e max(a_e / a_d, b_e / b_d)."""
    total = Fraction(0)
    for a_d, b_d in pairs:
        if a_d == 0 or b_d == 0:
            continue
        denom = sum(max(Fraction(a_e) / Fraction(a_d), Fraction(b_e) / Fraction(b_d))
                    for a_e, b_e in pairs)
        total += 1 / denom
    return total


def test_multiset_validation():
    for bad in ([], [(0, 0)], [(2, -1)], [(-1, 1)]):
        with pytest.raises(InvalidParamsError):
            WeightPairMultiset(bad)


@pytest.mark.parametrize("pairs", [
    [(1, 1)], [(1, 0), (0, 1)], [(1, 2), (2, 1)], [(4, 1), (1, 4), (2, 2)],
    [(3, 20), (30, 7)], [(1, 1), (1, 0)], [(5, 5), (1, 0), (0, 3), (2, 7)]])
def test_jaccard_p_equals_exact_rationals(pairs):
    assert jaccard_p_exact(pairs) == pytest.approx(float(_jp_fraction(pairs)), rel=1e-12)


def test_jaccard_exact_and_binary_coincidence():
    assert jaccard_exact({1, 2, 3}, {2, 3, 4}) == pytest.approx(0.5)
    with pytest.raises(InvalidParamsError):
        jaccard_exact(set(), set())
    rng = np.random.default_rng(1)
    for _ in range(300):
        n = int(rng.integers(1, 15))
        pairs = [[(1, 0), (0, 1), (1, 1)][int(k)] for k in rng.integers(0, 3, n)]
        A = {i for i, (a, _) in enumerate(pairs) if a}
        B = {i for i, (_, b) in enumerate(pairs) if b}
        j = jaccard_exact(A, B)
        assert jaccard_w_exact(pairs) == pytest.approx(j, abs=1e-12)
        assert jaccard_p_exact(pairs) == pytest.approx(j, abs=1e-12)
        if len(A) == len(B):
            assert jaccard_n_exact(pairs) == pytest.approx(j, abs=1e-12)


def test_scale_invariance_symmetry_range():
    rng = np.random.default_rng(2)
    for _ in range(300):
        n = int(rng.integers(1, 20))
        pairs = [(float(a), float(b)) for a, b in np.exp(rng.uniform(-5, 5, (n, 2)))]
        ca, cb = np.exp(rng.uniform(-5, 5, 2))
        scaled = [(a * ca, b * cb) for a, b in pairs]
        swapped = [(b, a) for a, b in pairs]
        for f in (jaccard_p_exact, jaccard_n_exact):
            assert f(scaled) == pytest.approx(f(pairs), rel=1e-9, abs=1e-12)
        for f in (jaccard_p_exact, jaccard_w_exact, jaccard_n_exact):
            v = f(pairs)
            assert -1e-12 <= v <= 1 + 1e-12
            assert f(swapped) == pytest.approx(v, rel=1e-12)


@pytest.mark.gpu
def test_estimate_similarity_and_bbit():
    sig = lambda v: Signature(np.array(v, np.uint64), len(v))  # noqa: E731
    assert estimate_similarity(sig([9, 8, 7]), sig([9, 1, 7])) == pytest.approx(2 / 3)
    with pytest.raises(InvalidParamsError):
        estimate_similarity(sig([1, 2]), sig([1, 2, 3]))
    r = bbit_reduce(sig(list(range(200))), 2)
    assert r.components.min() >= 0 and r.components.max() <= 3
    for bad in (0, 17):
        with pytest.raises(InvalidParamsError):
            bbit_reduce(sig([1]), bad)
    m, b = 32, 5
    a = np.zeros(m, np.int64)
    c = np.ones(m, np.int64)
    c[0] = 0                                   # 1 / 32 = 2^-5 matching -> estimate 0
    assert estimate_similarity_bbit(BBitSignature(a, b, m), BBitSignature(c, b, m)) == 0.0
    assert estimate_similarity_bbit(BBitSignature(a, b, m), BBitSignature(a, b, m)) == 1.0
    with pytest.raises(InvalidParamsError):
        estimate_similarity_bbit(BBitSignature(a, b, m), BBitSignature(a, 4, m))


def _alpha_rational(m, u):
    # alpha(m, u) = 1 - sum_{l=1}^{m-1} l^u ((l+1)^u + (l-1)^u - 2 l^u)
    #                   / ((m-1)^(u-1) m^u (u-1))        (SuperMinHash variance factor)
    s = sum(Fraction(l ** u * ((l + 1) ** u + (l - 1) ** u - 2 * l ** u)) for l in range(1, m))
    return 1 - s / Fraction((m - 1) ** (u - 1) * m ** u * (u - 1))


@pytest.mark.parametrize("m,u", [(2, 2), (3, 5), (16, 3), (64, 9), (100, 2), (17, 31)])
def test_improvement_factor_matches_rational(m, u):
    assert improvement_factor(m, u) == pytest.approx(float(_alpha_rational(m, u)), rel=1e-9)


def test_improvement_factor_limits_and_variance():
    for m in (2, 64, 1024):
        assert improvement_factor(m, 2) == pytest.approx(1 - (2 * m - 1) / (3 * m), rel=1e-12)
    assert 0.99 < improvement_factor(64, 10 ** 6) <= 1.0
    assert improvement_factor(8, 4096) > 0.99
    for bad in ((1, 2), (2, 1), (0, 5)):
        with pytest.raises(InvalidParamsError):
            improvement_factor(*bad)
    assert estimator_variance(0.25, 50) == pytest.approx(0.25 * 0.75 / 50)
    assert estimator_variance(1.0, 7) == 0.0
    assert superminhash_variance(0.3, 64, 5) == pytest.approx(
        0.3 * 0.7 / 64 * improvement_factor(64, 5))
    assert not math.isnan(superminhash_variance(0.5, 2, 2))
