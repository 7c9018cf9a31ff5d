"""Pin the C oracle restatement against golden vectors frozen from the live
reference (tests/golden/make_golden.py): signatures AND stats bit-exact."""
import numpy as np
import pytest

from golden_io import config_cases, load, unweighted_cases, weighted_cases
from oracle import oracle


def _check(algo, m, batch, sig, stats):
    ok = stats[:, 0] >= 0
    rsel = np.nonzero(ok)[0]
    sub = batch.subset(rsel) if not ok.all() else batch
    osig, ostats = oracle.sketch_csr(algo, m, sub.ids, sub.weights, sub.offsets)
    np.testing.assert_array_equal(osig, sig[rsel])
    np.testing.assert_array_equal(ostats, stats[rsel])


@pytest.mark.parametrize("case", list(weighted_cases()), ids=lambda c: f"{c[0]}-m{c[1]}-{c[3]}")
def test_weighted_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig, stats)


@pytest.mark.parametrize("case", list(unweighted_cases()), ids=lambda c: f"{c[0]}-m{c[1]}-{c[3]}")
def test_unweighted_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig, stats)


@pytest.mark.parametrize("case", list(config_cases()), ids=lambda c: f"{c[0]}-{c[3]}")
def test_config_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig, stats)


def test_stream_primitives_golden():
    z = load("primitives")
    for seed in [0, 1, 42, 2**63 + 5, 2**64 - 1]:
        np.testing.assert_array_equal(oracle.stream_words(seed, 257), z[f"words_{seed}"])
        np.testing.assert_array_equal(oracle.stream_uniform01(seed, 1000), z[f"u01_{seed}"])
        np.testing.assert_array_equal(oracle.stream_exp1(seed, 1000), z[f"exp1_{seed}"])
        for m in (3, 256, 1024, 4096):
            const = z[f"tconst_{m}"]
            lam = float(np.log1p(1.0 / (m - 1.0)))
            assert lam == const[0]
            np.testing.assert_array_equal(np.array(oracle.trunc_exp_consts(lam)), const[1:])
            np.testing.assert_array_equal(oracle.stream_trunc_exp(seed, lam, 2000),
                                          z[f"texp_{seed}_{m}"])


def test_bbit_golden():
    z = load("bbit")
    for b in (1, 2, 4, 8, 16):
        np.testing.assert_array_equal(oracle.bbit(z["sig"], b), z[f"bbit_{b}"])
