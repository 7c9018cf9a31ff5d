"""MSE-cell harness (harness.py:266-280 over K:920-963) without a GPU: the
oracle restatement of K._k_mse_cell against the live reference's match
counts (tests/golden/mse.npz), the Python mirror's seeding / statistics
against the reference's finished MseRow values, and argument validation."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import harness as H
from paper_1911_00675_b200.errors import InvalidParamsError
from paper_1911_00675_b200.estimate import jaccard_p_exact
from golden_io import load


def _cells():
    z = load("mse")
    ci = 0
    while f"m{ci}_matches" in z:
        algo, fx = (str(x) for x in z[f"m{ci}_key"])
        m, s, seed = (int(x) for x in z[f"m{ci}_ms"])
        yield algo, fx, m, s, seed, z[f"m{ci}_matches"], z[f"m{ci}_row"]
        ci += 1


CELLS = list(_cells())


def test_golden_covers_every_algorithm():
    assert {c[0] for c in CELLS} == set(H.ALGORITHM_IDS)
    assert len(CELLS) > 150


@pytest.mark.parametrize("cell", CELLS[::3], ids=lambda c: f"{c[0]}-{c[1]}-m{c[2]}")
def test_oracle_mse_cell_matches_reference(cell):
    algo, fx, m, s, seed, matches, _ = cell
    wa, wb = H.FIXTURES[fx].arrays()
    assert np.array_equal(orc.mse_cell(algo, m, wa, wb, seed, s), matches)


@pytest.mark.parametrize("cell", CELLS, ids=lambda c: f"{c[0]}-{c[1]}-m{c[2]}")
def test_row_statistics_match_reference(cell):
    algo, fx, m, s, seed, matches, row = cell
    assert H.cell_seed(7, "mse", algo, m, fx) == seed
    jp = jaccard_p_exact(H.FIXTURES[fx])
    assert jp == row[0]
    err = matches / m - jp
    mse = float(np.mean(err * err))
    assert mse == row[1]
    assert H._relative_mse(mse, jp, m) == row[2] or (math.isinf(row[2]))
    z = H.mse_zscore(mse, jp, m, s)
    assert z == row[3] or (math.isinf(z) and math.isinf(row[3]))


def test_generate_pair_round_trip():
    from paper_1911_00675_b200.rng import RandomStream
    for fx in ("skew4", "binary64", "pareto16"):
        V = H.FIXTURES[fx]
        A, B = H.generate_pair(V, RandomStream(3))
        assert sorted(H.pair_multiset(A, B).pairs) == sorted(V.pairs)


def test_generated_ids_are_the_cell_stream():
    """pair t, weight pair q -> word t*npairs + q of RandomStream(seed)."""
    from paper_1911_00675_b200.rng import RandomStream
    V = H.FIXTURES["binary8"]
    st = RandomStream(99)
    pairs = [H.generate_pair(V, st) for _ in range(3)]
    words = orc.stream_words(99, 3 * len(V))
    for t, (A, B) in enumerate(pairs):
        row = words[t * len(V):(t + 1) * len(V)]
        wa, wb = V.arrays()
        assert np.array_equal(A.ids, row[wa > 0])
        assert np.array_equal(B.ids, row[wb > 0])


def test_cell_validation():
    with pytest.raises(InvalidParamsError):
        H.run_mse_cell("probminhash3", 1, "binary3", 10, 0)
    with pytest.raises(InvalidParamsError):
        H.run_mse_cell("unweighted3", 16, "skew2", 10, 0)
    with pytest.raises(InvalidParamsError):
        H.run_mse_cell("nope", 16, "skew2", 10, 0)
    with pytest.raises(InvalidParamsError):
        H.ExperimentConfig(s=0)
    with pytest.raises(InvalidParamsError):
        H.ExperimentConfig(fixtures=("nope",))
    with pytest.raises(InvalidParamsError):  # native validation, before any device work
        H.mse_cell_matches(99, 16, [1.0], [1.0], 0, 4)
    with pytest.raises(InvalidParamsError):
        H.mse_cell_matches(1, 16, [1.0, 0.0], [1.0, 0.0, 2.0], 0, 4)
    with pytest.raises(InvalidParamsError):
        H.mse_cell_matches(1, 16, [0.0], [0.0], 0, 4)


def test_mse_csv_format():
    rows = [H.MseRow("probminhash1", 16, "skew2", 0.25, 0.0117, 1.0, -0.5, 40)]
    text = H.mse_csv(rows)
    assert text.splitlines()[0] == ",".join(H.MSE_COLUMNS)
    assert text.splitlines()[1] == "probminhash1,16,skew2,0.25,0.0117,1,-0.5,40"


def test_mse_cell_fails_loudly_without_cuda():
    """No CPU fallback for the cell either."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        H.run_mse_cell("probminhash1", 16, "skew2", 4, 0)


def test_timing_inputs_match_reference_stream():
    """The timing grid's inputs come from the same seeded stream as the
    reference's (harness.py:293-321): ids = whole words, weights = Pareto
    inverse CDF over the following 53-bit draws."""
    from paper_1911_00675_b200.rng import RandomStream
    dist = H.WeightDistributionSpec("pareto", 1.5)
    st = RandomStream(H.cell_seed(0, "timing", "probminhash4", 64, 7))
    ids, w = H._random_input(7, dist, st)
    ref = RandomStream(H.cell_seed(0, "timing", "probminhash4", 64, 7))
    exp_ids = np.array([ref.next_u64() for _ in range(7)], np.uint64)
    exp_w = np.array([(1.0 - ref.next_uniform01()) ** (-1.0 / 1.5) for _ in range(7)])
    assert np.array_equal(ids, exp_ids) and np.array_equal(w, exp_w)
    assert dist.name == "pareto(1,1.5)" and H.WeightDistributionSpec().name == "unweighted"
    with pytest.raises(InvalidParamsError):
        H.WeightDistributionSpec("zipf")
    with pytest.raises(InvalidParamsError):
        H.run_timing_experiment(H.ExperimentConfig())          # no n_values
    with pytest.raises(InvalidParamsError):
        H.run_buffer_experiment(H.ExperimentConfig(n_values=(10,)))
    assert H.timing_csv([H.TimingRow("pminhash", 16, 10, 12.5)]) == \
        "algorithm,m,n,mean_ns\npminhash,16,10,12.5\n"
