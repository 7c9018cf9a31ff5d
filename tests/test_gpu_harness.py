"""Fused MSE cell on the GPU (pmh_mse_cell, K:920-963): bit-exact match
counts against the live reference's (tests/golden/mse.npz) and the oracle,
finished rows equal to the reference's run_mse_cell, the chunked path, and
the statistical acceptance bands at scale."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as orc
from paper_1911_00675_b200 import harness as H
from test_harness_cpu import CELLS

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cell", CELLS, ids=lambda c: f"{c[0]}-{c[1]}-m{c[2]}")
def test_gpu_mse_cell_matches_reference(cell):
    algo, fx, m, s, seed, matches, row = cell
    wa, wb = H.FIXTURES[fx].arrays()
    assert np.array_equal(H.mse_cell_matches(H.ALGORITHM_IDS[algo], m, wa, wb, seed, s), matches)


@pytest.mark.parametrize("cell", CELLS[::5], ids=lambda c: f"{c[0]}-{c[1]}-m{c[2]}")
def test_gpu_run_mse_cell_row_equals_reference(cell):
    algo, fx, m, s, seed, matches, row = cell
    r = H.run_mse_cell(algo, m, fx, s, 7)
    got = np.array([r.jp, r.mse, r.relative_mse, r.zscore])
    assert np.array_equal(got, row) or all(
        a == b or (math.isinf(a) and math.isinf(b)) for a, b in zip(got, row))
    assert r.pairs == s and r.algorithm == algo and r.fixture == fx


@pytest.mark.parametrize("algo,m,fx", [("probminhash4", 256, "binary64"),
                                       ("pminhash", 64, "pareto16"),
                                       ("unweighted2", 1024, "tenth10"),
                                       ("superminhash", 64, "binary8")])
def test_gpu_mse_cell_vs_oracle_larger(algo, m, fx):
    wa, wb = H.FIXTURES[fx].arrays()
    seed = H.cell_seed(11, "mse", algo, m, fx)
    s = 600
    got = H.mse_cell_matches(H.ALGORITHM_IDS[algo], m, wa, wb, seed, s)
    assert np.array_equal(got, orc.mse_cell(algo, m, wa, wb, seed, s))


def test_gpu_mse_cell_chunked_equals_single():
    """PMH_MSE_CHUNK_PAIRS forces several generation/sketch/count chunks."""
    code = ("import numpy as np, sys; sys.path.insert(0, '.');"
            "from paper_1911_00675_b200 import harness as H;"
            "wa, wb = H.FIXTURES['skew4'].arrays();"
            "r = H.mse_cell_matches(6, 64, wa, wb, 12345, 1000);"
            "sys.stdout.write(','.join(map(str, r.tolist())))")
    env = dict(os.environ, PMH_MSE_CHUNK_PAIRS="97")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                         text=True, check=True).stdout
    chunked = np.array([int(x) for x in out.split(",")])
    wa, wb = H.FIXTURES["skew4"].arrays()
    assert np.array_equal(chunked, H.mse_cell_matches(6, 64, wa, wb, 12345, 1000))


Z_BAND = 4.9   # test_acceptance.py:36
SEED = 20191102


def test_gpu_criterion_01_unbiasedness_band():
    """test_acceptance.py:46-55: the default grid (independent-component
    algorithms x every fixture x m in 16/64/256, s = 2000) inside the band."""
    rows = H.run_mse_experiment(H.ExperimentConfig(seed=SEED))
    assert len(rows) == 4 * 3 * len(H.FIXTURES)
    worst = max(abs(r.zscore) for r in rows)
    assert worst <= Z_BAND, worst
    assert H.mse_csv(rows).count("\n") == len(rows) + 1


def test_gpu_criterion_02_correlated_variance_reduction():
    """test_acceptance.py:58-88 (PMH3 / PMH4 lower the MSE)."""
    from paper_1911_00675_b200.estimate import improvement_factor
    algos = ("probminhash3", "probminhash4")
    strong = [H.run_mse_cell(a, 256, f, 2000, SEED) for a in algos for f in ("skew2", "binary3")]
    weak = [H.run_mse_cell(a, 256, f, 20000, SEED) for a in algos
            for f in ("inverse2", "half2", "skew4")]
    degenerate = [H.run_mse_cell(a, 256, f, 2000, SEED) for a in algos
                  for f in ("single1", "disjoint2")]
    big = [H.run_mse_cell(a, 16, "binary64", 2000, SEED) for a in algos]
    alpha = improvement_factor(16, 64)
    worst_big = max(abs((r.mse - alpha * r.jp * (1 - r.jp) / 16)
                        / H.mse_sampling_sd(r.jp, 16, r.pairs)) for r in big)
    assert max(r.relative_mse for r in strong) < 0.85
    assert max(r.zscore for r in weak) <= -Z_BAND
    assert all(r.mse == 0.0 for r in degenerate)
    assert worst_big <= Z_BAND


def test_gpu_criterion_03_superminhash_variance_law():
    """test_acceptance.py:91-105."""
    from paper_1911_00675_b200.estimate import improvement_factor
    worst = 0.0
    for algo in ("superminhash", "unweighted4"):
        for m in (16, 64, 256):
            r = H.run_mse_cell(algo, m, "binary3", 2000, SEED)
            exp = improvement_factor(m, 3) * r.jp * (1 - r.jp) / m
            worst = max(worst, abs((r.mse - exp) / H.mse_sampling_sd(r.jp, m, r.pairs)))
    assert worst <= Z_BAND


def test_gpu_timing_experiment_rows():
    cfg = H.ExperimentConfig(algorithms=("probminhash3", "pminhash"), m_values=(64,),
                             n_values=(10, 1000), reps=50,
                             distribution=H.WeightDistributionSpec("pareto", 2.0))
    rows = H.run_timing_experiment(cfg)
    assert [(r.algorithm, r.m, r.n) for r in rows] == [
        ("probminhash3", 64, 10), ("probminhash3", 64, 1000), ("pminhash", 64, 10),
        ("pminhash", 64, 1000)]
    assert all(r.mean_ns > 0 for r in rows)
    assert H.timing_csv(rows).count("\n") == 5


def test_gpu_unweighted2_statistically_equivalent_to_minhash():
    """uw2 and MinHash estimate the same J: pooled match fractions agree
    (two-proportion z-test, the reference's test_sketch.py band)."""
    wa = np.array([1.0] * 6 + [0.0] * 2)
    wb = np.array([1.0] * 4 + [0.0, 0.0, 1.0, 1.0])
    m, s = 64, 4000
    ma = H.mse_cell_matches(H.ALGORITHM_IDS["unweighted2"], m, wa, wb, 5, s)
    mb = H.mse_cell_matches(H.ALGORITHM_IDS["minhash"], m, wa, wb, 6, s)
    pa, pb = ma.mean() / m, mb.mean() / m
    var = (ma / m).var() / s + (mb / m).var() / s
    assert abs(pa - pb) / math.sqrt(var) < Z_BAND


def test_gpu_criterion_11_bbit_calibration():
    """test_acceptance.py criterion 11: the b-bit estimator of P-MinHash
    signatures (m = 4096) is calibrated -- mean estimate within 0.01 of J_P
    for b = 1, 4, 8 over 2000 pairs of each fixture."""
    import torch
    from paper_1911_00675_b200 import sketch_batch
    from paper_1911_00675_b200.batch import (bbit_device, bbit_estimate, to_device_f64,
                                             to_device_i64, to_device_u64)
    from paper_1911_00675_b200.rng import RandomStream
    m, s = 4096, 2000
    worst = 0.0
    for fixture, jp in (("tenth10", 0.1), ("binary8", 0.5), ("ninety10", 0.9)):
        wa, wb = H.FIXTURES[fixture].arrays()
        sa_, sb_ = wa > 0, wb > 0
        st = RandomStream(H.cell_seed(SEED, "bbit", fixture))
        words = st.u64_batch(s * wa.size).reshape(s, wa.size)
        ids = np.concatenate([words[:, sa_].ravel(), words[:, sb_].ravel()])
        w = np.concatenate([np.tile(wa[sa_], s), np.tile(wb[sb_], s)])
        na, nb = int(sa_.sum()), int(sb_.sum())
        off = np.concatenate([np.arange(s + 1) * na, s * na + np.arange(1, s + 1) * nb])
        sig, _ = sketch_batch("pminhash", to_device_u64(ids), to_device_f64(w),
                              to_device_i64(off.astype(np.int64)), m, want_stats=False)
        for b in (1, 4, 8):
            r = bbit_device(sig, b)
            c = (r[:s] == r[s:]).sum(dim=1).cpu().numpy()
            worst = max(worst, abs(float(bbit_estimate(c, m, b).mean()) - jp))
        del sig
        torch.cuda.empty_cache()
    assert worst < 0.01, worst
