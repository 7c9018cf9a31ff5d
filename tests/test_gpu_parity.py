"""GPU parity: libpmh.so signatures vs the reference's golden vectors and vs
the CPU oracle, bit-exact (integer ids).  Calls go through the C ABI."""
import numpy as np
import pytest

from golden_io import config_cases, unweighted_cases, weighted_cases

pytestmark = pytest.mark.gpu

GPU_ALGOS = {"pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3",
             "probminhash3a", "probminhash4", "unweighted1", "unweighted1a", "unweighted2",
             "unweighted3", "unweighted3a", "unweighted4", "minhash", "superminhash", "oph"}


def _gpu_sig(algo, m, batch):
    from paper_1911_00675_b200 import sketch_batch
    from paper_1911_00675_b200.batch import (sigs_to_numpy, to_device_f64, to_device_i64,
                                             to_device_u64)
    ids = to_device_u64(batch.ids)
    w = to_device_f64(batch.weights) if batch.weights is not None else None
    off = to_device_i64(batch.offsets)
    sig, stats = sketch_batch(algo, ids, w, off, m)
    return sigs_to_numpy(sig), stats.cpu().numpy()


def _check(algo, m, batch, sig):
    if algo not in GPU_ALGOS:
        pytest.skip(f"{algo} not on the GPU path")
    got, _ = _gpu_sig(algo, m, batch)
    ok = np.ones(sig.shape[0], bool)
    if sig.shape[0] == batch.nsets:
        pass
    mism = (got[: sig.shape[0]] != sig)
    # rows the reference did not run (stats -1) are all-zero in the fixture
    ran = sig.any(axis=1) | (sig.shape[1] == 0)
    mism = mism[ran]
    assert mism.sum() == 0, f"{int(mism.sum())} of {mism.size} components differ"


@pytest.mark.parametrize("case", list(weighted_cases()), ids=lambda c: f"{c[0]}-m{c[1]}-{c[3]}")
def test_weighted_vs_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig)


@pytest.mark.parametrize("case", list(unweighted_cases()), ids=lambda c: f"{c[0]}-m{c[1]}-{c[3]}")
def test_unweighted_vs_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig)


@pytest.mark.parametrize("case", list(config_cases()), ids=lambda c: f"{c[0]}-{c[3]}")
def test_configs_vs_golden(case):
    key, m, batch, algo, sig, stats = case
    _check(algo, m, batch, sig)


@pytest.mark.parametrize("algo", ["pminhash", "probminhash1", "probminhash2", "probminhash3",
                                  "probminhash4"])
@pytest.mark.parametrize("dist", ["uniform", "pareto1.5", "wide"])
def test_random_vs_oracle(algo, dist):
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    rng = np.random.default_rng(hash((algo, dist)) & 0xFFFF)
    sizes = np.exp(rng.uniform(0, np.log(20000), 40)).astype(np.int64) + 1
    if algo == "pminhash":
        sizes = np.minimum(sizes, 2000)
    batch = datagen.random_sets(int(rng.integers(1 << 30)), sizes, dist)
    for m in (64, 1024):
        ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets, threads=8)
        got, _ = _gpu_sig(algo, m, batch)
        assert (got != ref).sum() == 0


@pytest.mark.parametrize("split_n,cap", [(256, 1024), (64, 3), (1024, 1)])
@pytest.mark.parametrize("algo", ["pminhash", "minhash"])
def test_pminhash_split_sets_vs_oracle(monkeypatch, split_n, cap, algo):
    """Large sets split across CTAs (partial minima merged with 128-bit global
    CAS) give the same signatures; with a small cap some large sets stay on
    the one-CTA path."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    monkeypatch.setenv("PMH_PM64_SPLIT_N", str(split_n))
    monkeypatch.setenv("PMH_PM64_SPLIT_CAP", str(cap))
    rng = np.random.default_rng(split_n + cap)
    sizes = np.concatenate([[5000, 3000, 1], rng.integers(1, 2500, 20)])
    batch = datagen.random_sets(int(rng.integers(1 << 30)), sizes, "pareto1.5")
    w = None if algo == "minhash" else batch.weights
    for m in (64, 1024):
        ref, _ = orc.sketch_csr(algo, m, batch.ids, w, batch.offsets, threads=8)
        got, _ = _gpu_sig(algo, m, batch)
        assert (got != ref).sum() == 0, (algo, m)


@pytest.mark.parametrize("cap", [1024, 2])
@pytest.mark.parametrize("algo", ["probminhash1", "probminhash2", "probminhash3", "probminhash4",
                                  "probminhash1a", "unweighted3", "unweighted4"])
def test_probminhash_split_sets_vs_oracle(monkeypatch, cap, algo):
    """ProbMinHash families with large sets split across CTAs (each part its
    own verified threshold, merged by 128-bit global CAS) == the oracle."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    monkeypatch.setenv("PMH_SPLIT_N", "64")
    monkeypatch.setenv("PMH_SPLIT_CAP", str(cap))
    rng = np.random.default_rng(cap + len(algo))
    sizes = np.concatenate([[6000, 2500, 1, 2], rng.integers(1, 3000, 16)])
    batch = datagen.random_sets(int(rng.integers(1 << 30)), sizes, "pareto1.5")
    w = None if algo.startswith("unweighted") else batch.weights
    for m in (64, 1024):
        ref, _ = orc.sketch_csr(algo, m, batch.ids, w, batch.offsets, threads=8)
        got, _ = _gpu_sig(algo, m, batch)
        assert (got != ref).sum() == 0, (algo, m)


def _edge_batch():
    from paper_1911_00675_b200.datagen import CSRBatch
    sets = [
        ([0, 2**64 - 1, 1, 2**63], [1.0, 1.0, 1.0, 1.0]),                # boundary ids
        ([5, 6, 7], [1e-300, 1.0, 1e300]),                                   # extreme weights
        ([11, 12], [5e-324, 2.0]),                                           # denormal weight
        ([21, 21, 22], [1.0, 3.0, 0.5]),                                     # duplicate id (validate=False)
        ([31], [123.456]),
        (list(range(100, 140)), list(np.geomspace(1e-12, 1e12, 40))),      # 24 decades
    ]
    ids = np.concatenate([np.array(i, np.uint64) for i, _ in sets])
    w = np.concatenate([np.array(x, np.float64) for _, x in sets])
    off = np.concatenate([[0], np.cumsum([len(i) for i, _ in sets])]).astype(np.int64)
    return CSRBatch(ids, w, off, "edge")


@pytest.mark.parametrize("algo", ["pminhash", "probminhash1", "probminhash1a", "probminhash2",
                                  "probminhash3", "probminhash3a", "probminhash4"])
@pytest.mark.parametrize("m", [1, 2, 63, 64, 1000, 4096])
def test_edge_inputs_vs_oracle(algo, m):
    """Boundary ids, extreme / denormal weights, duplicate ids and boundary m
    (1, 2, non-multiples of 64, 4096) give the oracle's signatures."""
    from oracle import oracle as orc
    if m < 2 and algo in ("probminhash3", "probminhash3a", "probminhash4"):
        pytest.skip("m >= 2 required")
    batch = _edge_batch()
    ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets)
    got, _ = _gpu_sig(algo, m, batch)
    assert (got != ref).sum() == 0


@pytest.mark.parametrize("algo", ["probminhash2", "probminhash4", "unweighted2", "unweighted4"])
@pytest.mark.parametrize("m", [2049, 3000, 4096, 4200, 5000, 6775])
def test_large_m_fisher_yates_16bit_maps_vs_oracle(algo, m):
    """Large m on 16-bit epoch maps (7 epochs, cleared on wrap: many wraps per
    set here): 2048 < m <= 4212 run 512-thread CTAs (sketch_use_big; 2049 and
    3000 are not powers of two), 4516 < m <= 6775 keep 256 threads with 16-bit
    maps (sketch_fy16_256; 6775 is the largest m that fits)."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    rng = np.random.default_rng(m)
    sizes = np.concatenate([[1, 2, 5, 17, 40], rng.integers(50, 400, 5)])
    batch = datagen.random_sets(int(rng.integers(1 << 30)), sizes, "pareto1.5")
    if algo.startswith("unweighted"):
        batch = type(batch)(batch.ids, None, batch.offsets, batch.name)
    ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets, threads=8)
    got, _ = _gpu_sig(algo, m, batch)
    assert (got != ref).sum() == 0


def test_large_m_limits():
    """Beyond the shared-memory slot table the C ABI refuses the call before
    any launch (InvalidParamsError), family by family."""
    from paper_1911_00675_b200 import InvalidParamsError
    from paper_1911_00675_b200 import datagen
    batch = datagen.random_sets(5, [3, 30], "exp")
    with pytest.raises(InvalidParamsError):
        _gpu_sig("probminhash2", 6776, batch)
    with pytest.raises(InvalidParamsError):
        _gpu_sig("probminhash1", 13841, batch)
    from oracle import oracle as orc
    # no Fisher-Yates map: fits, up to the largest m of the static families
    for algo, m in (("probminhash1", 6776), ("probminhash1", 13840), ("probminhash3", 13840)):
        got, _ = _gpu_sig(algo, m, batch)
        ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets)
        assert (got != ref).sum() == 0, (algo, m)


@pytest.mark.parametrize("algo", ["unweighted1", "unweighted2", "unweighted3", "unweighted4"])
@pytest.mark.parametrize("m,sizes", [
    (4096, (255, 256, 300, 520, 700, 800, 850, 900, 950, 1000, 1100, 1500, 4000)),
    (2048, (255, 256, 400, 450, 500, 600, 1000)),
    (1024, (250, 256, 300, 380, 420, 470, 520, 700, 1000, 3000)),
    (1000, (256, 300, 400, 500, 2000)),
])
def test_unweighted_lane_path_vs_oracle(algo, m, sizes):
    """Unweighted sets of >= 256 elements run lane-per-element with the
    Fisher-Yates families' per-lane hash maps (HashFY); the sizes straddle the
    set-size cutoff (256) and the point counts where a lane's map fills up and
    the element falls back to the warp path (~24 entries at m <= 1024, ~52 at
    larger m)."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    rep = np.repeat(np.asarray(sizes, np.int64), 3)
    st = datagen.CounterStream(1234 + m)
    ids = st.words(int(rep.sum()))
    off = np.concatenate([[0], np.cumsum(rep)]).astype(np.int64)
    batch = datagen.CSRBatch(ids, None, off, "uw-lane")
    ref, _ = orc.sketch_csr(algo, m, batch.ids, None, batch.offsets, threads=8)
    got, _ = _gpu_sig(algo, m, batch)
    assert (got != ref).sum() == 0


@pytest.mark.parametrize("algo", ["probminhash2", "probminhash4"])
@pytest.mark.parametrize("m", [512, 2048, 3000, 4096])
def test_weighted_fy_hash_maps_vs_oracle(algo, m):
    """Weighted Fisher-Yates families in the CTA kernel at signature sizes
    whose map regions hold 32 / 64 hash slots per lane, with and without the
    16-bit dense maps; equal weights inside a set make long lane sequences
    (the map fills, the element moves to the warp path)."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    rng = np.random.default_rng(m)
    sizes = np.concatenate([rng.integers(257, 3000, 12), [300, 600, 1200]]).astype(np.int64)
    batch = datagen.random_sets(77 + m, sizes, "uniform")
    w = batch.weights.copy()
    off = batch.offsets
    for s in range(0, len(sizes), 2):          # every other set: constant weights
        w[off[s]:off[s + 1]] = 0.5 + 0.01 * s
    batch = datagen.CSRBatch(batch.ids, w, off, "fy-hash")
    ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets, threads=8)
    got, _ = _gpu_sig(algo, m, batch)
    assert (got != ref).sum() == 0


@pytest.mark.parametrize("algo", ["probminhash1", "probminhash2", "probminhash3", "probminhash4",
                                  "unweighted3", "unweighted4"])
@pytest.mark.parametrize("m", [100, 128, 256])
def test_small_m_kernel_cutoffs_vs_oracle(algo, m):
    """m <= 256: sets around the warp-per-set / CTA-kernel cutoffs (128, 384 and
    512 elements, per family, pmh_kernel.cuh: small_n_for) and around the flat
    kernel's (255 for the unweighted family, 1024 otherwise)."""
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    sizes = np.array([1, 7, 100, 127, 128, 129, 254, 255, 256, 257, 383, 384, 385, 511, 512, 513,
                      600, 1023, 1024, 1025, 1500], np.int64)
    batch = datagen.random_sets(4242 + m, sizes, "exp")
    if algo.startswith("unweighted"):
        batch = type(batch)(batch.ids, None, batch.offsets, batch.name)
    ref, _ = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets, threads=8)
    got, _ = _gpu_sig(algo, m, batch)
    assert (got != ref).sum() == 0
