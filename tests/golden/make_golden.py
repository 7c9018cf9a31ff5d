"""Freeze golden vectors from the LIVE reference (numba) implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py

The reference is imported read-only from /root/reference/pkg/src with numba's
cache and Python bytecode redirected away from the reference tree.  Outputs
(committed): tests/golden/*.npz.  Every array is produced by the reference's
own kernels (K = probminhash/_kernels.py) or its RandomStream (rng.py), never
by this repo's code; inputs come from this repo's seeded datagen (stored in
the fixture, so consumers never regenerate them).
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/pmh_numba_cache")
sys.dont_write_bytecode = True
REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))
sys.path.insert(0, REF_SRC)

import numpy as np  # noqa: E402

import probminhash as ref  # noqa: E402
from probminhash import _kernels as K  # noqa: E402

from paper_1911_00675_b200 import datagen  # noqa: E402

WEIGHTED = {
    "pminhash": K._k_pminhash, "probminhash1": K._k_probminhash1,
    "probminhash1a": K._k_probminhash1a, "probminhash2": K._k_probminhash2,
    "probminhash3": K._k_probminhash3, "probminhash3a": K._k_probminhash3a,
    "probminhash4": K._k_probminhash4,
}
UNWEIGHTED = {
    "unweighted3": K._k_uw_probminhash3, "unweighted3a": K._k_uw_probminhash3a,
    "unweighted4": K._k_uw_probminhash4,
}
MIN_M2 = {"probminhash3", "probminhash3a", "probminhash4", "unweighted3",
          "unweighted3a", "unweighted4", "superminhash"}


def _run_weighted(name, batch, m):
    S = batch.nsets
    sig = np.zeros((S, m), np.uint64)
    stats = np.zeros((S, 3), np.int64)
    for s in range(S):
        ids, w = batch.set(s)
        a, b = WEIGHTED[name](np.ascontiguousarray(ids),
                              np.ascontiguousarray(w), m)
        sig[s], stats[s] = a, b
    return sig, stats


def _run_unweighted(name, batch, m):
    S = batch.nsets
    sig = np.zeros((S, m), np.uint64)
    stats = np.zeros((S, 3), np.int64)
    for s in range(S):
        ids, _ = batch.set(s)
        ids = np.ascontiguousarray(ids)
        if name in ("unweighted1", "unweighted1a", "unweighted2"):
            kern = {"unweighted1": K._k_probminhash1,
                    "unweighted1a": K._k_probminhash1a,
                    "unweighted2": K._k_probminhash2}[name]
            a, b = kern(ids, np.ones(ids.size), m)
        elif name in UNWEIGHTED:
            a, b = UNWEIGHTED[name](ids, m)
        else:
            a = {"minhash": K._k_minhash, "superminhash": K._k_superminhash,
                 "oph": K._k_oph_densified}[name](ids, m)
            b = np.zeros(3, np.int64)
        sig[s], stats[s] = a, b
    return sig, stats


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1e3:.0f} kB)")


def weighted_cases():
    """Small and medium sets over every weight law, pow2 and non-pow2 m."""
    cases = []
    sizes_small = [1, 1, 2, 3, 5, 8, 13, 30, 64, 200]
    sizes_med = [1000, 3000]
    for mi, m in enumerate([2, 3, 16, 17, 64, 100, 256, 1024]):
        dists = ["uniform", "exp", "pareto1.5", "pareto2", "unit", "wide"]
        if m >= 1024:
            dists = dists[:3]
        for di, dist in enumerate(dists):
            sizes = list(sizes_small)
            if m >= 64 and di < 2:
                sizes += sizes_med
            seed = 1000 + 37 * mi + di
            cases.append((m, dist, datagen.random_sets(seed, sizes, dist)))
    return cases


def main():
    # 1) stream primitives from RandomStream (rng.py:43-124)
    prims = {}
    for seed in [0, 1, 42, 2**63 + 5, 2**64 - 1]:
        s = ref.RandomStream(seed)
        prims[f"words_{seed}"] = s.u64_batch(257)
        s = ref.RandomStream(seed)
        prims[f"u01_{seed}"] = s.uniform01_batch(1000)
        s = ref.RandomStream(seed)
        prims[f"exp1_{seed}"] = s.exp1_batch(1000)
        for m in (3, 256, 1024, 4096):
            lam = float(np.log1p(1.0 / (m - 1.0)))
            p = ref.TruncExpParams.from_rate(lam)
            s = ref.RandomStream(seed)
            prims[f"texp_{seed}_{m}"] = s.trunc_exp_batch(p, 2000)
            prims[f"tconst_{m}"] = np.array([p.lam, p.c1, p.c2, p.c3])
    save("primitives", **prims)

    # 2) weighted kernels over many laws and m
    arrays = {}
    for ci, (m, dist, batch) in enumerate(weighted_cases()):
        arrays[f"c{ci}_ids"] = batch.ids
        arrays[f"c{ci}_w"] = batch.weights
        arrays[f"c{ci}_off"] = batch.offsets
        arrays[f"c{ci}_m"] = np.array(m)
        for name in WEIGHTED:
            if m < 2 and name in MIN_M2:
                continue
            if name == "pminhash" and m >= 256 and batch.nelems > 1000:
                sub = batch.subset(np.arange(batch.nsets - 2))   # skip big sets
                sig, st = _run_weighted(name, sub, m)
                sig = np.concatenate([sig, np.zeros((2, m), np.uint64)])
                st = np.concatenate([st, -np.ones((2, 3), np.int64)])
            else:
                sig, st = _run_weighted(name, batch, m)
            arrays[f"c{ci}_{name}_sig"] = sig
            arrays[f"c{ci}_{name}_stats"] = st
    save("weighted", **arrays)

    # 3) unweighted specialisations and baselines
    arrays = {}
    for ci, m in enumerate([2, 3, 16, 64, 100, 1024, 4096]):
        sizes = [1, 2, 4, 9, 40, 300] + ([2000] if m <= 1024 else [1000])
        batch = datagen.random_sets(5000 + ci, sizes, "unit")
        arrays[f"u{ci}_ids"] = batch.ids
        arrays[f"u{ci}_off"] = batch.offsets
        arrays[f"u{ci}_m"] = np.array(m)
        names = ["unweighted1", "unweighted1a", "unweighted2", "unweighted3",
                 "unweighted3a", "unweighted4", "minhash", "superminhash", "oph"]
        for name in names:
            if m < 2 and name in MIN_M2:
                continue
            if name in ("minhash", "superminhash") and m >= 1024:
                continue
            sig, st = _run_unweighted(name, batch, m)
            arrays[f"u{ci}_{name}_sig"] = sig
            arrays[f"u{ci}_{name}_stats"] = st
    save("unweighted", **arrays)

    # 4) config-shaped subsets at the BASELINE sizes
    arrays = {}
    c1 = datagen.config1(nsets=20)
    sig, st = _run_weighted("probminhash3", c1, 256)
    arrays.update(c1_ids=c1.ids, c1_w=c1.weights, c1_off=c1.offsets,
                  c1_sig=sig, c1_stats=st)
    sizes = np.array([1, 7, 150, 1200, 9000])
    c2 = datagen.random_sets(20002, sizes, "uniform")
    arrays.update(c2_ids=c2.ids, c2_w=c2.weights, c2_off=c2.offsets)
    for name in WEIGHTED:
        sub = c2 if name != "pminhash" else c2.subset(np.arange(4))
        sig, st = _run_weighted(name, sub, 1024)
        arrays[f"c2_{name}_sig"] = sig
        arrays[f"c2_{name}_stats"] = st
    c4 = datagen.config4(nsets=300)
    for name in ("probminhash2", "probminhash4"):
        sig, st = _run_weighted(name, c4, 64)
        arrays[f"c4_{name}_sig"] = sig
        arrays[f"c4_{name}_stats"] = st
    arrays.update(c4_ids=c4.ids, c4_w=c4.weights, c4_off=c4.offsets)
    save("configs", **arrays)

    # 5) b-bit reduction (estimate.py:105-114 -> K:851-861)
    arrays = {}
    sig = datagen.CounterStream(77).words(4096)
    for b in (1, 2, 4, 8, 16):
        arrays[f"bbit_{b}"] = ref.bbit_reduce(ref.Signature(sig, sig.size), b).components
    arrays["sig"] = sig
    save("bbit", **arrays)


def main_mse():
    # 6) harness MSE cells (K:920-963 via harness.run_mse_cell, harness.py:266-280):
    # raw match counts per cell and the reference's finished MseRow values
    from probminhash import harness as H
    arrays = {}
    cells = []
    for algo in H.ALGORITHM_IDS:
        for fixture in ("skew2", "binary3", "tenth10", "binary64", "pareto16", "single1",
                        "disjoint2"):
            if algo in H.UNWEIGHTED_ALGORITHMS and fixture in ("skew2", "pareto16"):
                continue
            for m in (16, 64):
                cells.append((algo, m, fixture))
    for ci, (algo, m, fixture) in enumerate(cells):
        V = H.FIXTURES[fixture]
        wa, wb = V.arrays()
        seed = H.cell_seed(7, "mse", algo, m, fixture)
        s = 40
        arrays[f"m{ci}_matches"] = K._k_mse_cell(H.ALGORITHM_IDS[algo], m, wa, wb,
                                                 np.uint64(seed), s)
        arrays[f"m{ci}_key"] = np.array([algo, fixture])
        arrays[f"m{ci}_ms"] = np.array([m, s, seed], np.uint64)
        row = H.run_mse_cell(algo, m, fixture, s, 7)
        arrays[f"m{ci}_row"] = np.array([row.jp, row.mse, row.relative_mse, row.zscore])
    save("mse", **arrays)


INGEST_TEXT = (
    "# header comment\n\n17 0.5\n0x1F 2\n  0o17\t3e-3 trailing tokens\n0b101 inf\n"
    "1_000_000 1_0.25\n+42 .5\n0X_ff 7.\n18446744073709551615 1e308\n00 1\n"
    "   # indented comment\n9 -2.5\n10 nan\n0_0 2\n")


def main_ingest():
    # 7) CLI text ingestion (cli._read_weighted_lines, cli.py:60-70)
    from probminhash import cli
    import io
    entries = cli._read_weighted_lines(io.StringIO(INGEST_TEXT))
    save("ingest", text=np.array(INGEST_TEXT),
         ids=np.array([e for e, _ in entries], np.uint64),
         weights=np.array([w for _, w in entries], np.float64))


if __name__ == "__main__":
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    if only == "mse":
        main_mse()
    elif only == "ingest":
        main_ingest()
    else:
        main()
        main_mse()
        main_ingest()
