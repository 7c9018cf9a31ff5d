"""Randomised GPU-vs-oracle parity sweep (development tool; the committed
parity tests are in tests/): random signature sizes (powers of two and not),
set-size mixes and weight laws for every sketch family, bit-exact comparison.

    python tools/fuzz_parity.py [rounds] [seed]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as orc  # noqa: E402  (checker only)
from paper_1911_00675_b200 import datagen, sketch_batch  # noqa: E402
from paper_1911_00675_b200.batch import sigs_to_numpy, to_device_f64, to_device_i64, to_device_u64  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
W = ["probminhash1", "probminhash2", "probminhash3", "probminhash4"]
U = ["unweighted1", "unweighted2", "unweighted3", "unweighted4"]
MS = [2, 3, 16, 64, 65, 100, 128, 200, 256, 257, 512, 1000, 1024, 1500, 2048, 2049, 3000, 4096, 5000]
bad = 0
t0 = time.time()
for r in range(rounds):
    m = int(rng.choice(MS))
    k = int(rng.integers(6, 30))
    kind = rng.integers(0, 3)
    if kind == 0:      # log-uniform sizes
        sizes = np.exp(rng.uniform(0, np.log(6000), k)).astype(np.int64) + 1
    elif kind == 1:    # around the kernels' cutoffs
        sizes = rng.choice([1, 2, 3, 4, 7, 8, 127, 128, 129, 255, 256, 257, 383, 384, 385, 511, 512,
                            513, 1023, 1024, 1025], k).astype(np.int64)
    else:              # equal sizes (balanced lanes)
        sizes = np.full(k, int(rng.choice([260, 400, 700, 1000, 1800])), np.int64)
    dist = str(rng.choice(["uniform", "exp", "pareto1.5", "wide", "unit"]))
    batch = datagen.random_sets(int(rng.integers(1 << 30)), sizes, dist)
    ids, off = to_device_u64(batch.ids), to_device_i64(batch.offsets)
    wd = to_device_f64(batch.weights)
    for algo in W + U:
        if m < 2 and algo[-1] in "34":
            continue
        un = algo.startswith("unweighted")
        sig, _ = sketch_batch(algo, ids, None if un else wd, off, m)
        ref, _ = orc.sketch_csr(algo, m, batch.ids, None if un else batch.weights, batch.offsets,
                                threads=8)
        d = int((sigs_to_numpy(sig) != ref).sum())
        if d:
            bad += 1
            print(f"MISMATCH round {r} {algo} m={m} dist={dist} sizes={sizes.tolist()} diff={d}", flush=True)
print(f"fuzz: {rounds} rounds, {bad} mismatching cases, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
