"""Quick per-algorithm GPU check (development helper; run under a timeout)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import oracle as orc  # noqa: E402
from paper_1911_00675_b200 import datagen, sketch_batch  # noqa: E402
from paper_1911_00675_b200.batch import sigs_to_numpy, to_device_f64, to_device_i64, to_device_u64  # noqa: E402

import torch  # noqa: E402

algos = sys.argv[1].split(",") if len(sys.argv) > 1 else [
    "pminhash", "probminhash1", "probminhash2", "probminhash3", "probminhash4",
    "unweighted3", "unweighted4", "minhash"]
for m in (2, 16, 1024):
    batch = datagen.random_sets(11, [1, 1, 2, 3, 5, 8, 13, 30, 64, 200, 3000], "uniform")
    ids, w, off = to_device_u64(batch.ids), to_device_f64(batch.weights), to_device_i64(batch.offsets)
    for algo in algos:
        t0 = time.time()
        sig, st = sketch_batch(algo, ids, w, off, m)
        torch.cuda.synchronize()
        t1 = time.time()
        ref, rst = orc.sketch_csr(algo, m, batch.ids, batch.weights, batch.offsets)
        got = sigs_to_numpy(sig)
        print(f"m={m} {algo}: {t1-t0:.3f}s mismatches={int((got != ref).sum())}/{got.size} "
              f"pts gpu={int(st[:,0].sum())} ref={int(rst[:,0].sum())}", flush=True)
