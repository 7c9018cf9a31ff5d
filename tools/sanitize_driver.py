"""Small workload touching every kernel family and entry point, for
compute-sanitizer (memcheck): all variants incl. forced splits, the small-set
kernel, estimator/all-pairs/b-bit, the MSE cell and the async host entry."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen, sketch_batch  # noqa: E402
from paper_1911_00675_b200 import harness as H  # noqa: E402
from paper_1911_00675_b200.batch import (allpairs_bbit_hist_device, allpairs_hist_device,  # noqa: E402
                                         bbit_pack_device, count_equal_device, sketch_csr_multi,
                                         to_device_f64, to_device_i64, to_device_u64)

os.environ["PMH_SPLIT_N"] = "64"
os.environ["PMH_PM64_SPLIT_N"] = "256"
b = datagen.random_sets(5, [1, 2, 3, 7, 40, 300, 1500, 3000, 9], "pareto1.5")
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
for algo in ["pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3",
             "probminhash3a", "probminhash4", "minhash", "superminhash", "oph", "unweighted1",
             "unweighted2", "unweighted3", "unweighted4"]:
    for m in (64, 100, 1024):
        if algo in ("oph",) and m == 100:
            continue
        sig, _ = sketch_batch(algo, ids, w, off, m)
        torch.cuda.synchronize()
print("sketches ok")
sig, _ = sketch_batch("probminhash4", ids, w, off, 128)
cnt = count_equal_device(sig[0::2][:4].contiguous(), sig[1::2][:4].contiguous())
allpairs_hist_device(sig, threshold=1)
for bb in (1, 3, 8):
    allpairs_bbit_hist_device(bbit_pack_device(sig, bb), 128, bb, threshold=1)
print("estimators ok")
H.mse_cell_matches(H.ALGORITHM_IDS["probminhash2"], 64, *H.FIXTURES["skew4"].arrays(), 7, 50)
sketch_csr_multi(["probminhash3", "pminhash"], 64, b.ids, b.weights, b.offsets)
print("host entries ok")
