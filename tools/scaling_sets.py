"""Time one variant on the first k sets of a size class of configs[1] for
several k (per-set latency vs throughput; development tool).
python tools/scaling_sets.py algo lo hi k1,k2,..."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

algo, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ks = [int(v) for v in sys.argv[4].split(",")]
M = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
full = datagen.config2()
sizes = np.diff(full.offsets)
sel = np.nonzero((sizes >= lo) & (sizes < hi))[0]
L = _lib.load()
err = ctypes.c_int64(-1)
for k in ks:
    b = full.subset(sel[:k])
    ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
    sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def run():
        _lib.check(L.pmh_sketch_csr(_lib.ALG[algo], M, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                    b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        a.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e))
    print(f"{algo} n in [{lo},{hi}) k={b.nsets:6d} ms={min(ts):8.3f}", flush=True)
