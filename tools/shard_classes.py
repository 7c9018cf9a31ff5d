"""Per-size-class time of one variant on the rank-0 shard of N (where a small
shard's time goes): python tools/shard_classes.py algo N"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402
from paper_1911_00675_b200.dist import local_batch, shard_ranges_multi  # noqa: E402

algo, N = sys.argv[1], int(sys.argv[2])
M = 1024
V = ["pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3", "probminhash3a",
     "probminhash4"]
full = datagen.config2()
sh = local_batch(full, shard_ranges_multi(full.offsets, N, M, V)[0])
sizes = np.diff(sh.offsets)
L = _lib.load()
err = ctypes.c_int64(-1)
edges = [1, 4, 16, 64, 256, 1024, 4096, 16384, 100001]


def t(b, reps=5):
    ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
    sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def run():
        _lib.check(L.pmh_sketch_csr(_lib.ALG[algo], M, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                    b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))
    run(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        a.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e))
    return min(ts)


print(f"{algo} shard 0/{N}: {sh.nsets} sets, whole shard {t(sh):.3f} ms")
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = np.nonzero((sizes >= lo) & (sizes < hi))[0]
    if sel.size:
        print(f"  n in [{lo:6d},{hi:6d}): {sel.size:4d} sets {t(sh.subset(sel)):.3f} ms", flush=True)
