"""A/B timing of one variant on the config-2 batch for the library in
PMH_LIB_PATH (default: the in-tree libpmh.so); prints ms per call and a
signature checksum so builds can be compared for identical output.

    PMH_LIB_PATH=... python tools/pm_ab.py [variant] [reps] [m]
"""
import ctypes
import hashlib
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

v = sys.argv[1] if len(sys.argv) > 1 else "pminhash"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
M = int(sys.argv[3]) if len(sys.argv) > 3 else 1024
b = datagen.config2()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def call():
    _lib.check(L.pmh_sketch_csr(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))


call()
torch.cuda.synchronize()
times = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    call()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
h = hashlib.sha256(sig.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"{os.path.basename(os.environ.get('PMH_LIB_PATH', 'libpmh.so'))} {v} m={M} "
      f"min {min(times):.3f} ms median {float(np.median(times)):.3f} ms sig {h}")
