"""Run one variant once on (a subset of) the config-2 batch -- ncu target."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

v = sys.argv[1]
minn = int(sys.argv[2]) if len(sys.argv) > 2 else 0
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
M = int(sys.argv[4]) if len(sys.argv) > 4 else 1024
maxn = int(sys.argv[5]) if len(sys.argv) > 5 else 0
full = datagen.config2()
sizes = np.diff(full.offsets)
sel = (sizes >= minn) & ((sizes <= maxn) if maxn else True)
b = full.subset(np.nonzero(sel)[0]) if (minn or maxn) else full
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(reps):
    _lib.check(L.pmh_sketch_csr(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))
torch.cuda.synchronize()
print("ok", v, b.nsets, b.nelems)
