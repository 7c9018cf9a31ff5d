"""One sketch call on the first S sets of a BASELINE config (an ncu target):
python tools/ncu_driver_cfg.py <config fn, e.g. config3> <algo> <m> <S>"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

fn, algo, M, S = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
b = getattr(datagen, fn)()
b = b.subset(np.arange(min(S, b.nsets)))
ids, off = to_device_u64(b.ids), to_device_i64(b.offsets)
w = to_device_f64(b.weights) if b.weights is not None else None
sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.pmh_sketch_csr(_lib.ALG[algo], M, ids.data_ptr(), w.data_ptr() if w is not None else None,
                            off.data_ptr(), b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))
torch.cuda.synchronize()
print("ok", algo, b.nsets, b.nelems)
