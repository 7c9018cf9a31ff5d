"""One ProbMinHash4 m = 256 sketch call on the first S sets of the configs[4]
pair batch (an ncu target): python tools/ncu_driver_c5.py [S] [algo]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
algo = sys.argv[2] if len(sys.argv) > 2 else "probminhash4"
b, _, _ = datagen.config5_pairs()
b = b.subset(np.arange(min(S, b.nsets)))
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, 256), dtype=torch.int64, device="cuda")
st = torch.empty((b.nsets, 3), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.pmh_sketch_csr(_lib.ALG[algo], 256, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                            b.nsets, sig.data_ptr(), st.data_ptr(), ctypes.byref(err), s))
torch.cuda.synchronize()
stn = st.cpu().numpy()
print("ok", algo, b.nsets, b.nelems, "points/elt", stn[:, 0].sum() / b.nelems,
      "multi/elt", stn[:, 1].sum() / b.nelems)
