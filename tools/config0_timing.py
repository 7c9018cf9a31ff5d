"""configs[0] (PMH3 / 3a, m = 256, 1000 x 1000) device time, repeated."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

b = datagen.config1()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, 256), dtype=torch.int64, device="cuda")
st = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for v in ("probminhash3", "probminhash3a", "probminhash3"):
    ts = []
    for r in range(6):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], 256, ids.data_ptr(), w.data_ptr(),
                                          off.data_ptr(), b.nsets, sig.data_ptr(), None,
                                          st.data_ptr(), sp))
        e.record()
        torch.cuda.synchronize()
        ts.append(round(a.elapsed_time(e), 3))
    print(v, ts, flush=True)
