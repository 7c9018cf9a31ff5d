"""Per-call device time of one variant over many consecutive calls (looks for
outliers: a slow call would be a retry storm or scheduling pathology)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

v = sys.argv[1] if len(sys.argv) > 1 else "probminhash1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 60
b = datagen.config2()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, 1024), dtype=torch.int64, device="cuda")
st = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
evs = []
for r in range(reps):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], 1024, ids.data_ptr(), w.data_ptr(),
                                      off.data_ptr(), b.nsets, sig.data_ptr(), None,
                                      st.data_ptr(), sp))
    e.record()
    evs.append((a, e))
torch.cuda.synchronize()
t = np.array([a.elapsed_time(e) for a, e in evs])
print(v, "min %.2f median %.2f max %.2f (call %d)" % (t.min(), np.median(t), t.max(), t.argmax()),
      "slow calls:", [(i, round(x, 1)) for i, x in enumerate(t) if x > 2 * np.median(t)])
