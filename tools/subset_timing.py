"""Per-variant device time of the config-2 batch vs the batch without its
smallest sets (how much of the overlapped step the tiny-set phase costs)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

full = datagen.config2()
sizes = np.diff(full.offsets)
L = _lib.load()
st = torch.cuda.current_stream()
sp = ctypes.c_void_p(st.cuda_stream)
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["probminhash1", "probminhash2",
                                                             "probminhash3", "probminhash4"]
for minn in (1, 4, 16, 64):
    b = full if minn == 1 else full.subset(np.nonzero(sizes >= minn)[0])
    ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
    sig = torch.empty((b.nsets, 1024), dtype=torch.int64, device="cuda")
    status = torch.zeros(2, dtype=torch.int64, device="cuda")
    out = []
    for v in variants:
        ts = []
        for rep in range(4):
            L.pmh_status_reset(status.data_ptr(), sp)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], 1024, ids.data_ptr(), w.data_ptr(),
                                              off.data_ptr(), b.nsets, sig.data_ptr(), None,
                                              status.data_ptr(), sp))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.append(f"{v}={min(ts[1:]):.2f}")
    print(f"n>={minn:3d} sets={b.nsets:5d}", " ".join(out), flush=True)
