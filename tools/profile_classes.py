"""Per-size-class kernel timing of the config-2 batch (development tool)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

M = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
variants = sys.argv[1].split(",") if len(sys.argv) > 1 else ["probminhash3"]
full = datagen.config2()
sizes = np.diff(full.offsets)
edges = [1, 4, 16, 64, 256, 1024, 4096, 16384, 100001]
L = _lib.load()
err = ctypes.c_int64(-1)
for v in variants:
    tot = 0.0
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = np.nonzero((sizes >= lo) & (sizes < hi))[0]
        if sel.size == 0:
            continue
        b = full.subset(sel)
        ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
        sig = torch.empty((b.nsets, M), dtype=torch.int64, device="cuda")
        st = torch.empty((b.nsets, 3), dtype=torch.int64, device="cuda")
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        def run():
            rc = L.pmh_sketch_csr(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                  b.nsets, sig.data_ptr(), st.data_ptr(), ctypes.byref(err), s)
            _lib.check(rc)
        run(); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            a.record(); run(); e.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(e))
        stn = st.cpu().numpy()
        t = min(ts); tot += t
        print(f"{v:14s} n in [{lo:6d},{hi:6d}): sets={b.nsets:5d} elems={b.nelems:9d} "
              f"ms={t:8.3f} (max {max(ts):8.3f}) pts/elt={stn[:,0].sum()/b.nelems:7.3f} "
              f"pts/set={stn[:,0].mean():9.1f}", flush=True)
    print(f"{v}: sum over classes {tot:.2f} ms", flush=True)
