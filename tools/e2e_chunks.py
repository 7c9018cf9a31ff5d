import ctypes, sys, time, os
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen
from paper_1911_00675_b200.batch import to_device_u64, to_device_f64, to_device_i64
L = _lib.load()
b = datagen.config2()
S, N, M = b.nsets, b.nelems, 1024
h_ids = torch.from_numpy(b.ids.view(np.int64)).pin_memory()
h_w = torch.from_numpy(b.weights).pin_memory()
h_off = torch.from_numpy(b.offsets).pin_memory()
err = ctypes.c_int64(-1)
vs = sys.argv[1].split(",")
aids = (ctypes.c_int * len(vs))(*[_lib.ALG[v] for v in vs])
outs = [torch.empty((S, M), dtype=torch.int64).pin_memory() for _ in vs]
ptrs = (ctypes.c_void_p * len(vs))(*[o.data_ptr() for o in outs])
f = lambda: _lib.check(L.pmh_sketch_csr_host_multi(aids, len(vs), M, h_ids.data_ptr(), h_w.data_ptr(), h_off.data_ptr(), S, N, ptrs, None, ctypes.byref(err)))
f(); ts = []
for _ in range(3):
    t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
print(os.environ.get("PMH_H2D_CHUNKS"), vs[0], len(vs), "ms", round(min(ts) * 1e3, 1), flush=True)
