"""Break down the e2e path: raw pinned H2D/D2H bandwidth and host_multi timings."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen
L = _lib.load()
b = datagen.config2()
S, N, M = b.nsets, b.nelems, 1024
h_ids = torch.from_numpy(b.ids.view(np.int64)).pin_memory()
h_w = torch.from_numpy(b.weights).pin_memory()
h_off = torch.from_numpy(b.offsets).pin_memory()
d = torch.empty(N, dtype=torch.int64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h_ids, non_blocking=True); torch.cuda.synchronize()
print("H2D ids GB/s", h_ids.numel() * 8 / (time.perf_counter() - t) / 1e9)
hs = torch.empty((S, M), dtype=torch.int64).pin_memory()
ds = torch.empty((S, M), dtype=torch.int64, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); hs.copy_(ds, non_blocking=True); torch.cuda.synchronize()
print("D2H sig GB/s", hs.numel() * 8 / (time.perf_counter() - t) / 1e9)
err = ctypes.c_int64(-1)
def run(vs):
    aids = (ctypes.c_int * len(vs))(*[_lib.ALG[v] for v in vs])
    outs = [torch.empty((S, M), dtype=torch.int64).pin_memory() for _ in vs]
    ptrs = (ctypes.c_void_p * len(vs))(*[o.data_ptr() for o in outs])
    f = lambda: _lib.check(L.pmh_sketch_csr_host_multi(aids, len(vs), M, h_ids.data_ptr(), h_w.data_ptr(), h_off.data_ptr(), S, N, ptrs, None, ctypes.byref(err)))
    f(); ts = []
    for _ in range(3):
        t = time.perf_counter(); f(); ts.append(time.perf_counter() - t)
    print(vs, "ms", round(min(ts) * 1e3, 1))
run(["probminhash3"])
run(["pminhash"])
run(["probminhash1", "probminhash3"])
run(["pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3", "probminhash3a", "probminhash4"])
