import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64
b = datagen.config2()
S, N, M = b.nsets, b.nelems, 1024
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((S, M), dtype=torch.int64, device="cuda")
status = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
main = torch.cuda.current_stream()
vs = ["probminhash1", "probminhash1a", "probminhash2", "probminhash3", "probminhash3a", "probminhash4"]
for NC in (1, 4):
    cut = [0] + [int(np.searchsorted(b.offsets, N * c // NC)) for c in range(1, NC)] + [S]
    streams = [torch.cuda.Stream() for _ in range(NC)]
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for c in range(NC):
            s = streams[c]; s.wait_event(e0)
            for v in vs:
                _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(), off.data_ptr() + 8 * cut[c], cut[c+1]-cut[c], sig.data_ptr() + 8 * M * cut[c], None, status.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
            ev = torch.cuda.Event(); ev.record(s); main.wait_event(ev)
        e1.record(main); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print("6 PMH variants NC", NC, "ms", round(min(ts[1:]), 2), flush=True)
