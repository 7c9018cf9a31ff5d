"""Device time of one variant over the whole batch vs NC set-chunks launched
on NC streams (data already resident): does chunking itself cost time?"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

v = sys.argv[1] if len(sys.argv) > 1 else "pminhash"
b = datagen.config2()
S, N, M = b.nsets, b.nelems, 1024
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((S, M), dtype=torch.int64, device="cuda")
status = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
main = torch.cuda.current_stream()
for NC, same in ((1, False), (2, False), (4, False), (2, True), (4, True), (8, True)):
    cut = [0] + [int(np.searchsorted(b.offsets, N * c // NC)) for c in range(1, NC)] + [S]
    streams = [torch.cuda.Stream() for _ in range(NC)]
    if same:
        streams = [streams[0]] * NC
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
        for c in range(NC):
            s = streams[c]
            s.wait_event(e0)
            ns = cut[c + 1] - cut[c]
            _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(),
                                              off.data_ptr() + 8 * cut[c], ns,
                                              sig.data_ptr() + 8 * M * cut[c], None,
                                              status.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(v, "NC", NC, "one stream" if same else "NC streams", "ms", round(min(ts[1:]), 2),
          flush=True)
