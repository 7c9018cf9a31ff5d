"""The asynchronous entry (pmh_sketch_csr_w_async, W given) timed K times
back to back, signatures compared with the first call each time."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "pminhash"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 16
given = (sys.argv[3] if len(sys.argv) > 3 else "1") == "1"
b = datagen.config2()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
S = b.nsets
sig = torch.empty((S, 1024), dtype=torch.int64, device="cuda")
setw = torch.empty(S, dtype=torch.float64, device="cuda")
status = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
_lib.check(L.pmh_status_reset(status.data_ptr(), sp))
_lib.check(L.pmh_set_weights(w.data_ptr(), off.data_ptr(), S, setw.data_ptr(), sp))


def run():
    _lib.check(L.pmh_sketch_csr_w_async(_lib.ALG[algo], 1024, ids.data_ptr(), w.data_ptr(),
                                        off.data_ptr(), S, setw.data_ptr() if given else None,
                                        sig.data_ptr(), None, status.data_ptr(), sp))


run()
torch.cuda.synchronize()
ref = sig.clone()
for k in range(K):
    a = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    a.record(); run(); e.record(); torch.cuda.synchronize()
    print(f"{algo} given={given} {a.elapsed_time(e):8.2f} ms identical={bool(torch.equal(sig, ref))}",
          flush=True)
