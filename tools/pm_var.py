"""Run-to-run spread of one variant on the configs[1] batch: K timed calls in
one process (CUDA events), printed with the SM clock sampled around each."""
import ctypes
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

algo = sys.argv[1] if len(sys.argv) > 1 else "pminhash"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 12
b = datagen.config2()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, 1024), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    _lib.check(L.pmh_sketch_csr(_lib.ALG[algo], 1024, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                b.nsets, sig.data_ptr(), None, ctypes.byref(err), s))


run()
for k in range(K):
    a = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    a.record(); run(); e.record(); torch.cuda.synchronize()
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                        "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(f"{algo} {a.elapsed_time(e):8.2f} ms  [{q}]", flush=True)
