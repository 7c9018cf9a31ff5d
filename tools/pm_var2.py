"""P-MinHash run-to-run spread with NVML sampled DURING each call (clock, power,
throttle reasons) and the time of every launch of the call (a slow call:
which kernel, and did the clock move?)."""
import ctypes
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 16
b = datagen.config2()
ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
sig = torch.empty((b.nsets, 1024), dtype=torch.int64, device="cuda")
st = torch.empty((b.nsets, 3), dtype=torch.int64, device="cuda")
L = _lib.load()
err = ctypes.c_int64(-1)
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def run():
    _lib.check(L.pmh_sketch_csr(0, 1024, ids.data_ptr(), w.data_ptr(), off.data_ptr(),
                                b.nsets, sig.data_ptr(), st.data_ptr(), ctypes.byref(err), s))


run()
torch.cuda.synchronize()
ref = sig.clone()
for k in range(K):
    samples = []
    stop = threading.Event()

    def samp():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
            time.sleep(0.005)
    t = threading.Thread(target=samp)
    t.start()
    a = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    a.record(); run(); e.record(); torch.cuda.synchronize()
    stop.set(); t.join()
    ms = a.elapsed_time(e)
    clk = [x[0] for x in samples] or [0]
    pw = [x[1] for x in samples] or [0]
    reasons = sorted({x[2] for x in samples})
    same = bool(torch.equal(sig, ref))
    print(f"{ms:8.2f} ms  clk min/max {min(clk)}/{max(clk)}  power max {max(pw):.0f} W  "
          f"reasons {[hex(r) for r in reasons]}  n={len(samples)} identical={same}", flush=True)
