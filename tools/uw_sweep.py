"""Sets of n elements each (unweighted, or Exp(1) weights for the probminhash* variants) (n swept) at m = 1024 / 4096: per-variant
device time for the library in PMH_LIB_PATH (development tool: where the
lane-per-element and warp-per-element modes cross over)."""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

L = _lib.load()
algos = sys.argv[1].split(",") if len(sys.argv) > 1 else ["unweighted1"]
ms_ = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1024, 4096]
ns = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [32, 64, 128, 256, 512, 1000, 2048, 8192]
total = int(sys.argv[4]) if len(sys.argv) > 4 else 8_000_000
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for m in ms_:
    for n in ns:
        S = max(296, total // n)
        weighted = any(a.startswith(("prob", "pmin")) for a in algos)   # Exp(1) weights for the weighted variants
        b = datagen.random_sets(11, [n] * S, "exp") if weighted else datagen.config3(S, n, seed=11)
        ids, off = to_device_u64(b.ids), to_device_i64(b.offsets)
        wd = to_device_f64(b.weights) if weighted else None
        sig = torch.empty((S, m), dtype=torch.int64, device="cuda")
        status = torch.empty(2, dtype=torch.int64, device="cuda")
        for a in algos:
            def f():
                _lib.check(L.pmh_sketch_csr_w_async(_lib.ALG[a], m, ids.data_ptr(), wd.data_ptr() if wd is not None else None, off.data_ptr(),
                                                    S, None, sig.data_ptr(), None, status.data_ptr(), sp))
            _lib.check(L.pmh_status_reset(status.data_ptr(), None))
            f(); torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record(); f(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
            print(json.dumps({"algo": a, "m": m, "n": n, "sets": S, "ms": round(min(ts), 3),
                              "chk": int(sig.sum().item()) % 100000}), flush=True)
