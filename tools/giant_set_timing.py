"""P-MinHash on one very large set (robustness of the one-CTA-per-set design)."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
algo = sys.argv[2] if len(sys.argv) > 2 else "pminhash"
rng = np.random.default_rng(0)
ids = to_device_u64(rng.integers(0, 2**63, n).astype(np.uint64))
w = to_device_f64(rng.random(n) + 1e-3)
off = to_device_i64(np.array([0, n], np.int64))
sig = torch.empty((1, 1024), dtype=torch.int64, device="cuda")
st = torch.zeros(2, dtype=torch.int64, device="cuda")
L = _lib.load()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for r in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _lib.check(L.pmh_sketch_csr_async(_lib.ALG[algo], 1024, ids.data_ptr(), w.data_ptr(), off.data_ptr(), 1,
                                      sig.data_ptr(), None, st.data_ptr(), sp))
    b.record()
    torch.cuda.synchronize()
    print(f"{algo} n={n} m=1024: {a.elapsed_time(b):.2f} ms", flush=True)
