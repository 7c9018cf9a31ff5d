"""Strong-scaling projection on ONE GPU: time every rank's shard of the
configs[1] step (dist.shard_ranges_multi, the split bench.py --gpus N uses)
back to back on this GPU; the N-GPU step is the slowest shard (there is no
collective on the sketch path).  Prints one JSON line per N with the shard
times, the projected step and the projected efficiency against N x the
1-GPU value.  A projection, not a multi-GPU measurement.

    python tools/shard_sim.py [N1,N2,...] [--concurrent]
"""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64  # noqa: E402
from paper_1911_00675_b200.dist import local_batch, shard_ranges_multi  # noqa: E402

M = 1024
VARIANTS = ["pminhash", "probminhash1", "probminhash1a", "probminhash2", "probminhash3",
            "probminhash3a", "probminhash4"]
L = _lib.load()


CONCURRENT = "--concurrent" in sys.argv


def step_ms(b, reps=3):
    ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
    S = b.nsets
    sig = torch.empty((S, M), dtype=torch.int64, device="cuda")
    sigs = [torch.empty((S, M), dtype=torch.int64, device="cuda") for _ in VARIANTS] if CONCURRENT else []
    arr_a = (ctypes.c_int * len(VARIANTS))(*[_lib.ALG[v] for v in VARIANTS])
    arr_s = (ctypes.c_void_p * len(VARIANTS))(*[t.data_ptr() for t in sigs])
    setw = torch.empty(S, dtype=torch.float64, device="cuda")
    status = torch.zeros(2, dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.pmh_status_reset(status.data_ptr(), sp))

    def one():
        if CONCURRENT:   # the variants on concurrent internal streams (one set-weights pass)
            _lib.check(L.pmh_sketch_csr_multi_async(arr_a, len(VARIANTS), M, ids.data_ptr(),
                                                    w.data_ptr(), off.data_ptr(), S, arr_s, None,
                                                    status.data_ptr(), sp))
            return
        _lib.check(L.pmh_set_weights(w.data_ptr(), off.data_ptr(), S, setw.data_ptr(), sp))
        for v in VARIANTS:
            _lib.check(L.pmh_sketch_csr_w_async(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(),
                                                off.data_ptr(), S, setw.data_ptr(), sig.data_ptr(),
                                                None, status.data_ptr(), sp))
    one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        a.record()
        one()
        e.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(e))
    err = ctypes.c_int64(-1)
    _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
    return min(ts)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    worlds = [int(v) for v in (args[0] if args else "1,2,4,8").split(",")]
    full = datagen.config2()
    v1 = None
    for n in worlds:
        shards = shard_ranges_multi(full.offsets, n, M, VARIANTS)
        ms = [step_ms(local_batch(full, r)) for r in shards]
        step = max(ms)
        value = len(VARIANTS) * full.nelems / (step / 1e3)
        if n == 1:
            v1 = value
        print(json.dumps({"n_gpus_projected": n, "shard_ms": [round(t, 3) for t in ms],
                          "step_ms": round(step, 3), "value": value,
                          "efficiency_vs_1": (value / (n * v1)) if v1 else None,
                          "imbalance": round(step / float(np.mean(ms)), 4), "concurrent": CONCURRENT}), flush=True)


def per_variant(n, r=0, reps=3):
    """ms of each variant alone on shard r of n (the scaling breakdown)."""
    full = datagen.config2()
    b = local_batch(full, shard_ranges_multi(full.offsets, n, M, VARIANTS)[r])
    ids, w, off = to_device_u64(b.ids), to_device_f64(b.weights), to_device_i64(b.offsets)
    S = b.nsets
    sig = torch.empty((S, M), dtype=torch.int64, device="cuda")
    setw = torch.empty(S, dtype=torch.float64, device="cuda")
    status = torch.zeros(2, dtype=torch.int64, device="cuda")
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.pmh_status_reset(status.data_ptr(), sp))
    _lib.check(L.pmh_set_weights(w.data_ptr(), off.data_ptr(), S, setw.data_ptr(), sp))
    out = {}
    for v in VARIANTS:
        def one():
            _lib.check(L.pmh_sketch_csr_w_async(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(),
                                                off.data_ptr(), S, setw.data_ptr(), sig.data_ptr(),
                                                None, status.data_ptr(), sp))
        one()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record()
            one()
            e.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(e))
        out[v] = round(min(ts), 3)
    print(json.dumps({"shard": f"{r}/{n}", "sets": S, "elements": b.nelems, "variant_ms": out}))


if __name__ == "__main__":
    if "--per-variant" in sys.argv:
        for n in (1, 8):
            per_variant(n)
    elif "--pminhash" in sys.argv:   # P-MinHash alone on shard 0 of 1 and of 8
        VARIANTS[:] = ["pminhash"]
        for n in (1, 8):
            per_variant(n)
    else:
        main()
