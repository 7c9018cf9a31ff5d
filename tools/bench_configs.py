"""Secondary measurements for BASELINE.json configs[0], [2], [3], [4] on one
GPU (bench.py measures the headline configs[1]).  Device-resident inputs,
CUDA-event timing (1 warm-up + 3 timed runs, min and mean reported), one JSON
line per measurement.  Elements/s counts every element of the batch once per
variant; all-pairs reports pairs/s and equal-component compares/s."""
import argparse
import ctypes
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1911_00675_b200 import _lib, datagen  # noqa: E402
from paper_1911_00675_b200.batch import (allpairs_bbit_hist_device, allpairs_hist_device,  # noqa: E402
                                         bbit_pack_device, to_device_f64, to_device_i64,
                                         to_device_u64)

L = _lib.load()


def timed(fn, reps=3):
    """Per-call device time.  Short calls (< 20 ms) are timed as a burst of
    back-to-back calls between the events (an idle GPU between synchronised
    single calls measures launch latency and clock ramp, not the kernels)."""
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    inner = max(1, min(50, int(20.0 / max(a.elapsed_time(b), 1e-3))))
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(inner):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / inner)
    return min(ts), float(np.mean(ts))


def sketch_fn(algo, m, ids, w, off, S, sig, status, setw=None):
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def f():
        _lib.check(L.pmh_sketch_csr_w_async(_lib.ALG[algo], m, ids.data_ptr(),
                                            w.data_ptr() if w is not None else None, off.data_ptr(),
                                            S, setw.data_ptr() if setw is not None else None,
                                            sig.data_ptr(), None, status.data_ptr(), sp))
    return f


def run_sketch(cfg, batch, algos, m):
    ids = to_device_u64(batch.ids)
    w = to_device_f64(batch.weights) if batch.weights is not None else None
    off = to_device_i64(batch.offsets)
    S, N = batch.nsets, batch.nelems
    sig = torch.empty((S, m), dtype=torch.int64, device="cuda")
    status = torch.empty(2, dtype=torch.int64, device="cuda")
    out = {}
    setw = None
    if any(a.startswith("nonstreaming") for a in algos):
        # the non-streaming variants: the sets' total weights are known in
        # advance (computed here, outside the timing, as a caller would have them)
        setw = torch.empty(S, dtype=torch.float64, device="cuda")
        _lib.check(L.pmh_set_weights(w.data_ptr(), off.data_ptr(), S, setw.data_ptr(), None))
    for a in algos:
        _lib.check(L.pmh_status_reset(status.data_ptr(), None))
        ns = a.startswith("nonstreaming")
        fn = sketch_fn("probminhash" + a[-1] if ns else a, m, ids, w, off, S, sig, status,
                       setw if ns else None)
        tmin, tmean = timed(fn)
        err = ctypes.c_int64(-1)
        _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), None), err.value)
        line = {"config": cfg, "algo": a, "m": m, "sets": S, "elements": N,
                "ms_min": tmin, "ms_mean": tmean, "elements_per_s": N / (tmin / 1e3),
                # wrapping sum of all signature words: identical across builds
                "sig_checksum": int(sig.sum().item())}
        print(json.dumps(line), flush=True)
        out[a] = sig.clone() if a == algos[-1] else None
    return sig


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,3,4,5")
    args = ap.parse_args()
    cfgs = args.configs.split(",")
    if "1" in cfgs:
        run_sketch("configs[0] PMH3 m=256 1000x1000", datagen.config1(), ["probminhash3",
                                                                          "probminhash3a"], 256)
    if "3" in cfgs:
        b = datagen.config3()
        run_sketch("configs[2] unweighted m=4096 100000x1000", b,
                   ["unweighted1", "unweighted1a", "unweighted2", "unweighted3", "unweighted3a",
                    "unweighted4"], 4096)
        del b
    if "4" in cfgs:
        run_sketch("configs[3] PMH2/PMH4 (non-streaming == streaming) m=64 1e6x100 Pareto1.5",
                   datagen.config4(), ["probminhash2", "probminhash4", "nonstreaming2", "nonstreaming4"], 64)
    if "5" in cfgs:
        b, jt, jx = datagen.config5_pairs()
        sig = run_sketch("configs[4] PMH4 m=256 100000x500 (50k pairs)", b, ["probminhash4"], 256)
        n = sig.shape[0]
        box = {}

        npairs = n * (n - 1) // 2
        for method in ("dense", "join"):
            def ap_fn():
                box["r"] = allpairs_hist_device(sig, threshold=1, cap=1 << 20, method=method)
            tmin, tmean = timed(ap_fn, reps=2)
            hist, pairs, k = box["r"]
            print(json.dumps({"config": f"configs[4] all-pairs equal-component counts ({method})",
                              "n": n, "m": 256, "pairs": npairs, "ms_min": tmin, "ms_mean": tmean,
                              "pairs_per_s": npairs / (tmin / 1e3),
                              "compares_per_s": npairs * 256 / (tmin / 1e3),
                              "pairs_with_count_ge_1": k,
                              "hist_checksum": int((hist.cpu().numpy() * np.arange(257)).sum())}),
                  flush=True)
        # packed b-bit signatures (reduction + packing fused, SWAR all-pairs)
        for bb in (1, 4, 8):
            box2 = {}

            def pack_fn():
                box2["p"] = bbit_pack_device(sig, bb)
            pmin, _ = timed(pack_fn, reps=2)
            packed = box2["p"]

            def apb_fn():
                box2["r"] = allpairs_bbit_hist_device(packed, 256, bb, threshold=256, cap=1 << 20)
            tmin, tmean = timed(apb_fn, reps=2)
            print(json.dumps({"config": f"configs[4] all-pairs on packed {bb}-bit signatures",
                              "n": n, "m": 256, "b": bb, "pairs": npairs, "pack_ms": pmin,
                              "ms_min": tmin, "ms_mean": tmean,
                              "pairs_per_s": npairs / (tmin / 1e3),
                              "component_compares_per_s": npairs * 256 / (tmin / 1e3)}),
                  flush=True)


if __name__ == "__main__":
    main()
