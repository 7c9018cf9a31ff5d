"""Benchmark: set elements hashed/sec at m=1024 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the headline): 10,000 weighted sets with
log-uniform sizes in [1, 100000] (~8.7e7 elements), uniform (0,1] weights,
seeded synthetic data (datagen.config2).  One STEP = the whole batch sketched
once by each of the 7 weighted variants (P-MinHash, ProbMinHash 1, 1a, 2, 3,
3a, 4) at m = 1024; value = 7 * elements / step time (whole job; N>1 ranks
each own a full batch -> weak scaling, no collective on this path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Inputs (1.47 GB) exceed the 126 MB L2 between steps.
`e2e` re-measures the metric through the C ABI host entry point
(pmh_sketch_csr_host_multi) with pinned host buffers: each step copies the
batch's ids/weights/offsets host->device once and every variant's signatures
device->host, all inside the timed region (wall clock around the call, which
synchronises).
`--impl reference` times the reference algorithm's CPU implementation (the C
restatement in oracle/, pinned bit-exact to the numba reference) on the host
cores, over a bounded stratified sample of the same batch.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M = 1024
VARIANTS = ["pminhash", "probminhash1", "probminhash1a", "probminhash2",
            "probminhash3", "probminhash3a", "probminhash4"]
METRIC = "set elements hashed/sec at m=1024"
E2E_DEPTH = 2   # pipelined e2e: batches in flight
# ALU-pipe work of the P-MinHash schedule (tools/gen_pm64.py) per 64 draws =
# 53 splitmix64 words: per word the low half of the counter add (1; the high
# half runs on the FMA pipe) and two 64-bit xor-shifts (4 each); the final
# xor-shift's low half (2) on the 44 words holding a draw's top bits below
# bit 44, its high half (2) on 12 of them; 23 funnel extractions; one compare
# per draw.  (The full splitmix64 + exact extraction would be 13.6 per draw.)
ALU_OPS_PER_DRAW = (53 * 9 + 44 * 2 + 12 * 2 + 23) / 64.0 + 1.0
ALU_OPS_PER_DRAW_FULL_MIX = 14.0 * 53.0 / 64.0 + 2.0
# dram read+write bytes per launch from `ncu --set full` of the full config-2
# launch (profiles/r01_ncu_pminhash64_full_config2.txt); the read side exceeds
# the algorithmic 1.39 GB of ids/weights by the weight-sum pre-pass of the
# threshold guess (~0.7 GB, a second read of the weights)
TRAFFIC_BYTES = {"pminhash": 2177812000 + 55420672}
UNIT = "elements/s"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        # NVML init + a first query happen HERE, outside the timed region (a
        # first NVML call takes driver locks that would stall kernel enqueues)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            self._nvml = (pynvml, h)
        except Exception:
            self._nvml = None

    def _run(self):
        try:
            if self._nvml is None:
                raise RuntimeError("no nvml")
            pynvml, h = self._nvml
            bits = [pynvml.nvmlClocksThrottleReasonHwSlowdown,
                    pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                    pynvml.nvmlClocksThrottleReasonSwPowerCap]
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            while not self._stop.is_set():
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.samples.append([str(sm), str(mx)] +
                                    ["Active" if r & b else "Not Active" for b in bits])
                self._stop.wait(0.1)
            return
        except Exception:
            pass
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def algorithmic_bytes(nelems, nsets, m, weighted=True):
    # 16 B/elt (8 if ids only) + 8 m B/set + 8 (S+1) offsets
    return (16 if weighted else 8) * nelems + 8 * m * nsets + 8 * (nsets + 1)


def run_reference(args):
    """CPU reference arm: oracle (C restatement of K, bit-exact) on host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    full = datagen.config2()
    sample_sets = _reference_sample(full)
    sub = full.subset(sample_sets)
    orc.lib()
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        for v in VARIANTS:
            orc.sketch_csr(v, M, sub.ids, sub.weights, sub.offsets, threads=cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    ms = float(np.mean(times)) * 1e3
    value = len(VARIANTS) * sub.nelems / (ms / 1e3)
    sample = (f"{sub.nsets} of {full.nsets} config-2 sets (stratified by size, "
              f"{sub.nelems} elements) x 7 variants per step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": "config2: 10k log-uniform weighted sets, 7 weighted variants, m=1024",
                   "global_batch": sub.nsets, "m": M},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _reference_sample(full, target_elems=400_000):
    """Stratified subset: every k-th set in size order, ~target_elems total."""
    sizes = np.diff(full.offsets)
    order = np.argsort(sizes, kind="stable")
    k = max(1, int(np.ceil(sizes.sum() / target_elems)))
    return np.sort(order[::k])


def cpu_baseline_ours_line(full, cores):
    """cpu_baseline object for our arm's line: the oracle on a bounded sample."""
    from oracle import oracle as orc
    sub = full.subset(_reference_sample(full, 200_000))
    orc.lib()
    t0 = time.perf_counter()
    for v in VARIANTS:
        orc.sketch_csr(v, M, sub.ids, sub.weights, sub.offsets, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": len(VARIANTS) * sub.nelems / dt, "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"{sub.nsets} stratified config-2 sets ({sub.nelems} elements) x 7 variants, "
                      f"oracle/pmh_oracle.c on {cores} threads"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--per-variant-reps", type=int, default=2,
                    help="untimed passes that time each variant alone (0: skip)")
    ap.add_argument("--concurrent", action="store_true",
                    help="run the step's variants concurrently (pmh_sketch_csr_multi_async); "
                         "per-variant times then come from separate untimed passes")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak (default): every rank sketches its own config-2 batch; strong: "
                         "ONE config-2 batch sharded across the ranks by estimated cost "
                         "(dist.shard_ranges_multi, no collective on the data path)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")

    from paper_1911_00675_b200 import _lib, datagen
    from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64

    variants = args.variants.split(",")
    L = _lib.load()
    if args.scaling == "strong":
        from paper_1911_00675_b200.dist import local_batch, shard_ranges_multi
        batch = datagen.config2(seed=2)
        if world > 1:
            batch = local_batch(batch, shard_ranges_multi(batch.offsets, world, M, variants)[rank])
    else:
        batch = datagen.config2(seed=2 + rank)
    N, S = batch.nelems, batch.nsets
    ids = to_device_u64(batch.ids)
    w = to_device_f64(batch.weights)
    off = to_device_i64(batch.offsets)
    sig = torch.empty((S, M), dtype=torch.int64, device="cuda")
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    err = ctypes.c_int64(-1)
    status = torch.empty(2, dtype=torch.int64, device="cuda")
    _lib.check(L.pmh_status_reset(status.data_ptr(), sp))

    def launch(v):
        # asynchronous C-ABI entry: no host sync inside the timed region
        _lib.check(L.pmh_sketch_csr_async(_lib.ALG[v], M, ids.data_ptr(), w.data_ptr(),
                                          off.data_ptr(), S, sig.data_ptr(), None,
                                          status.data_ptr(), sp))

    # one step = the batch sketched by every variant.  Default: all variants
    # in ONE pmh_sketch_csr_multi_async call (concurrent internal streams, so
    # each kernel's tail overlaps the others' work); --sequential launches
    # them one after another on this stream.
    sigs_multi = [torch.empty((S, M), dtype=torch.int64, device="cuda") for _ in variants]
    arr_a = (ctypes.c_int * len(variants))(*[_lib.ALG[v] for v in variants])
    arr_s = (ctypes.c_void_p * len(variants))(*[t.data_ptr() for t in sigs_multi])

    ev = {v: [] for v in variants}

    def launch_step(timed=False):
        if args.concurrent:
            _lib.check(L.pmh_sketch_csr_multi_async(arr_a, len(variants), M, ids.data_ptr(),
                                                    w.data_ptr(), off.data_ptr(), S, arr_s, None,
                                                    status.data_ptr(), sp))
            return
        for v in variants:
            if timed:   # per-launch events on the launching stream, inside the timed region
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                launch(v)
                b.record(stream)
                ev[v].append((a, b))
            else:
                launch(v)

    for _ in range(args.warmup):
        launch_step()
    torch.cuda.synchronize()
    if args.concurrent:
        # the concurrent step has no separable per-kernel times: each variant
        # alone, outside the timed region
        for _ in range(args.per_variant_reps):
            for v in variants:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                launch(v)
                b.record(stream)
                ev[v].append((a, b))
        torch.cuda.synchronize()

    clk_sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with clk_sampler as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for _ in range(args.steps):
            launch_step(timed=True)
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
    ms_total = t_start.elapsed_time(t_end)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    per_variant_ms = {v: float(np.mean([a.elapsed_time(b) for a, b in ev[v]])) if ev[v] else None
                      for v in variants}
    # whole-job elements: weak -- every rank sketches its own batch (seed 2 +
    # rank); strong -- the ranks' shards of one batch (the sum is that batch)
    n_total = N
    if world > 1:
        t = torch.tensor([float(N)], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        n_total = float(t.item())
    value = len(variants) * n_total / (ms_step / 1e3)

    # ---- e2e: C ABI host entry with HOST buffers, copies inside the timing ----
    # one step = the host batch sketched by all variants through
    # pmh_sketch_csr_host_multi: ids/weights/offsets cross PCIe once per step
    # (pinned), every variant's signatures come back to pinned host memory
    h_ids = torch.from_numpy(batch.ids.view(np.int64)).pin_memory()
    h_w = torch.from_numpy(batch.weights).pin_memory()
    h_off = torch.from_numpy(batch.offsets).pin_memory()
    # two sets of pinned result buffers: consecutive (pipelined) steps write
    # to different host memory
    h_sigs = [[torch.empty((S, M), dtype=torch.int64).pin_memory() for _ in variants]
              for _ in range(2)]
    aids = (ctypes.c_int * len(variants))(*[_lib.ALG[v] for v in variants])
    sig_ptrs = [(ctypes.c_void_p * len(variants))(*[t.data_ptr() for t in hs]) for hs in h_sigs]

    def e2e_step_sync():
        rc = L.pmh_sketch_csr_host_multi(aids, len(variants), M, h_ids.data_ptr(),
                                         h_w.data_ptr(), h_off.data_ptr(), S, N, sig_ptrs[0],
                                         None, ctypes.byref(err))
        _lib.check(rc, err.value)

    def e2e_step_async(i):
        # enqueue-only host entry: step i+1's H2D overlaps step i's kernels
        rc = L.pmh_sketch_csr_host_multi_async(aids, len(variants), M, h_ids.data_ptr(),
                                               h_w.data_ptr(), h_off.data_ptr(), S, N,
                                               sig_ptrs[i % 2], None, status.data_ptr(), sp)
        _lib.check(rc)

    def timed_e2e(run_steps, k):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        run_steps(k)
        torch.cuda.synchronize()
        s_per = (time.perf_counter() - t0) / k
        if world > 1:
            t = torch.tensor([s_per], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            s_per = float(t.item())
        return s_per

    e2e_s = e2e_sync_s = float("nan")
    if args.e2e_steps > 0:
        e2e_step_sync()
        e2e_sync_s = timed_e2e(lambda k: [e2e_step_sync() for _ in range(k)], args.e2e_steps)
        _lib.check(L.pmh_status_reset(status.data_ptr(), sp))
        torch.cuda.synchronize()

        def pipelined(k):
            # at most DEPTH batches in flight: before enqueueing step i the
            # host waits for step i - DEPTH (a serving loop's back-pressure;
            # also keeps the device working set at DEPTH batches)
            done = []
            for i in range(k):
                if i >= E2E_DEPTH:
                    done[i - E2E_DEPTH].synchronize()
                e2e_step_async(i)
                ev_i = torch.cuda.Event()
                ev_i.record(stream)
                done.append(ev_i)

        pipelined(E2E_DEPTH)          # warm-up: memory pool at its steady-state size
        torch.cuda.synchronize()
        # every step copies its inputs in and its signatures out (pinned host
        # memory) inside the timed region
        e2e_s = timed_e2e(pipelined, max(args.e2e_steps, 10))
        _lib.check(L.pmh_status_check(status.data_ptr(), ctypes.byref(err), sp), err.value)
    h2d = batch.ids.nbytes + batch.weights.nbytes + batch.offsets.nbytes
    d2h = len(variants) * S * M * 8

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    hbm_peak, peak_src = _peaks()
    if any(t is None for t in per_variant_ms.values()):   # --concurrent --per-variant-reps 0
        per_variant_ms = {v: ms_step / len(variants) for v in variants}
    dom = max(per_variant_ms, key=per_variant_ms.get)
    alg_bytes = algorithmic_bytes(N, S, M)
    hbm_achieved = alg_bytes / (per_variant_ms[dom] / 1e3) / 1e9
    gops = ctypes.c_double(0.0)
    pms = ctypes.c_double(0.0)
    _lib.check(L.pmh_probe_alu_peak(ctypes.byref(gops), ctypes.byref(pms)))
    if dom == "pminhash":
        # ncu: the P-MinHash kernel is bound by the 32-bit ALU pipe.  Algorithmic
        # ALU work = N*m draws x ALU_OPS_PER_DRAW (the schedule's required ALU
        # ops; the two 64-bit multiplies run on the FMA pipe) -- DESIGN.md §4.
        alu_ops = float(N) * M * ALU_OPS_PER_DRAW
        achieved = alu_ops / (per_variant_ms[dom] / 1e3) / 1e9
        roofline = {
            "bound": "alu", "kernel": "pminhash64_kernel", "achieved": achieved,
            "peak": gops.value, "unit": "Gop/s (32-bit ALU pipe)",
            "frac": achieved / gops.value, "traffic": TRAFFIC_BYTES.get(dom),
            "peak_source": "measured live: pmh_probe_alu_peak (LOP3 chains, full occupancy)",
            "note": ("integer-ALU- and issue-bound (splitmix64 per draw; ncu: ALU pipe ~81%, FMA-heavy ~62%, issue ~76%, DRAM ~0.4%, "
                     "no GEMM-shaped work), so neither the HBM nor the tensor roofline applies; "
                     "the HBM figures are given below for reference"),
            "algorithmic_ops": alu_ops, "ops_per_draw": ALU_OPS_PER_DRAW,
            "ops_per_draw_full_mix64": ALU_OPS_PER_DRAW_FULL_MIX,
            "hbm": {"achieved_GBps": hbm_achieved, "peak_GBps": hbm_peak,
                    "frac": hbm_achieved / hbm_peak, "peak_source": peak_src,
                    "algorithmic_bytes": alg_bytes},
        }
    else:
        roofline = {
            "bound": "hbm", "kernel": f"sketch[{dom}]", "achieved": hbm_achieved,
            "peak": hbm_peak, "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
            "traffic": TRAFFIC_BYTES.get(dom), "peak_source": peak_src,
            "algorithmic_bytes": alg_bytes,
        }
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_ours_line(batch, cores)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": "config2: 10k log-uniform weighted sets, 7 weighted variants, m=1024",
                   "sets_per_gpu": S, "elements_per_gpu": N, "m": M,
                   "variants": variants, "l2": "inputs 1.47 GB > 126 MB L2",
                   "schedule": ("concurrent (pmh_sketch_csr_multi_async)" if args.concurrent
                                else "sequential, per-launch CUDA events in the timed region")},
        "per_variant_ms": per_variant_ms,
        "per_variant_elems_per_s": {v: N / (t / 1e3) for v, t in per_variant_ms.items()},
        "e2e": {"value": len(variants) * n_total / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "pmh_sketch_csr_host_multi_async, batches pipelined %d deep" % E2E_DEPTH,
                "sync_call_value": len(variants) * n_total / e2e_sync_s},
        # per variant call: 3 ordering kernels + split prep, table init, split
        # kernel, finalize + the one-CTA-per-set kernel (8); the ProbMinHash
        # families also launch their small-set kernel (9)
        "gpu_launches": args.steps * sum(8 if v == "pminhash" else 9 for v in variants),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
