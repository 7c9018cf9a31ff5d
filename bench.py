"""Benchmark: set elements hashed/sec at m=1024 (BASELINE.json metric).

Workload (BASELINE.json configs[1], the headline): 10,000 weighted sets with
log-uniform sizes in [1, 100000] (~8.7e7 elements), uniform (0,1] weights,
seeded synthetic data (datagen.config2).  One STEP = the whole batch sketched
once by each of the 7 weighted variants (P-MinHash, ProbMinHash 1, 1a, 2, 3,
3a, 4) at m = 1024; value = 7 * elements / step time (whole job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling strong|weak] [--workload config2|config5]

Multi-GPU: one process per GPU.  Under torchrun the ranks come from the
environment; `--gpus N` without it re-launches this script under
torch.distributed.run with N ranks (and refuses if fewer than N devices are
visible).  Default `--scaling strong`: ONE configs[1] batch split into
contiguous set ranges balanced on the summed cost of the 7 variants
(dist.shard_ranges_multi) -- no collective on the data path; value = the
batch's elements x 7 / the max-over-ranks step time.  `--scaling weak`: every
rank sketches its own configs[1] batch; for N > 1 the strong line also
carries a weak-scaling value measured the same way (`weak`).

Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Inputs (1.47 GB) exceed the 126 MB L2 between steps.
`e2e` re-measures the metric through the C ABI host entry point
(pmh_sketch_csr_host_multi_async) with pinned host buffers: each step copies
the batch's ids/weights/offsets host->device once and every variant's
signatures device->host, all inside the timed region.

Rooflines: `roofline` is the dominant kernel's (P-MinHash: the 32-bit ALU
pipe against the measured LOP3 peak); `per_variant` adds, for every variant,
the HBM fraction (SURVEY.md §8d algorithmic bytes) and the point-rate
fraction: points_min (profiles/points_min_config2_m1024.json,
computed once by tools/points_min.py) per second against the measured
per-point ceiling of pmh_probe_point_rate.

`--impl reference` times the reference algorithm's CPU implementation (the C
restatement in oracle/, pinned bit-exact to the numba reference) on all host
cores over a bounded stratified sample of the same batch, with equal-cost
work items (P-MinHash sets cut into element parts, merged exactly).

`--workload config5`: BASELINE.json configs[4] end to end -- 50,000 designed
pairs (100,000 sets x 500 elements), ProbMinHash4 at m = 256, NCCL all-gather
of the signatures, exact all-pairs histogram over block rows, per-J-bucket
estimator statistics (similarity.run_pairs).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
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
WORKLOAD = "config2: 10k log-uniform weighted sets, 7 weighted variants, m=1024"
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
# launch (profiles/r01_ncu_pminhash64_full_config2.txt)
TRAFFIC_BYTES = {"pminhash": 2177812000 + 55420672}
UNIT = "elements/s"
# point-rate probe kind per variant (pmh_probe_point_rate): log1p points
# (ProbMinHash 1/1a/2) or TruncExp points (3/3a/4)
POINT_KIND = {"probminhash1": 0, "probminhash1a": 0, "probminhash2": 0,
              "probminhash3": 1, "probminhash3a": 1, "probminhash4": 1}
# c_v of SURVEY.md §8d: SASS instructions (issue slots) per point of the
# per-point probe's loop body, by point kind (tools/sass_loop_cost.py ->
# profiles/r02b_point_cost_sass.txt): a log1p point 183, a TruncExp point 81
C_V = {0: 183, 1: 81}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _points_min():
    p = os.path.join(ROOT, "profiles", f"points_min_config2_m{M}.json")
    try:
        with open(p) as f:
            return json.load(f)["points_min"]
    except Exception:
        return {}


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


def _cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def _reference_sample(full, target_elems):
    """Stratified subset: every k-th set in size order, ~target_elems total."""
    sizes = np.diff(full.offsets)
    order = np.argsort(sizes, kind="stable")
    k = max(1, int(np.ceil(sizes.sum() / target_elems)))
    return np.sort(order[::k])


def _oracle_step(orc, sub, cores, variants=VARIANTS):
    for v in variants:
        orc.sketch_csr_balanced(v, M, sub.ids, sub.weights, sub.offsets, threads=cores)


def run_reference(args):
    """CPU reference arm: oracle (C restatement of K, bit-exact) on all host
    cores with equal-cost work items (rank 0 only; other ranks exit 0)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc
    from paper_1911_00675_b200 import datagen
    cores = _cores()
    full = datagen.config2()
    sub = full.subset(_reference_sample(full, args.ref_sample_elems))
    orc.lib()
    times = []
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _oracle_step(orc, sub, cores)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    ms = float(np.mean(times)) * 1e3
    value = len(VARIANTS) * sub.nelems / (ms / 1e3)
    sample = (f"{sub.nsets} of {full.nsets} config-2 sets (stratified by size, "
              f"{sub.nelems} elements) x 7 variants per step; equal-cost work items "
              f"(P-MinHash sets cut into 2048-element parts, merged exactly; LPT order)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "global_batch": sub.nsets, "m": M},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_ours_line(full, cores, target_elems=400_000):
    """cpu_baseline object for our arm's line: the oracle on a bounded sample."""
    from oracle import oracle as orc
    sub = full.subset(_reference_sample(full, target_elems))
    orc.lib()
    t0 = time.perf_counter()
    _oracle_step(orc, sub, cores)
    dt = time.perf_counter() - t0
    return {"value": len(VARIANTS) * sub.nelems / dt, "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"{sub.nsets} stratified config-2 sets ({sub.nelems} elements) x 7 variants, "
                      f"oracle/pmh_oracle.c on {cores} threads, equal-cost work items"}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _relaunch(args):
    """--gpus N without torchrun: re-exec under torch.distributed.run."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible\n")
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


class Ctx:
    def __init__(self, always_pg=False):
        """always_pg: also create the (NCCL) process group at world size 1, so
        the collective path runs for real (config5's all-gather)."""
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.pg = self.world > 1 or always_pg
        if self.world > 1:
            dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        elif always_pg:
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}",
                                    rank=0, world_size=1,
                                    device_id=torch.device("cuda", self.local))

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, v, op="max"):
        if self.world == 1:
            return v
        t = self.torch.tensor([float(v)], device="cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.pg:
            self.dist.destroy_process_group()


class Step:
    """One configs[1] batch resident on this rank's GPU and its step launcher
    (every variant through the asynchronous C ABI entry, no host sync)."""

    def __init__(self, ctx, batch, variants, concurrent=False, shared_w=True):
        torch = ctx.torch
        from paper_1911_00675_b200 import _lib
        from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64
        self.ctx, self.batch, self.variants, self.concurrent = ctx, batch, variants, concurrent
        self.L, self.lib = _lib.load(), _lib
        self.N, self.S = batch.nelems, batch.nsets
        self.ids = to_device_u64(batch.ids)
        self.w = to_device_f64(batch.weights)
        self.off = to_device_i64(batch.offsets)
        self.sig = torch.empty((self.S, M), dtype=torch.int64, device="cuda")
        self.stream = torch.cuda.current_stream()
        self.sp = ctypes.c_void_p(self.stream.cuda_stream)
        self.status = torch.empty(2, dtype=torch.int64, device="cuda")
        _lib.check(self.L.pmh_status_reset(self.status.data_ptr(), self.sp))
        self.sigs_multi = [torch.empty((self.S, M), dtype=torch.int64, device="cuda")
                           for _ in variants] if concurrent else []
        self.arr_a = (ctypes.c_int * len(variants))(*[_lib.ALG[v] for v in variants])
        self.arr_s = (ctypes.c_void_p * len(variants))(*[t.data_ptr() for t in self.sigs_multi])
        self.ev = {v: [] for v in variants}
        # the sets' total weights, computed ONCE per step for all variants
        # (pmh_set_weights; each kernel would otherwise re-read every weight
        # for its threshold guess) -- inside the timed step
        self.shared_w = shared_w
        self.setw = torch.empty(self.S, dtype=torch.float64, device="cuda")
        self.ev["set_weights"] = []

    def launch_setw(self, timed=False):
        if timed:
            torch = self.ctx.torch
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(self.stream)
        self.lib.check(self.L.pmh_set_weights(self.w.data_ptr(), self.off.data_ptr(), self.S,
                                              self.setw.data_ptr(), self.sp))
        if timed:
            b.record(self.stream)
            self.ev["set_weights"].append((a, b))

    def launch(self, v):
        self.lib.check(self.L.pmh_sketch_csr_w_async(
            self.lib.ALG[v], M, self.ids.data_ptr(), self.w.data_ptr(), self.off.data_ptr(),
            self.S, self.setw.data_ptr() if self.shared_w else None, self.sig.data_ptr(), None,
            self.status.data_ptr(), self.sp))

    def timed_launch(self, v):
        torch = self.ctx.torch
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(self.stream)
        self.launch(v)
        b.record(self.stream)
        self.ev[v].append((a, b))

    def step(self, timed=False):
        if self.concurrent:
            self.lib.check(self.L.pmh_sketch_csr_multi_async(
                self.arr_a, len(self.variants), M, self.ids.data_ptr(), self.w.data_ptr(),
                self.off.data_ptr(), self.S, self.arr_s, None, self.status.data_ptr(), self.sp))
            return
        if self.shared_w:
            self.launch_setw(timed)
        for v in self.variants:
            self.timed_launch(v) if timed else self.launch(v)

    def run(self, steps, warmup, clk=None):
        """W untimed + K timed steps: max-over-ranks ms per step."""
        torch = self.ctx.torch
        for _ in range(warmup):
            self.step()
        torch.cuda.synchronize()
        self.ctx.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        if clk is not None:
            clk.__enter__()
        t0.record(self.stream)
        for _ in range(steps):
            self.step(timed=True)
        t1.record(self.stream)
        torch.cuda.synchronize()
        if clk is not None:
            clk.__exit__()
        self.ctx.barrier()
        err = ctypes.c_int64(-1)
        self.lib.check(self.L.pmh_status_check(self.status.data_ptr(), ctypes.byref(err), self.sp),
                       err.value)
        return self.ctx.reduce(t0.elapsed_time(t1)) / steps

    def per_variant_ms(self, reps):
        if self.concurrent:   # no separable per-kernel times: each variant alone
            torch = self.ctx.torch
            for _ in range(reps):
                for v in self.variants:
                    self.timed_launch(v)
            torch.cuda.synchronize()
        return {v: float(np.mean([a.elapsed_time(b) for a, b in self.ev[v]])) if self.ev[v]
                else None for v in self.variants}

    def setw_ms(self):
        e = self.ev["set_weights"]
        return float(np.mean([a.elapsed_time(b) for a, b in e])) if e else 0.0


def run_e2e(ctx, step, steps):
    """The metric through the C ABI host entry with HOST buffers (pinned):
    every step copies its inputs in and every variant's signatures out inside
    the timed region; batches pipelined E2E_DEPTH deep."""
    torch = ctx.torch
    L, lib, b = step.L, step.lib, step.batch
    variants, S, N = step.variants, step.S, step.N
    h_ids = torch.from_numpy(b.ids.view(np.int64)).pin_memory()
    h_w = torch.from_numpy(b.weights).pin_memory()
    h_off = torch.from_numpy(b.offsets).pin_memory()
    h_sigs = [[torch.empty((S, M), dtype=torch.int64).pin_memory() for _ in variants]
              for _ in range(2)]
    aids = (ctypes.c_int * len(variants))(*[lib.ALG[v] for v in variants])
    sig_ptrs = [(ctypes.c_void_p * len(variants))(*[t.data_ptr() for t in hs]) for hs in h_sigs]
    err = ctypes.c_int64(-1)

    def sync_step():
        lib.check(L.pmh_sketch_csr_host_multi(aids, len(variants), M, h_ids.data_ptr(),
                                              h_w.data_ptr(), h_off.data_ptr(), S, N, sig_ptrs[0],
                                              None, ctypes.byref(err)), err.value)

    def async_step(i):
        lib.check(L.pmh_sketch_csr_host_multi_async(aids, len(variants), M, h_ids.data_ptr(),
                                                    h_w.data_ptr(), h_off.data_ptr(), S, N,
                                                    sig_ptrs[i % 2], None, step.status.data_ptr(),
                                                    step.sp))

    def timed(run_steps, k):
        ctx.barrier()
        t0 = time.perf_counter()
        run_steps(k)
        torch.cuda.synchronize()
        return ctx.reduce((time.perf_counter() - t0) / k)

    def pipelined(k):
        done = []
        for i in range(k):
            if i >= E2E_DEPTH:
                done[i - E2E_DEPTH].synchronize()
            async_step(i)
            e = torch.cuda.Event()
            e.record(step.stream)
            done.append(e)

    sync_step()
    sync_s = timed(lambda k: [sync_step() for _ in range(k)], steps)
    lib.check(L.pmh_status_reset(step.status.data_ptr(), step.sp))
    pipelined(E2E_DEPTH)
    torch.cuda.synchronize()
    pipe_s = timed(pipelined, max(steps, 10))
    lib.check(L.pmh_status_check(step.status.data_ptr(), ctypes.byref(err), step.sp), err.value)
    h2d = b.ids.nbytes + b.weights.nbytes + b.offsets.nbytes
    d2h = len(variants) * S * M * 8
    return pipe_s, sync_s, h2d, d2h


def _probe(L, lib, fn, kind):
    v = ctypes.c_double(0.0)
    t = ctypes.c_double(0.0)
    lib.check(fn(kind, ctypes.byref(v), ctypes.byref(t)))
    return v.value


def run_config2(args, ctx):
    torch = ctx.torch
    from paper_1911_00675_b200 import _lib, datagen
    from paper_1911_00675_b200.dist import local_batch, shard_ranges_multi
    variants = args.variants.split(",")
    world, rank = ctx.world, ctx.rank
    if args.scaling == "strong":
        full = datagen.config2(seed=2)
        batch = full if world == 1 else local_batch(
            full, shard_ranges_multi(full.offsets, world, M, variants)[rank])
    else:
        full = None
        batch = datagen.config2(seed=2 + rank)
    # N > 1: a rank's shard (~1/N of the sets) leaves the GPU underfilled by any
    # one variant's latency-bound sets, so the variants run concurrently there
    # (tools/shard_sim.py: projected 8-GPU step 17.3 -> 15.2 ms); N = 1 keeps the
    # sequential step with per-launch events (equal time, exact per-variant split)
    args.concurrent = args.concurrent or world > 1
    step = Step(ctx, batch, variants, args.concurrent, shared_w=not args.no_shared_w)
    clk = ClockSampler(ctx.local)
    ms_step = step.run(args.steps, args.warmup, clk)
    per_variant_ms = step.per_variant_ms(args.per_variant_reps)
    n_total = ctx.reduce(step.N, "sum")
    value = len(variants) * n_total / (ms_step / 1e3)

    weak = None
    if world > 1 and args.scaling == "strong" and not args.no_weak:
        wb = datagen.config2(seed=2 + rank)
        wstep = Step(ctx, wb, variants, args.concurrent, shared_w=not args.no_shared_w)
        wms = wstep.run(args.steps, args.warmup)
        wn = ctx.reduce(wb.nelems, "sum")
        weak = {"value": len(variants) * wn / (wms / 1e3), "ms_per_step": wms,
                "note": "every rank sketches its own configs[1] batch (seed 2 + rank)"}
        del wstep

    e2e = None
    if args.e2e_steps > 0:
        pipe_s, sync_s, h2d, d2h = run_e2e(ctx, step, args.e2e_steps)
        e2e = {"value": len(variants) * n_total / pipe_s, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "api": "pmh_sketch_csr_host_multi_async, batches pipelined %d deep" % E2E_DEPTH,
               "sync_call_value": len(variants) * n_total / sync_s}

    if rank != 0:
        return None

    L = _lib.load()
    hbm_peak, peak_src = _peaks()
    if any(t is None for t in per_variant_ms.values()):   # --concurrent --per-variant-reps 0
        per_variant_ms = {v: ms_step / len(variants) for v in variants}
    N, S = step.N, step.S
    alg_bytes = algorithmic_bytes(N, S, M)
    lop3 = _probe(L, _lib, L.pmh_probe_pipe_peak, 0)
    peaks = {"lop3_gops": lop3,
             "imad_gops": _probe(L, _lib, L.pmh_probe_pipe_peak, 1),
             "dfma_gops": _probe(L, _lib, L.pmh_probe_pipe_peak, 2),
             "ffma_gops": _probe(L, _lib, L.pmh_probe_pipe_peak, 3),
             "point_rate_gpts": {"log1p": _probe(L, _lib, L.pmh_probe_point_rate, 0),
                                 "truncexp": _probe(L, _lib, L.pmh_probe_point_rate, 1)},
             "source": "measured live (pmh_probe_pipe_peak / pmh_probe_point_rate; csrc/pmh_probe.cuh)"}
    pmin = _points_min() if (args.scaling == "weak" or world == 1) else {}
    per_variant = {}
    for v, t in per_variant_ms.items():
        hbm = alg_bytes / (t / 1e3) / 1e9
        d = {"ms": t, "elems_per_s": N / (t / 1e3), "hbm_GBps": hbm, "hbm_frac": hbm / hbm_peak}
        if v in POINT_KIND and v in pmin:
            rate = pmin[v] / (t / 1e3) / 1e9
            ceil = peaks["point_rate_gpts"]["log1p" if POINT_KIND[v] == 0 else "truncexp"]
            cv = C_V[POINT_KIND[v]]
            issue = pmin[v] * cv / (t / 1e3) / 1e9
            d.update({"points_min": pmin[v], "points_min_gpts": rate,
                      "point_rate_peak_gpts": ceil, "point_frac": rate / ceil,
                      "c_v": cv, "issue_gops": issue, "issue_frac": issue / peaks["ffma_gops"]})
            d["bound"] = "points" if d["point_frac"] >= d["hbm_frac"] else "hbm"
        elif v == "pminhash":
            alu = float(N) * M * ALU_OPS_PER_DRAW / (t / 1e3) / 1e9
            d.update({"alu_gops": alu, "alu_frac": alu / lop3, "bound": "alu"})
        per_variant[v] = d
    dom = max(per_variant_ms, key=per_variant_ms.get)
    hbm_achieved = alg_bytes / (per_variant_ms[dom] / 1e3) / 1e9
    if dom == "pminhash":
        alu_ops = float(N) * M * ALU_OPS_PER_DRAW
        achieved = alu_ops / (per_variant_ms[dom] / 1e3) / 1e9
        roofline = {
            "bound": "alu", "kernel": "pminhash64_kernel", "achieved": achieved,
            "peak": lop3, "unit": "Gop/s (32-bit ALU pipe)", "frac": achieved / lop3,
            "traffic": TRAFFIC_BYTES.get(dom),
            "peak_source": "measured live: pmh_probe_pipe_peak(LOP3 chains, full occupancy)",
            "note": ("integer-ALU- and issue-bound (splitmix64 per draw; no GEMM-shaped work), "
                     "so neither the HBM nor the tensor roofline applies"),
            "algorithmic_ops": alu_ops, "ops_per_draw": ALU_OPS_PER_DRAW,
            "ops_per_draw_full_mix64": ALU_OPS_PER_DRAW_FULL_MIX,
            "hbm": {"achieved_GBps": hbm_achieved, "peak_GBps": hbm_peak,
                    "frac": hbm_achieved / hbm_peak, "peak_source": peak_src,
                    "algorithmic_bytes": alg_bytes},
        }
    else:
        roofline = {"bound": "hbm", "kernel": f"sketch[{dom}]", "achieved": hbm_achieved,
                    "peak": hbm_peak, "unit": "GB/s", "frac": hbm_achieved / hbm_peak,
                    "traffic": None, "peak_source": peak_src, "algorithmic_bytes": alg_bytes}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_ours_line(full if full is not None else batch, _cores())
    # per variant call: 3 ordering kernels; P-MinHash: + split prep, table
    # init, split kernel, finalize, the regular kernel (8); ProbMinHash
    # families: + the small-set kernel (9)
    launches = args.steps * (sum(8 if v == "pminhash" else 9 for v in variants)
                             + (0 if args.no_shared_w else 1))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sets": S if world == 1 else None,
                   "sets_this_rank": S, "elements_total": int(n_total),
                   "elements_this_rank": N, "m": M, "variants": variants,
                   "l2": "inputs 1.47 GB > 126 MB L2",
                   "parallelism": f"{args.scaling} x{world}",
                   "schedule": ("concurrent (pmh_sketch_csr_multi_async)" if args.concurrent
                                else "sequential, per-launch CUDA events in the timed region")},
        "per_variant_ms": per_variant_ms,
        "set_weights_ms": step.setw_ms(),
        "per_variant": per_variant,
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roofline,
        "peaks": peaks,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    if weak is not None:
        line["weak"] = weak
    return line


def run_config5(args, ctx):
    """BASELINE.json configs[4] end to end (similarity.run_pairs)."""
    from paper_1911_00675_b200 import datagen
    from paper_1911_00675_b200 import similarity as psim
    b, jt, jx = datagen.config5_pairs(npairs=args.pairs, n=500, seed=5)
    m = 256
    for _ in range(args.warmup):
        psim.run_pairs(b, jt, jx, m, ctx.rank, ctx.world)
    clk = ClockSampler(ctx.local)
    runs = []
    with clk:
        for _ in range(args.steps):
            runs.append(psim.run_pairs(b, jt, jx, m, ctx.rank, ctx.world))
    if ctx.rank != 0:
        return None
    last = runs[-1]
    keys = sorted(last.ms)
    ms = {k: float(np.mean([r.ms[k] for r in runs])) for k in keys}
    gpu_ms = ms["sketch"] + ms["allpairs"]
    S = b.nsets
    npairs_all = S * (S - 1) // 2
    return {
        "metric": "configs[4] end to end: set pairs compared/sec (PMH4 m=256 sketch + exact "
                  "all-pairs equal-component histogram)",
        "value": npairs_all / (gpu_ms / 1e3), "unit": "pairs/s", "n_gpus": ctx.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": gpu_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64+u64", "data": "synthetic",
        "config": {"workload": "config5: 50k designed pairs, 100k sets x 500, PMH4 m=256, "
                               "NCCL all-gather + block-row all-pairs",
                   "sets": S, "elements": b.nelems, "m": m, "pairs": args.pairs},
        "stage_ms": ms, "elements_per_s_sketch": b.nelems / (ms["sketch"] / 1e3),
        "statistics": last.summary(),
        "clocks": clk.summary(),
    }


def main():
    # stdout carries exactly one JSON line: NCCL's own banner (NCCL_DEBUG set
    # on the box) goes to stderr
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config2", choices=["config2", "config5"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-weak", action="store_true")
    ap.add_argument("--no-shared-w", action="store_true",
                    help="every variant sums the set weights itself (no pmh_set_weights pass)")
    ap.add_argument("--per-variant-reps", type=int, default=2,
                    help="untimed passes that time each variant alone (--concurrent only)")
    ap.add_argument("--concurrent", action="store_true",
                    help="run the step's variants concurrently (pmh_sketch_csr_multi_async); "
                         "per-variant times then come from separate untimed passes")
    ap.add_argument("--variants", default=",".join(VARIANTS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default): ONE config-2 batch sharded across the ranks by "
                         "estimated cost (no collective on the data path); weak: every rank "
                         "sketches its own config-2 batch")
    ap.add_argument("--pairs", type=int, default=50_000, help="config5: designed pairs")
    ap.add_argument("--ref-sample-elems", type=int, default=1_200_000,
                    help="--impl reference: elements of the stratified per-step sample")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _relaunch(args)
    ctx = Ctx(always_pg=args.workload == "config5")
    if ctx.world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={ctx.world} but --gpus {args.gpus}; "
                         f"measuring {ctx.world} rank(s)\n")
    try:
        line = run_config5(args, ctx) if args.workload == "config5" else run_config2(args, ctx)
        if line is not None:
            print(json.dumps(line), flush=True)
    finally:
        ctx.close()


if __name__ == "__main__":
    main()
