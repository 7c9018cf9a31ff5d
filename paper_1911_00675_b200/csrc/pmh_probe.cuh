// pmh_probe.cuh -- pipe-peak microbenchmarks: the roofline denominators of the
// integer/FP64-bound signature kernels (MEASURED_PEAKS.json only carries HBM
// and bf16 peaks).  Every thread runs 8 independent dependency chains of one
// instruction kind, so the pipe, not latency, bounds the rate:
//   PROBE_LOP3  lop3.b32      32-bit ALU pipe
//   PROBE_IMAD  mad.lo.u32    integer multiply-add (FMA pipe)
//   PROBE_DFMA  fma.rn.f64    FP64 pipe (one DFMA = 2 flops; counted as 1 op)
//   PROBE_FFMA  fma.rn.f32    FP32 FMA: the issue-slot ceiling (one warp
//                             instruction per scheduler per clock)
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

enum ProbeKind : int { PROBE_LOP3 = 0, PROBE_IMAD = 1, PROBE_DFMA = 2, PROBE_FFMA = 3 };

#define PMH_PROBE_CHAINS(stmt) stmt(a0) stmt(a1) stmt(a2) stmt(a3) stmt(a4) stmt(a5) stmt(a6) stmt(a7)

__global__ void __launch_bounds__(256) alu_probe_kernel(int iters, uint32_t* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u,
           a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
  const uint32_t b = blockIdx.x | 1u, c = 0x9E3779B9u;
#define PMH_LOP3(x) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x) : "r"(b), "r"(c));
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) { PMH_PROBE_CHAINS(PMH_LOP3) }
  }
#undef PMH_LOP3
  if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 0x12345678u) out[0] = 1;
}

__global__ void __launch_bounds__(256) imad_probe_kernel(int iters, uint32_t* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u,
           a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
  const uint32_t b = blockIdx.x | 1u, c = 0x9E3779B9u;
#define PMH_IMAD(x) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(b), "r"(c));
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) { PMH_PROBE_CHAINS(PMH_IMAD) }
  }
#undef PMH_IMAD
  if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 0x12345678u) out[0] = 1;
}

__global__ void __launch_bounds__(256) dfma_probe_kernel(int iters, uint32_t* out) {
  double a0 = threadIdx.x, a1 = a0 * 3.0, a2 = a0 * 5.0, a3 = a0 * 7.0, a4 = a0 * 11.0,
         a5 = a0 * 13.0, a6 = a0 * 17.0, a7 = a0 * 19.0;
  const double b = 0.999999, c = 1e-3 * (blockIdx.x + 1);
#define PMH_DFMA(x) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x) : "d"(b), "d"(c));
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) { PMH_PROBE_CHAINS(PMH_DFMA) }
  }
#undef PMH_DFMA
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1.2345) out[0] = 1;
}

__global__ void __launch_bounds__(256) ffma_probe_kernel(int iters, uint32_t* out) {
  float a0 = threadIdx.x, a1 = a0 * 3.f, a2 = a0 * 5.f, a3 = a0 * 7.f, a4 = a0 * 11.f,
        a5 = a0 * 13.f, a6 = a0 * 17.f, a7 = a0 * 19.f;
  const float b = 0.9999f, c = 1e-3f * (blockIdx.x + 1);
#define PMH_FFMA(x) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(x) : "f"(b), "f"(c));
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) { PMH_PROBE_CHAINS(PMH_FFMA) }
  }
#undef PMH_FFMA
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 1.2345f) out[0] = 1;
}

#undef PMH_PROBE_CHAINS

// Per-point work probe: the practical ceiling of the ProbMinHash point loop.
// Every thread generates points of its own element stream in a tight loop --
// one splitmix64 word per point (53 value bits + a 10-bit label, as a point
// consumes 63 stream bits at m = 1024), the value (KIND 0: E = -log1p(-U) and
// x += winv E, the ProbMinHash1/2 point, K:320-328, K:436-440; KIND 1:
// TruncExp's fast path x = winv (i - 1 + c1 U), the ProbMinHash3/4 point,
// K:130-132, K:477-480), and the 128-bit CAS offer into a shared 1024-slot
// table (K:324) -- at full occupancy with no control flow beyond the loop.
// points/s of this kernel is the denominator of bench.py's per-variant
// point-rate roofline; its SASS loop body gives c_v (profiles/).
template <int KIND>
__global__ void __launch_bounds__(256) point_probe_kernel(int iters, uint32_t* out) {
  __shared__ Slot slots[1024];
  for (int k = threadIdx.x; k < 1024; k += blockDim.x) { slots[k].h = EMPTY_H; slots[k].idx = EMPTY_IDX; }
  __syncthreads();
  const uint64_t id = (blockIdx.x * 256ull + threadIdx.x) * 0x9E3779B97F4A7C15ULL + 12345ull;
  const double winv = 1.0 + 1e-3 * (threadIdx.x & 31);
  const double c1 = 1.000488;   // m = 1024: 1/c1 = P(fast path)
  double x = 0.0;
  uint32_t acc = 0;
  for (int i = 1; i <= iters; i++) {
    const uint64_t wd = mix64(id + (uint64_t)i * GOLDEN);
    const double U = (double)(wd & ((1ULL << 53) - 1ULL)) * INV53;
    const uint32_t lab = (uint32_t)(wd >> 53) & 1023u;
    if constexpr (KIND == 0) {
      x = x + winv * -g_log1p_negu(-U);
    } else {
      x = winv * ((double)i - 1.0) + winv * (c1 * U);
    }
    const unsigned long long prev = slot_offer(&slots[lab], x, (unsigned long long)threadIdx.x);
    acc += (uint32_t)prev;
  }
  if (acc == 0x12345678u) out[0] = 1;
}

// Device build of the glibc restatements (pmh_math.cuh) over an input array:
// fn 0 = log1p, fn 1 = expm1 (NaN where the restatement reports no result).
// Lets a GPU test compare the DEVICE transcendental bit-for-bit with the host
// glibc -- signature parity alone would not pin it (a rare 1-ulp flip seldom
// changes a signature).
__global__ void math_eval_kernel(int fn, const double* __restrict__ x, int64_t n,
                                 double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (fn == 0) {
      out[i] = g_log1p(x[i]);
    } else if (fn == 2) {
      out[i] = g_log1p_negu(x[i]);   // the sampled-domain specialisation (x = -U)
    } else {
      bool ok = true;
      const double e = g_expm1(x[i], &ok);
      out[i] = ok ? e : __longlong_as_double(0x7FF8000000000000LL);
    }
  }
}

}  // namespace pmh
