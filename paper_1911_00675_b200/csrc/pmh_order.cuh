// pmh_order.cuh -- device-side largest-cost-first set ordering (LPT).
//
// One CTA processes one set, so the batch makespan is set by the order in
// which CTAs start: the most expensive sets must start first.  The cost key
// is floor(log2(n + c)) with a family-specific offset c (the ProbMinHash
// families pay ~m ln m points per set even for n = 1; P-MinHash pays n*m).
// Three small kernels build a counting-sort permutation by descending key
// without any host round trip: histogram -> scan -> scatter.
#pragma once
#include <stdint.h>

namespace pmh {

constexpr int ORDER_BUCKETS = 64;

// key 0 is reserved for "small" sets (n <= small_n) handled by a separate
// warp-per-set kernel; they sort after every large set.
__device__ __forceinline__ int order_key(int64_t n, int64_t c, int64_t small_n) {
  if (n <= small_n) return 0;
  const unsigned long long v = (unsigned long long)(n + c);
  const int k = v ? 64 - __clzll((long long)v) : 1;
  return k > ORDER_BUCKETS - 1 ? ORDER_BUCKETS - 1 : k;
}

// counts[0] = #sets with n > small_n, counts[1] = #sets with n >= big_n
__global__ void order_hist_kernel(const int64_t* __restrict__ offsets, int64_t nsets, int64_t c,
                                  int64_t small_n, int64_t big_n, unsigned int* __restrict__ hist,
                                  unsigned int* __restrict__ n_large) {
  __shared__ unsigned int sh[ORDER_BUCKETS];
  __shared__ unsigned int s_big;
  for (int i = threadIdx.x; i < ORDER_BUCKETS; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) s_big = 0;
  __syncthreads();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nsets;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = offsets[s + 1] - offsets[s];
    atomicAdd(&sh[order_key(n, c, small_n)], 1u);
    if (n >= big_n) atomicAdd(&s_big, 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ORDER_BUCKETS; i += blockDim.x) {
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
    if (i > 0 && sh[i]) atomicAdd(n_large, sh[i]);
  }
  if (threadIdx.x == 0 && s_big) atomicAdd(n_large + 1, s_big);
}

// single warp: exclusive scan in DESCENDING key order -> bucket cursors
__global__ void order_scan_kernel(unsigned int* __restrict__ hist) {
  const int lane = threadIdx.x;
  unsigned int a = hist[ORDER_BUCKETS - 1 - 2 * lane], b = hist[ORDER_BUCKETS - 2 - 2 * lane];
  unsigned int v = a + b, inc = v;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  const unsigned int ex = inc - v;
  hist[ORDER_BUCKETS - 1 - 2 * lane] = ex;
  hist[ORDER_BUCKETS - 2 - 2 * lane] = ex + a;
}

__global__ void order_scatter_kernel(const int64_t* __restrict__ offsets, int64_t nsets, int64_t c,
                                     int64_t small_n, unsigned int* __restrict__ cursor,
                                     int32_t* __restrict__ order) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nsets;
       s += (int64_t)gridDim.x * blockDim.x) {
    const unsigned int pos =
        atomicAdd(&cursor[order_key(offsets[s + 1] - offsets[s], c, small_n)], 1u);
    order[pos] = (int32_t)s;
  }
}

}  // namespace pmh
