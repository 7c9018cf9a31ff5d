// pmh_harness.cuh -- device side of the fused MSE cell (K:920-963,
// harness.run_mse_cell harness.py:266-280).
//
// The reference draws, for pair t and weight pair q of the fixture, one id
// from a single splitmix64 stream seeded with the cell seed: word
// j = t * npairs + q, i.e. eid = mix64(seed + (j + 1) * GOLDEN) (K:47-60), and
// adds it to side A where wa[q] > 0 and to side B where wb[q] > 0, in q
// order.  The words are random-access, so a chunk of C pairs is materialised
// directly in HBM as one CSR batch of 2C sets: the C A-sides first, then the
// C B-sides, so the two signature halves are contiguous [C, m] blocks for
// the equal-component count.
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

struct MseGenArgs {
  const double* wa;        // [npairs] fixture weights (0 = absent)
  const double* wb;
  const int32_t* rank_a;   // [npairs] position of q among A's elements
  const int32_t* rank_b;
  int64_t npairs;
  int64_t na, nb;          // elements per A / B set
  uint64_t seed;
  int64_t t0;              // first pair of this chunk
  int64_t C;               // pairs in this chunk
  uint64_t* ids;           // [C (na + nb)]
  double* w;
  int64_t* offsets;        // [2C + 1]
};

__global__ void mse_gen_kernel(MseGenArgs a) {
  const int64_t total = a.C * a.npairs;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += stride) {
    const int64_t t = x / a.npairs, q = x - t * a.npairs;
    const uint64_t j = (uint64_t)(a.t0 + t) * (uint64_t)a.npairs + (uint64_t)q;
    const uint64_t eid = stream_word(a.seed, j + 1);
    const double wa = a.wa[q], wb = a.wb[q];
    if (wa > 0.0) {
      const int64_t p = t * a.na + a.rank_a[q];
      a.ids[p] = eid;
      a.w[p] = wa;
    }
    if (wb > 0.0) {
      const int64_t p = a.C * a.na + t * a.nb + a.rank_b[q];
      a.ids[p] = eid;
      a.w[p] = wb;
    }
  }
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= 2 * a.C; s += stride)
    a.offsets[s] = s <= a.C ? s * a.na : a.C * a.na + (s - a.C) * a.nb;
}

// int32 counts -> the reference's int64 match vector (K:942)
__global__ void widen_counts_kernel(const int32_t* c, int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = c[i];
}

}  // namespace pmh
