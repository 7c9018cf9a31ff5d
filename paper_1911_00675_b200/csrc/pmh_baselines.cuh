// pmh_baselines.cuh -- the reference's conventional-Jaccard baselines on the
// GPU: SuperMinHash (K:784-807) and one-permutation hashing with re-draw
// densification (K:810-846).  (MinHash, K:768-781, is the EXPO = false
// instance of the P-MinHash kernels.)  One CTA per set; minima are the
// lexicographic (h, element index) slot table of pmh_device.cuh, so element
// order does not matter and ties resolve like the reference's strict `<`.
#pragma once
#include "pmh_device.cuh"

namespace pmh {

struct BaseArgs {
  const uint64_t* ids;
  const int64_t* offsets;
  int64_t nsets;
  int64_t m;
  uint64_t* sig;
  int64_t* stats;
  long long* err_set;
  unsigned long long* err_flags;
};

// SuperMinHash: per element a fresh Fisher-Yates permutation p of {0..m-1};
// step k draws u = U, r = k + uniform_int(m - k), swaps p[k], p[r] and offers
// h = u + p[k] to component k.  One warp per element: lane 0 runs the
// sequential stream / swap chain on a per-warp shared permutation (m steps,
// the bit offsets are data dependent), the offers go to the shared table.
__global__ void __launch_bounds__(256) superminhash_kernel(BaseArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t m = a.m;
  Slot* slots = reinterpret_cast<Slot*>(smem);
  int32_t* perm = reinterpret_cast<int32_t*>(smem + sizeof(Slot) * m) + (size_t)wid * m;
  for (int64_t s = blockIdx.x; s < a.nsets; s += gridDim.x) {
    const int64_t off = a.offsets[s], n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) { slots[k].h = EMPTY_H; slots[k].idx = EMPTY_IDX; }
    __syncthreads();
    for (int64_t e = wid; e < n; e += nw) {
      for (int64_t k = lane; k < m; k += 32) perm[k] = (int32_t)k;
      __syncwarp();
      if (lane == 0) {
        Stream st;
        st.seed(a.ids[off + e]);
        for (int64_t k = 0; k < m; k++) {
          const double u = st.uniform01();
          const int64_t r0 = uniform_int(st, m - k);
          if (r0 < 0) {
            atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
            atomicMin(a.err_set, (long long)s);
            break;
          }
          const int64_t r = k + r0;
          const int32_t tmp = perm[k];
          perm[k] = perm[r];
          perm[r] = tmp;
          const double h = u + (double)perm[k];
          slot_offer(&slots[k], h, (unsigned long long)e);
        }
      }
      __syncwarp();
    }
    __syncthreads();
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const unsigned long long ix = slots[k].idx;
      a.sig[(size_t)s * m + k] = ix < (unsigned long long)n ? a.ids[off + ix] : 0ULL;
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = 0; a.stats[s * 3 + 1] = 0; a.stats[s * 3 + 2] = 0;
    }
    __syncthreads();
  }
}

// OPH with densification: each element lands in bin uniform_int(m) with
// value U; every empty bin k then re-draws bins from the stream seeded with
// OPH_SALT + k * GOLDEN until it hits a filled bin and copies its id.
__global__ void __launch_bounds__(256) oph_kernel(BaseArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t m = a.m;
  Slot* slots = reinterpret_cast<Slot*>(smem);
  const uint32_t kbits = bits_for(m);
  const int64_t cap = (int64_t)(64.0 * (double)m * (1.0 + log((double)m)) + 64.0);
  for (int64_t s = blockIdx.x; s < a.nsets; s += gridDim.x) {
    const int64_t off = a.offsets[s], n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) { slots[k].h = EMPTY_H; slots[k].idx = EMPTY_IDX; }
    __syncthreads();
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
      Stream st;
      st.seed(a.ids[off + e]);
      const int64_t b = uniform_int_masked(st, (uint64_t)m, kbits);
      if (b < 0) {
        atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
        atomicMin(a.err_set, (long long)s);
        continue;
      }
      slot_offer(&slots[b], st.uniform01(), (unsigned long long)e);
    }
    __syncthreads();
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const unsigned long long ix = slots[k].idx;
      if (ix != EMPTY_IDX) { sig[k] = a.ids[off + ix]; continue; }
      Stream st;
      st.seed(OPH_SALT + (uint64_t)k * GOLDEN);
      int64_t attempts = 0;
      for (;;) {
        const int64_t j = uniform_int_masked(st, (uint64_t)m, kbits);
        if (j < 0 || ++attempts > cap + 1) {
          atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
          atomicMin(a.err_set, (long long)s);
          break;
        }
        const unsigned long long jx = slots[j].idx;
        if (jx != EMPTY_IDX) { sig[k] = a.ids[off + jx]; break; }
      }
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = 0; a.stats[s * 3 + 1] = 0; a.stats[s * 3 + 2] = 0;
    }
    __syncthreads();
  }
}

}  // namespace pmh
