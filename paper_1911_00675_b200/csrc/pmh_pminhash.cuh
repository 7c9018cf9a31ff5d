// pmh_pminhash.cuh -- P-MinHash (Alg. 1, K:284-300) and the stream-per-
// component baselines on sm_100a.
//
// Every element draws one Exp(1) per component k at the STATIC bit offset
// 53*k of its stream (53 bits per draw, no rejection), so the (element,
// component) grid is fully parallel.  Each thread owns C consecutive
// components and keeps their running (h, argmin) in registers; a thread walks
// its elements in increasing index order with the reference's strict `<`, so
// ties resolve to the lowest index exactly like the reference.  Groups of
// threads covering all m components split the element range; their partial
// minima are merged lexicographically on (h, index) in shared memory.
// log1p is evaluated only when the provable lower bound winv*U*(1-2^-40) of
// the candidate does not already exceed the component's running minimum.
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

struct PMinArgs {
  const uint64_t* ids;
  const double* w;
  const int64_t* offsets;
  const int32_t* order;
  int64_t nsets;
  int64_t m;
  uint64_t* sig;
  int64_t* stats;
  long long* err_set;
};

constexpr int PMIN_THREADS = 256;
constexpr int PMIN_CHUNK = 256;

// C components per thread; words of thread's bit range are generated once per
// element with an incremental splitmix state.
// EXPO = true: P-MinHash h = winv * Exp(1) (K:284-300);
// EXPO = false: MinHash h = U (K:768-781), unit weights.
template <int C, bool EXPO>
__global__ void __launch_bounds__(PMIN_THREADS) pminhash_kernel(PMinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t s_id[PMIN_CHUNK];
  __shared__ double s_winv[PMIN_CHUNK];
  const int64_t m = a.m;
  const int tpg = (int)((m + C - 1) / C);          // threads per group
  const int groups = PMIN_THREADS / tpg;           // >= 1 (host guarantees)
  const int g = threadIdx.x / tpg, t = threadIdx.x % tpg;
  const bool active = g < groups;
  const int64_t k0 = (int64_t)t * C;
  Slot* part = reinterpret_cast<Slot*>(smem);      // [groups][m]

  for (int64_t bs = blockIdx.x; bs < a.nsets; bs += gridDim.x) {
    const int64_t s = a.order ? (int64_t)a.order[bs] : bs;
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    double hmin[C];
    unsigned long long arg[C];
#pragma unroll
    for (int q = 0; q < C; q++) { hmin[q] = __longlong_as_double(0x7FF0000000000000LL); arg[q] = EMPTY_IDX; }

    for (int64_t c0 = 0; c0 < n; c0 += PMIN_CHUNK) {
      const int64_t cn = n - c0 < PMIN_CHUNK ? n - c0 : PMIN_CHUNK;
      __syncthreads();
      if (threadIdx.x < cn) {
        s_id[threadIdx.x] = a.ids[off + c0 + threadIdx.x];
        s_winv[threadIdx.x] = (EXPO && a.w) ? 1.0 / a.w[off + c0 + threadIdx.x] : 1.0;
      }
      __syncthreads();
      if (!active) continue;
      for (int64_t le = g; le < cn; le += groups) {
        const uint64_t id = s_id[le];
        const double winv = s_winv[le];
        const uint64_t e = (uint64_t)(c0 + le);
        uint64_t bitpos = 53ULL * (uint64_t)k0;
        uint64_t wi = bitpos >> 6;                  // 0-based word index
        uint32_t sh = (uint32_t)(bitpos & 63);
        uint64_t st = id + (wi + 1) * GOLDEN;
        uint64_t lo = mix64(st);
        st += GOLDEN;
        uint64_t hi = mix64(st);
#pragma unroll
        for (int q = 0; q < C; q++) {
          if (k0 + q < m) {
            uint64_t b = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
            b &= (1ULL << 53) - 1ULL;
            if constexpr (EXPO) {
              if (!(exp1_scaled_lower_bound(winv, b) > hmin[q])) {
                const double h = winv * exp1_from_bits(b);
                if (h < hmin[q]) { hmin[q] = h; arg[q] = e; }
              }
            } else {
              const double h = (double)b * INV53;
              if (h < hmin[q]) { hmin[q] = h; arg[q] = e; }
            }
          }
          sh += 53;
          if (sh >= 64) {
            sh -= 64;
            lo = hi;
            if (q + 1 < C) { st += GOLDEN; hi = mix64(st); }
          }
        }
      }
    }
    // merge groups lexicographically on (h, index)
    __syncthreads();
    if (active) {
#pragma unroll
      for (int q = 0; q < C; q++) {
        if (k0 + q < m) {
          part[(size_t)g * m + k0 + q].h = dbl_bits(hmin[q]);
          part[(size_t)g * m + k0 + q].idx = arg[q];
        }
      }
    }
    __syncthreads();
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      unsigned long long bh = part[k].h, bi = part[k].idx;
      for (int gg = 1; gg < groups; gg++) {
        const unsigned long long h = part[(size_t)gg * m + k].h, ix = part[(size_t)gg * m + k].idx;
        if (h < bh || (h == bh && ix < bi)) { bh = h; bi = ix; }
      }
      sig[k] = bi < (unsigned long long)n ? a.ids[off + bi] : 0ULL;
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = n * m;
      a.stats[s * 3 + 1] = 0;
      a.stats[s * 3 + 2] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// Estimator: equal-component counts (estimate.py:91-95; K:958-962).
// ---------------------------------------------------------------------------

// one warp per pair; coalesced 16-byte loads
__global__ void count_equal_kernel(const uint64_t* __restrict__ A,
                                   const uint64_t* __restrict__ B,
                                   int64_t npairs, int64_t m,
                                   int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = warp; p < npairs; p += nwarps) {
    const uint64_t* a = A + p * m;
    const uint64_t* b = B + p * m;
    int c = 0;
    if ((m & 1) == 0) {
      const ulonglong2* a2 = reinterpret_cast<const ulonglong2*>(a);
      const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(b);
      for (int64_t k = lane; k < (m >> 1); k += 32) {
        ulonglong2 x = __ldg(&a2[k]), y = __ldg(&b2[k]);
        c += (x.x == y.x) + (x.y == y.y);
      }
    } else {
      for (int64_t k = lane; k < m; k += 32) c += (__ldg(&a[k]) == __ldg(&b[k]));
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[p] = c;
  }
}

// All-pairs tile: counts[i - r0][j - c0] for i in [r0,r1), j in [c0,c1) with
// j > i (upper triangle; other entries untouched).  Signatures are u64 rows;
// 64x64 pair tile per CTA, components staged through shared memory in
// k-slices of 32.
constexpr int AP_TILE = 64;
constexpr int AP_KS = 32;

__global__ void __launch_bounds__(256) allpairs_tile_kernel(
    const uint64_t* __restrict__ sigs, int64_t n, int64_t m, int64_t r0,
    int64_t r1, int64_t c0, int64_t c1, uint16_t* __restrict__ out,
    int64_t ld) {
  __shared__ uint64_t sa[AP_KS][AP_TILE + 1];
  __shared__ uint64_t sb[AP_KS][AP_TILE + 1];
  const int64_t ti = r0 + (int64_t)blockIdx.y * AP_TILE;
  const int64_t tj = c0 + (int64_t)blockIdx.x * AP_TILE;
  if (ti >= r1 || tj >= c1) return;
  if (tj + AP_TILE <= ti + 1) return;  // tile entirely on/below the diagonal
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16x16 threads, 4x4 pairs each
  int cnt[4][4];
#pragma unroll
  for (int u = 0; u < 4; u++)
#pragma unroll
    for (int v = 0; v < 4; v++) cnt[u][v] = 0;
  for (int64_t k0 = 0; k0 < m; k0 += AP_KS) {
    __syncthreads();
    for (int q = threadIdx.x; q < AP_KS * AP_TILE; q += blockDim.x) {
      const int r = q / AP_KS, kk = q % AP_KS;
      const int64_t gi = ti + r, gj = tj + r, k = k0 + kk;
      sa[kk][r] = (gi < r1 && k < m) ? sigs[gi * m + k] : 0x1ULL;
      sb[kk][r] = (gj < c1 && k < m) ? sigs[gj * m + k] : 0x2ULL;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < AP_KS; kk++) {
      uint64_t av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) av[u] = sa[kk][ty * 4 + u];
#pragma unroll
      for (int v = 0; v < 4; v++) bv[v] = sb[kk][tx * 4 + v];
#pragma unroll
      for (int u = 0; u < 4; u++)
#pragma unroll
        for (int v = 0; v < 4; v++) cnt[u][v] += (av[u] == bv[v]);
    }
  }
#pragma unroll
  for (int u = 0; u < 4; u++) {
    const int64_t i = ti + ty * 4 + u;
    if (i >= r1) continue;
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int64_t j = tj + tx * 4 + v;
      if (j < c1 && j > i) out[(i - r0) * ld + (j - c0)] = (uint16_t)cnt[u][v];
    }
  }
}

// b-bit reduction (K:851-861): component i -> low b bits of
// mix64(sig_i + GOLDEN*(i+1)); one thread per component of a [nsets, m] batch
__global__ void bbit_kernel(const uint64_t* __restrict__ sig, int64_t total,
                            int64_t m, int b, int64_t* __restrict__ out) {
  const uint64_t mask = (1ULL << (uint64_t)b) - 1ULL;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(q % m);
    out[q] = (int64_t)(mix64(sig[q] + GOLDEN * (i + 1)) & mask);
  }
}

}  // namespace pmh
