// pmh_wps.cuh -- lean warp-per-set ProbMinHash kernel for small signatures
// (m <= 64) and small sets (n <= WPS_NMAX): BASELINE configs[3] (m = 64,
// 10^6 sets of 100 elements).
//
// One warp per set, nothing shared across warps:
//   * the set's ids and weights stream into the warp's shared-memory buffer
//     with cp.async, one set ahead (the next set's copy overlaps this one's
//     work);
//   * slot table (m x 16 B, 128-bit CAS) and stop limit in shared memory;
//     the per-m constant tables in shared memory per CTA;
//   * every lane runs one element at a time through lane_step (pmh_lane.cuh)
//     and takes the next element the moment its element finishes;
//   * the lazy Fisher-Yates permutation of each lane's element (K:222-235) is
//     a dense per-lane map in shared memory, byte entries laid out [p][lane]
//     (bank-conflict free for equal p), validity in a 64-bit register mask,
//     reset per element in O(1).
// The threshold guess, verification and retry are those of the CTA kernel
// (pmh_kernel.cuh: sketch_range).  Measured and rejected on configs[3]
// (PMH2 / PMH4 ms, this kernel 23.4 / 21.7): long elements to the warp-
// cooperative mode B (55 / 59); 2, 3 or 4 sets in flight per warp, lanes
// taking elements of any of them (25 / 38, 34 / 62, 53 / 79: the context
// bookkeeping and the lower occupancy cost more than the idle lanes); 64
// registers (24 / 42: spills).
#pragma once
#include "pmh_lane.cuh"

namespace pmh {

constexpr int WPS_MMAX = 64;
#ifndef PMH_WPS_NMAX
#define PMH_WPS_NMAX 128
#endif
constexpr int WPS_NMAX = PMH_WPS_NMAX;   // largest set the warp-per-set kernel takes
constexpr int WPS_THREADS = 128;
#ifndef PMH_WPS_HEAVY_FIRST
#define PMH_WPS_HEAVY_FIRST 1
#endif
#ifndef PMH_WPS_MINB
#define PMH_WPS_MINB 6   // CTAs per SM the register budget allows (80 registers)
#endif

// per-lane dense Fisher-Yates map, m <= 64 (entries 1-based, p -> col[(p-1)*32])
struct LaneDenseFY {
  uint64_t mask;
  uint8_t* col;
  __device__ __forceinline__ void reset() { mask = 0; }
  __device__ __forceinline__ int32_t get(int32_t p) const {
    return ((mask >> (p - 1)) & 1ULL) ? (int32_t)col[(p - 1) * 32] : p;
  }
  __device__ __forceinline__ int32_t swap_step(int32_t i, int32_t j) {
    const int32_t vj = get(j), vi = get(i);
    mask |= 1ULL << (j - 1);
    col[(j - 1) * 32] = (uint8_t)vi;
    return vj;
  }
};

struct WpsWarp {
  Slot slots[WPS_MMAX];
  unsigned long long hmax;
  unsigned int filled, pad;
  uint64_t ids[2][WPS_NMAX];
  double w[2][WPS_NMAX];
  uint8_t fy[WPS_MMAX][32];   // [p][lane]
  uint8_t ord[WPS_NMAX];      // processing order of the set's elements (heaviest first)
};

__host__ __device__ inline bool wps_eligible(int family, int64_t m) {
  return m <= WPS_MMAX && m >= 2 && (family_weighted(family) || family == FAM_UW3 || family == FAM_UW4);
}

template <int F>
__global__ void __launch_bounds__(WPS_THREADS, PMH_WPS_MINB) sketch_wps_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  WpsWarp* ws = reinterpret_cast<WpsWarp*>(smem) + wid;
  const int64_t m = a.m;
  const bool weighted = family_weighted(F) && a.w;
  const int64_t n_large = (int64_t)a.counts[0];
  const int64_t n_small = a.nsets - n_large;
  const int64_t stride = (int64_t)gridDim.x * wpc;
  const double lnm = log((double)m);
  // the per-m constant tables (K:418-420, K:568-579) in shared memory: every
  // point reads them, and from global memory (even L1) their latency sits on
  // the lane's dependency chain
  __shared__ double s_beta[WPS_MMAX + 1], s_gam[WPS_MMAX], s_dgam[WPS_MMAX];
  __shared__ TruncExpConsts s_c4[WPS_MMAX];
  Tables T = a.T;
  if constexpr (F == FAM_PMH2) {
    for (int i = threadIdx.x; i <= m; i += blockDim.x) s_beta[i] = a.T.beta[i];
    T.beta = s_beta;
  } else if constexpr (F == FAM_PMH4) {
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      s_gam[i] = a.T.gam[i];
      s_dgam[i] = a.T.dgam[i];
      s_c4[i] = a.T.c4[i];
    }
    T.gam = s_gam;
    T.dgam = s_dgam;
    T.c4 = s_c4;
  }
  __syncthreads();
  // copy set bs (of the small partition) into buffer b
  auto fetch = [&](int64_t bs, int b) -> void {
    if (bs < n_small) {
      const int64_t s = (int64_t)a.order[n_large + bs];
      const int64_t off = a.offsets[s];
      const int64_t n = a.offsets[s + 1] - off;
      for (int64_t e = lane; e < n && e < WPS_NMAX; e += 32) {
        cp_async8(&ws->ids[b][e], a.ids + off + e);
        if (weighted) cp_async8(&ws->w[b][e], a.w + off + e);
      }
    }
    cp_async_commit();
  };
  int64_t bs = (int64_t)blockIdx.x * wpc + wid;
  int buf = 0;
  fetch(bs, 0);
  for (; bs < n_small; bs += stride, buf ^= 1) {
    fetch(bs + stride, buf ^ 1);
    const int64_t s = (int64_t)a.order[n_large + bs];
    const int64_t n = a.offsets[s + 1] - a.offsets[s];
    if (n <= 0 || n > WPS_NMAX) {
      PMH_ASSERT(n <= WPS_NMAX);
      if (lane == 0) atomicMin(a.err_set, (long long)s);
      cp_async_wait_group1();
      continue;
    }
    for (int64_t k = lane; k < m; k += 32) { ws->slots[k].h = EMPTY_H; ws->slots[k].idx = EMPTY_IDX; }
    if (lane == 0) { ws->hmax = EMPTY_H; ws->filled = 0; }
    cp_async_wait_group1();
    __syncwarp();
    const uint64_t* ids = ws->ids[buf];
    const double* w = ws->w[buf];
    double W = 0.0;
    if (weighted && a.setw && a.setw[s] > 0.0) {
      W = a.setw[s];
    } else if (weighted) {
      for (int64_t e = lane; e < n; e += 32) W += w[e];
      for (int o = 16; o > 0; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
    } else {
      W = (double)n;
    }
    SetCtx c;
    c.slots = ws->slots;
    c.hmax_bits = &ws->hmax;
    c.filled = &ws->filled;
    c.m = (int32_t)m;
    c.kbits = bits_for(m);
    c.cap = (int32_t)coupon_cap(m);
    c.points = 0; c.updates = 0; c.multi = 0; c.tprev = -1.0; c.since_refresh = 0;
    c.trig = false;
    c.eoff = 0;
    double tg = (double)m * (lnm + a.tconst) / W;
    if (!(tg > 0.0)) tg = __longlong_as_double(0x7FF0000000000000LL);
    bool failed = false;
    // Heaviest first (longest-processing-time order): an element's point
    // count is ~ t w (at most m without replacement), so with skewed weights
    // (configs[3]: Pareto 1.5) a heavy element taken last leaves its lane
    // running alone while the other lanes idle at the end of the set.  A
    // counting sort on floor(log2(1 + t w)) (8 buckets, descending) orders
    // the lanes' refill; element indices (the tie-break) are unchanged.
    if (weighted && PMH_WPS_HEAVY_FIRST) {
      int key[WPS_NMAX / 32];
      int base[8];
#pragma unroll
      for (int r = 0; r < WPS_NMAX / 32; r++) {
        const int64_t e = lane + 32 * r;
        key[r] = -1;
        if (e < n) {
          const double pts = tg * w[e];
          const int k = pts < 1.0 ? 0 : 1 + ilogb(pts);
          key[r] = k > 7 ? 7 : k;
        }
      }
      const unsigned lt = (1u << lane) - 1u;
      int run = 0;
#pragma unroll
      for (int b = 7; b >= 0; b--) {
        base[b] = run;
#pragma unroll
        for (int r = 0; r < WPS_NMAX / 32; r++) run += __popc(__ballot_sync(0xffffffffu, key[r] == b));
      }
#pragma unroll
      for (int r = 0; r < WPS_NMAX / 32; r++) {
#pragma unroll
        for (int b = 7; b >= 0; b--) {
          const unsigned mk = __ballot_sync(0xffffffffu, key[r] == b);
          if (key[r] == b) ws->ord[base[b] + __popc(mk & lt)] = (uint8_t)(lane + 32 * r);
          base[b] += __popc(mk);
        }
      }
    } else {
      for (int64_t e = lane; e < n; e += 32) ws->ord[e] = (uint8_t)e;
    }
    __syncwarp();
    LaneElT<LaneDenseFY> st;
    st.fy.col = &ws->fy[0][lane];
    st.e = 0;
    for (int attempt = 0;; attempt++) {
      c.tguess = tg;
      // lane refill over the set's elements
      int64_t next = 0;
      bool act = false;
      const unsigned lt = (1u << lane) - 1u;
      for (;;) {
        unsigned am = __ballot_sync(0xffffffffu, act);
        while (am != 0xffffffffu && next < n) {
          // idle lanes take the next elements in order
          const int idle = 32 - __popc(am);
          const int take = n - next < idle ? (int)(n - next) : idle;
          const int rank = __popc(~am & lt);
          if (!act && rank < take) {
            const int32_t e = (int32_t)ws->ord[next + rank];
            const double winv = weighted ? 1.0 / w[e] : 1.0;
            act = lane_init<F>(c, T, st, e, ids[e], winv, ctx_thr(c));
          }
          next += take;
          am = __ballot_sync(0xffffffffu, act);
        }
        if (am == 0) break;
        if (act) {
          const int r = lane_step<F>(c, T, st, ctx_thr(c));
          if (r != EL_CONT) {
            act = false;
            if (r == EL_FAIL) failed = true;
          }
        }
        if (__any_sync(0xffffffffu, c.trig)) {
          c.trig = false;
          hmax_refresh_warp(c, lane);
        }
      }
      unsigned long long mx = 0;
      for (int64_t k = lane; k < m; k += 32) {
        const unsigned long long h = ws->slots[k].h;
        mx = h > mx ? h : mx;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx ? v : mx;
      }
      if (__any_sync(0xffffffffu, failed) || !(__longlong_as_double((long long)mx) > tg)) break;
      c.tprev = tg;
      tg = attempt >= 2 ? __longlong_as_double(0x7FF0000000000000LL) : tg * 4.0;
    }
    if (__any_sync(0xffffffffu, failed) && lane == 0) {
      atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
      atomicMin(a.err_set, (long long)s);
    }
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = lane; k < m; k += 32) {
      const unsigned long long ix = ws->slots[k].idx;
      sig[k] = ix < (unsigned long long)n ? ids[ix] : 0ULL;
    }
    if (a.stats) {
      long long pts = c.points, upd = c.updates, mul = c.multi;
      for (int o = 16; o > 0; o >>= 1) {
        pts += __shfl_xor_sync(0xffffffffu, pts, o);
        upd += __shfl_xor_sync(0xffffffffu, upd, o);
        mul += __shfl_xor_sync(0xffffffffu, mul, o);
      }
      if (lane == 0) {
        a.stats[s * 3 + 0] = pts;
        a.stats[s * 3 + 1] = mul;
        a.stats[s * 3 + 2] = upd;
      }
    }
    __syncwarp();
  }
  cp_async_wait_all();
}

}  // namespace pmh
