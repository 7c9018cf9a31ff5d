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
#include "pmh_split.cuh"

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
  // order[0, split_info[0]) are split across CTAs (pmh_split.cuh) and skipped
  // by the one-CTA-per-set kernel; nullptr: no split
  const long long* split_info;
  const double* setw;   // device [nsets] total weights known in advance, or nullptr
};

constexpr int PMIN_THREADS = 256;
constexpr int PMIN_CHUNK = 256;

// Thread (g, t) owns components [t*C, t*C + C) and walks elements g, g+G, ...
// of its set in increasing order; G groups of ceil(m/C) threads per CTA.
//
// Hot loop (almost every draw is rejected once the minima are small): with
// T_t = max of the thread's C running minima and sw(e) = w_e * 2^53 * (1 +
// 2^-40), any draw with raw bits b >= Tb = ceil(T_t * sw(e)) + 1 satisfies
// fl(winv * E(b)) >= winv * b * 2^-53 * (1 - 2^-51) > T_t >= hmin_q, so it
// cannot lower any of the thread's minima: the per-draw work is integer
// only (splitmix64 words, a funnel-shift extraction and one 64-bit compare).
// Draws below Tb take the exact path: the reference's
// h = winv * (-log1p(-U)) with glibc-exact log1p and strict `<`.
//
// EXPO = true: P-MinHash (K:284-300); EXPO = false: MinHash h = U (K:768-781).
template <int C, bool EXPO>
__global__ void __launch_bounds__(PMIN_THREADS) pminhash_kernel(PMinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ uint64_t s_id[PMIN_CHUNK];
  __shared__ double s_winv[PMIN_CHUNK];
  __shared__ double s_sw[PMIN_CHUNK];
  const int64_t m = a.m;
  const int tpg = (int)((m + C - 1) / C);          // threads per group
  const int groups = PMIN_THREADS / tpg;           // >= 1 (host guarantees)
  const int g = threadIdx.x / tpg, t = threadIdx.x % tpg;
  const bool active = g < groups;
  const int64_t k0 = (int64_t)t * C;
  Slot* table = reinterpret_cast<Slot*>(smem);     // [m] merged minima
  const double two53m = 9007199254740992.0 * 1.0000000000009095;  // 2^53 (1 + 2^-40)

  for (int64_t bs = blockIdx.x; bs < a.nsets; bs += gridDim.x) {
    const int64_t s = a.order ? (int64_t)a.order[bs] : bs;
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      table[k].h = EMPTY_H;
      table[k].idx = EMPTY_IDX;
    }
    double hmin[C];
    uint32_t arg[C];
#pragma unroll
    for (int q = 0; q < C; q++) { hmin[q] = __longlong_as_double(0x7FF0000000000000LL); arg[q] = 0xFFFFFFFFu; }
    double tmax = __longlong_as_double(0x7FF0000000000000LL);   // max_q hmin[q]

    for (int64_t c0 = 0; c0 < n; c0 += PMIN_CHUNK) {
      const int64_t cn = n - c0 < PMIN_CHUNK ? n - c0 : PMIN_CHUNK;
      __syncthreads();
      if (threadIdx.x < cn) {
        s_id[threadIdx.x] = a.ids[off + c0 + threadIdx.x];
        if (EXPO) {
          const double w = a.w ? a.w[off + c0 + threadIdx.x] : 1.0;
          s_winv[threadIdx.x] = 1.0 / w;
          s_sw[threadIdx.x] = w * two53m;
        } else {
          s_sw[threadIdx.x] = two53m;
        }
      }
      __syncthreads();
      if (!active) continue;
      for (int64_t le = g; le < cn; le += groups) {
        const uint64_t id = s_id[le];
        const uint32_t e = (uint32_t)(c0 + le);
        // integer rejection threshold for this element
        const double tb = tmax * s_sw[le];
        const uint64_t Tb = tb < 9007199254740992.0 ? (uint64_t)tb + 1ULL : (1ULL << 53);
        uint64_t bitpos = 53ULL * (uint64_t)k0;
        uint64_t wi = bitpos >> 6;                  // 0-based word index
        uint32_t sh = (uint32_t)(bitpos & 63);
        uint64_t st = id + (wi + 1) * GOLDEN;
        uint64_t lo = mix64(st);
        st += GOLDEN;
        uint64_t hi = mix64(st);
        bool changed = false;
#pragma unroll
        for (int q = 0; q < C; q++) {
          if (k0 + q < m) {
            uint64_t b = sh ? ((lo >> sh) | (hi << (64 - sh))) : lo;
            b &= (1ULL << 53) - 1ULL;
            if (b < Tb) {
              if constexpr (EXPO) {
                const double winv = s_winv[le];
                if (!(exp1_scaled_lower_bound(winv, b) > hmin[q])) {
                  const double h = winv * exp1_from_bits(b);
                  if (h < hmin[q]) { hmin[q] = h; arg[q] = e; changed = true; }
                }
              } else {
                const double h = (double)b * INV53;
                if (h < hmin[q]) { hmin[q] = h; arg[q] = e; changed = true; }
              }
            }
          }
          sh += 53;
          if (sh >= 64) {
            sh -= 64;
            lo = hi;
            if (q + 1 < C) { st += GOLDEN; hi = mix64(st); }
          }
        }
        if (changed) {
          double mx = 0.0;
#pragma unroll
          for (int q = 0; q < C; q++)
            if (k0 + q < m) mx = hmin[q] > mx ? hmin[q] : mx;
          tmax = mx;
        }
      }
    }
    // merge the groups' partial minima lexicographically on (h, index)
    __syncthreads();
    if (active) {
#pragma unroll
      for (int q = 0; q < C; q++)
        if (k0 + q < m && arg[q] != 0xFFFFFFFFu)
          slot_offer(&table[k0 + q], hmin[q], (unsigned long long)arg[q]);
    }
    __syncthreads();
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const unsigned long long bi = table[k].idx;
      sig[k] = bi < (unsigned long long)n ? a.ids[off + bi] : 0ULL;
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = n * m;
      a.stats[s * 3 + 1] = 0;
      a.stats[s * 3 + 2] = 0;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Static-schedule variant for m % 64 == 0 (every configuration): thread t of
// a 16-lane... group owns components [64t, 64t + 64), whose 64 * 53 = 3392 bits
// are exactly words 53t .. 53t + 52 of each element's stream, so every bit
// extraction below has a compile-time shift.  The hot loop keeps only the
// TOP 32 bits of each draw: b < Tb implies (b >> 21) <= ((Tb - 1) >> 21), so
// testing top32 <= Tb_hi flags a superset of the candidates (false positives
// only on top-bit ties, probability 2^-32).  Minima live in ONE shared slot
// table per CTA (128-bit CAS, lexicographic (h, index)); every group of
// threads refreshes its rejection threshold tmax from that table, so all
// groups prune with everyone's minima.
// ---------------------------------------------------------------------------
constexpr int PM64_C = 64;
#ifndef PM64_REFRESH
// elements between threshold refreshes (configs[1], after the candidate-scan
// skip: 8 / 16 / 32 / 64 / 128 -> 74.2 / 72.6 / 71.9 / 71.5 / 71.4 ms; the
// threshold only moves slowly below its guess, so fresher is not better)
#define PM64_REFRESH 64
#endif
#ifndef PM64_TCONST
#define PM64_TCONST 8.0    // threshold guess (ln m + c) / W
#endif
#ifndef PM64_CQ_SIZE
#define PM64_CQ_SIZE 128   // 64 / 128 / 256: equal within 0.2% on configs[1]
#endif
constexpr int PM64_CQ = PM64_CQ_SIZE;   // queued candidates per warp

// Shared table layout: component k = 64 t + q (thread t, draw q) lives at
// TRANSPOSED index q * tpg + t, so the 16..32 threads of a warp touch
// consecutive 16-byte entries when they walk their own 64 components
// (conflict-free refresh).
__device__ __forceinline__ int64_t pm64_slot(int64_t t, int q, int tpg) {
  return (int64_t)q * tpg + t;
}

// exact check of draw q of thread t for element e (1-2 stream words and a
// compare against the slot's own minimum; the log only when that passes)
template <bool EXPO>
__device__ __forceinline__ void pm64_check(uint64_t id, double winv, uint32_t e, int64_t t,
                                           int q, int tpg, Slot* table) {
  const uint64_t bitpos = 53ULL * (uint64_t)(t * PM64_C + q);
  const uint64_t wi = bitpos >> 6;
  const uint32_t sh = (uint32_t)(bitpos & 63);
  const uint64_t lo = stream_word(id, wi + 1);
  uint64_t b = lo >> sh;
  if (sh > 11) b |= stream_word(id, wi + 2) << (64 - sh);
  b &= (1ULL << 53) - 1ULL;
  PMH_ASSERT(t * PM64_C + q < (int64_t)tpg * PM64_C && q >= 0 && q < PM64_C);
  Slot* sl = &table[pm64_slot(t, q, tpg)];
  const double cur = __longlong_as_double((long long)*(volatile unsigned long long*)&sl->h);
  double h;
  if constexpr (EXPO) {
    if (exp1_scaled_lower_bound(winv, b) > cur) return;
    h = winv * exp1_from_bits(b);
  } else {
    h = (double)b * INV53;
  }
  if (h <= cur) slot_offer(sl, h, (unsigned long long)e);
}

// exact path for all flagged draws of one element (the divergent fallback:
// a group's first elements, while its threshold is still infinite)
template <bool EXPO>
__device__ __noinline__ void pm64_candidates(uint64_t cand, uint64_t id, double w, uint32_t e,
                                             int64_t t, int tpg, Slot* table) {
  const double winv = EXPO ? 1.0 / w : 1.0;
  while (cand) {
    const int q = __ffsll((long long)cand) - 1;
    cand &= cand - 1;
    pm64_check<EXPO>(id, winv, e, t, q, tpg, table);
  }
}

// one queued candidate per lane: (element, t << 6 | q)
template <bool EXPO>
__device__ __noinline__ void pm64_check_entry(uint2 en, const uint64_t* ids, const double* ws,
                                              int tpg, Slot* table) {
  const uint64_t id = __ldg(&ids[en.x]);
  const double winv = (EXPO && ws) ? 1.0 / __ldg(&ws[en.x]) : 1.0;
  pm64_check<EXPO>(id, winv, en.x, (int64_t)(en.y >> 6), (int)(en.y & 63u), tpg, table);
}

__device__ __forceinline__ double pm64_tmax(const Slot* table, int64_t t, int tpg) {
  unsigned long long mx = 0;
#pragma unroll 8
  for (int q = 0; q < PM64_C; q++) {
    const unsigned long long h =
        *(volatile const unsigned long long*)&table[pm64_slot(t, q, tpg)].h;
    mx = h > mx ? h : mx;
  }
  return __longlong_as_double((long long)mx);
}

// Each group of tpg = m/64 threads walks its elements g, g + G, ... straight
// from global memory (broadcast loads, next element prefetched): no block
// barrier inside a set, so warps with more candidates do not stall the CTA.
// st + (chi:clo): the low word on the ALU with carry-out, the high word as a
// multiply-add with carry-in (IMAD.X, FMA pipe).  `one` is 1 loaded from
// shared memory per element, so ptxas can neither fold nor hoist the product.
template <uint32_t CLO, uint32_t CHI>
__device__ __forceinline__ uint64_t add_fma_t(uint64_t st, uint32_t one) {
  uint64_t z;
  asm("{\n\t.reg .u32 l, h, sl, sh;\n\t"
      "mov.b64 {sl, sh}, %2;\n\t"
      "add.cc.u32 l, sl, %3;\n\t"
      "madc.lo.u32 h, %1, %4, sh;\n\t"
      "mov.b64 %0, {l, h};\n\t}"
      : "=l"(z) : "r"(one), "l"(st), "n"(CLO), "n"(CHI));
  return z;
}
#define add_fma(st, one, clo, chi) add_fma_t<clo, chi>(st, one)


// Exact (verified) minima of elements [e0, e1) of the set at `off` into the
// shared `table` (all threads of the CTA; returns after a final barrier).
// The threshold guess uses the range's own weight sum: the minima over a
// range are Exp(W_range), and the verification makes any guess exact-safe.
template <bool EXPO>
__device__ __forceinline__ void pm64_range(const PMinArgs& a, int64_t off, int64_t e0, int64_t e1,
                                           Slot* table, unsigned char* smem, uint32_t* s_onep,
                                           double* s_wsum, int* s_retryp, double w_given) {
  const int64_t m = a.m;
  const int tpg = (int)(m / PM64_C);               // threads per group
  const int groups = PMIN_THREADS / tpg;
  const int g = threadIdx.x / tpg, t = threadIdx.x % tpg;
  const bool active = g < groups;
  const double two53m = 9007199254740992.0 * 1.0000000000009095;  // 2^53 (1 + 2^-40)
  const uint64_t wbase = 53ULL * (uint64_t)t + 1ULL;                // first word (1-based)
  uint32_t& s_one = *s_onep;
  int& s_retry = *s_retryp;
  // Threshold guess: every slot minimum is Exp(W) (W = total weight), so
  // tg = (ln m + PM64_TCONST) / W bounds all m of them unless a rare set
  // (~m e^-(ln m + c) = e^-c) exceeds it; the final table is verified and
  // such a set re-runs with 4 tg, then without a bound.  Draws above tg are
  // never candidates, so no element starts with an infinite threshold.
  double W;
  if (EXPO && a.w && w_given > 0.0) {
    W = w_given;   // known in advance (SketchArgs.setw): no weight pre-pass
    __syncthreads();   // (the pre-pass's barrier also fenced the previous set's table reads)
  } else if (EXPO && a.w) {
    double p = 0.0;
    for (int64_t k = e0 + threadIdx.x; k < e1; k += blockDim.x) p += __ldg(&a.w[off + k]);
    for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
    if ((threadIdx.x & 31) == 0) s_wsum[threadIdx.x >> 5] = p;
    __syncthreads();
    W = 0.0;
    for (int k = 0; k < PMIN_THREADS / 32; k++) W += s_wsum[k];
  } else {
    W = (double)(e1 - e0);
  }
  const double inf_d = __longlong_as_double(0x7FF0000000000000LL);
  double tg = (log((double)m) + PM64_TCONST) / W;
  if (!(tg > 0.0) || !(tg < 1e300)) tg = inf_d;
  for (int attempt = 0;; attempt++) {
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      table[k].h = EMPTY_H;
      table[k].idx = EMPTY_IDX;
    }
    __syncthreads();
    if (active) {
      const uint64_t* ids = a.ids + off;
      const double* ws = (EXPO && a.w) ? a.w + off : nullptr;
      double tmax = tg;
      int since = 0;
      // groups per warp (2 when m = 1024): the trip count is made warp-uniform
      // so a full-warp __syncwarp can reconverge the lanes every element
      const int gpw = tpg >= 32 ? 1 : 32 / tpg;
      const int gsub = g % gpw;
      int64_t ew = e0 + g - gsub;                  // first group of this warp
      int64_t e = ew + gsub;
      // per-warp candidate queue (warp-aligned groups only: the trip count
      // and every lane must be warp-uniform for the collectives)
      const bool use_q = (32 % tpg == 0) || (tpg % 32 == 0);
      const int lane = threadIdx.x & 31;
      uint2* cq = reinterpret_cast<uint2*>(smem + sizeof(Slot) * m) + (threadIdx.x >> 5) * PM64_CQ;
      int qn = 0;
      uint64_t id_n = e < e1 ? __ldg(&ids[e]) : 0;
      double w_n = (ws && e < e1) ? __ldg(&ws[e]) : 1.0;
      for (; ew < e1; ew += groups) {
        e = ew + gsub;
        const bool live = e < e1;
        const uint64_t id = id_n;
        const double w = w_n;
        if (e + groups < e1) {                     // prefetch the next element
          id_n = __ldg(&ids[e + groups]);
          if (ws) w_n = __ldg(&ws[e + groups]);
        }
        const double tb = tmax * (w * two53m);
        // b < Tb = floor(tb) + 1  =>  b >> 21 <= tb >> 21
        const uint32_t tbh = tb < 9007199254740992.0 ? (uint32_t)((uint64_t)tb >> 21)
                                                      : 0xFFFFFFFFu;
        uint64_t st = id + wbase * GOLDEN;
        const uint32_t one = *(volatile uint32_t*)&s_one;
        uint32_t c_lo = 0, c_hi = 0;
#define MIXZ mix64_z
#define PM64_TEST(x, thr, mask, bit) if ((x) <= (thr)) mask |= (bit)
#include "pm64_body.inc"
#undef PM64_TEST
#undef MIXZ
        const uint64_t cand = live ? (((uint64_t)c_hi << 32) | c_lo) : 0ULL;
        // candidates are cheap (1-2 stream words + a compare against the
        // slot's own minimum) but scattered: a few lanes per warp-step.  They
        // are queued per warp and checked 32 at a time with every lane busy;
        // only the all-candidate start (infinite threshold) or a queue
        // overflow runs them in place.  The threshold refresh is periodic --
        // a stale, larger tmax only admits more candidates.
        const bool inf = !(tmax < 1e300);
        // most warp-steps of a large set have no candidate at all: skip the scan
        if (use_q && __any_sync(0xffffffffu, cand != 0ULL)) {
          const int c = __popcll(cand);
          int x = c;                                   // inclusive lane scan
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          const int total = __shfl_sync(0xffffffffu, x, 31);
          const bool direct = __any_sync(0xffffffffu, inf) || qn + total > PM64_CQ;
          if (direct) {
            if (cand) pm64_candidates<EXPO>(cand, id, w, (uint32_t)e, t, tpg, table);
          } else if (total) {
            int pos = qn + x - c;
            for (uint64_t cb = cand; cb; cb &= cb - 1) {
              PMH_ASSERT(pos < PM64_CQ);
              cq[pos++] = make_uint2((uint32_t)e, ((uint32_t)t << 6) | (uint32_t)(__ffsll((long long)cb) - 1));
            }
            qn += total;
            __syncwarp();
            while (qn >= 32) {
              qn -= 32;
              const uint2 en = cq[qn + lane];
              __syncwarp();
              pm64_check_entry<EXPO>(en, ids, ws, tpg, table);
            }
          }
        } else if (!use_q && cand) {
          pm64_candidates<EXPO>(cand, id, w, (uint32_t)e, t, tpg, table);
        }
        if (++since >= PM64_REFRESH || (cand && inf)) {
          tmax = fmin(pm64_tmax(table, t, tpg), tg);
          since = 0;
        }
        // reconverge: lanes that took the candidate path would otherwise run
        // the straight-line body out of phase (independent thread scheduling)
        __syncwarp();
      }
      if (use_q && lane < qn) pm64_check_entry<EXPO>(cq[lane], ids, ws, tpg, table);
    }
    __syncthreads();
    // verification: every slot filled and <= tg
    {
      unsigned long long mx = 0;
      for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        const unsigned long long h = table[k].h;
        mx = h > mx ? h : mx;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx ? v : mx;
      }
      if (threadIdx.x == 0) s_retry = 0;
      __syncthreads();
      if ((threadIdx.x & 31) == 0 && __longlong_as_double((long long)mx) > tg) atomicOr(&s_retry, 1);
      __syncthreads();
      const int retry = s_retry;
      __syncthreads();
      if (!retry || !(tg < 1e300)) break;
      tg = attempt >= 1 ? inf_d : tg * 4.0;
    }
  }
}

#ifndef PM64_MINBLOCKS
#define PM64_MINBLOCKS 4   // 64 registers, 4 CTAs (32 warps) per SM
#endif
template <bool EXPO>
__global__ void __launch_bounds__(PMIN_THREADS, PM64_MINBLOCKS) pminhash64_kernel(PMinArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t m = a.m;
  const int tpg = (int)(m / PM64_C);
  Slot* table = reinterpret_cast<Slot*>(smem);
  __shared__ uint32_t s_one;
  __shared__ double s_wsum[PMIN_THREADS / 32];
  __shared__ int s_retry;
  if (threadIdx.x == 0) s_one = 1u;
  __syncthreads();
  // the split sets (an order prefix) belong to pminhash64_split_kernel
  const int64_t first = a.split_info ? (int64_t)a.split_info[0] : 0;
  for (int64_t bs = first + blockIdx.x; bs < a.nsets; bs += gridDim.x) {
    const int64_t s = a.order ? (int64_t)a.order[bs] : bs;
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    pm64_range<EXPO>(a, off, 0, n, table, smem, &s_one, s_wsum, &s_retry,
                     a.setw ? a.setw[s] : -1.0);
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const unsigned long long bi = table[pm64_slot(k / PM64_C, (int)(k % PM64_C), tpg)].idx;
      sig[k] = bi < (unsigned long long)n ? a.ids[off + bi] : 0ULL;
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = n * m;
      a.stats[s * 3 + 1] = 0;
      a.stats[s * 3 + 2] = 0;
    }
    __syncthreads();
  }
}

// ---- large sets split across CTAs ------------------------------------------
// One CTA per set caps a set's speed at one SM (a 10^6-element set at m = 1024
// would take ~0.4 s alone).  The largest sets (an LPT-order prefix, n >=
// split_n) are cut into parts of <= split_n elements; persistent CTAs take
// parts from a counter, compute each part's exact minima in shared memory
// (pm64_range) and merge them into the set's global table with 128-bit CAS
// (lexicographic (h, index): the merge is order-independent), and a final
// pass writes the ids.

template <bool EXPO>
__global__ void __launch_bounds__(PMIN_THREADS, PM64_MINBLOCKS)
    pminhash64_split_kernel(PMinArgs a, SplitArgs sp) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t m = a.m;
  const int tpg = (int)(m / PM64_C);
  Slot* table = reinterpret_cast<Slot*>(smem);
  __shared__ uint32_t s_one;
  __shared__ double s_wsum[PMIN_THREADS / 32];
  __shared__ int s_retry;
  __shared__ long long s_t;
  if (threadIdx.x == 0) s_one = 1u;
  SplitPart p;
  while (split_next_part(sp, &s_t, &p)) {
    pm64_range<EXPO>(a, p.off, p.e0, p.e1, table, smem, &s_one, s_wsum, &s_retry, -1.0);
    Slot* gt = sp.gtab + (size_t)p.i * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const Slot v = table[pm64_slot(k / PM64_C, (int)(k % PM64_C), tpg)];
      if (v.idx != EMPTY_IDX) slot_offer_global(&gt[k], v.h, v.idx);
    }
    if (a.stats && threadIdx.x == 0)
      atomicAdd((unsigned long long*)&a.stats[p.s * 3], (unsigned long long)((p.e1 - p.e0) * m));
    __syncthreads();
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

// c += (a == b) as a compare and a predicated add (the compiler's own
// lowering is compare, increment, predicated move: 3 instructions)
__device__ __forceinline__ void acc_eq32(uint32_t& c, uint32_t a, uint32_t b) {
  asm("{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
      : "+r"(c) : "r"(a), "r"(b));
}
__device__ __forceinline__ void acc_eq64(uint32_t& c, uint64_t a, uint64_t b) {
  asm("{\n\t.reg .pred p;\n\tsetp.eq.u64 p, %1, %2;\n\t@p add.u32 %0, %0, 1;\n\t}"
      : "+r"(c) : "l"(a), "l"(b));
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
  uint32_t cnt[4][4];
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
        for (int v = 0; v < 4; v++) acc_eq64(cnt[u][v], av[u], bv[v]);
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

// All-pairs reduction (configs[4]): persistent CTAs walk the 64x64 pair
// tiles of rows [r0,r1) x cols [c0,c1) (upper triangle j > i only), count
// equal components exactly (64-bit compares of the staged signatures), and
// reduce on the fly: a per-CTA shared histogram of the counts (flushed once
// to `hist`, m+1 bins) and, for count >= thr, the pair appended to `pairs`
// as (i << 32 | j, count) through a global cursor (dropped beyond `cap`; the
// cursor still counts them).  No dense count matrix is materialised.
// Comparison policies for the all-pairs reduction.  EqU64: rows of m full
// signature components, count = number of equal components.  BBitNeq: rows
// of W packed b-bit words (bbit_pack_kernel), per word the number of UNEQUAL
// b-bit fields by a carry-free SWAR test -- t = (x & L) + L sets each field's
// top bit iff its low b-1 bits are nonzero (L = low b-1 bits of every field,
// H = top bit of every field), nz = (t | x) & H -- so count = m - sum popc.
// Padding fields are zero in both rows and never counted as unequal.
struct EqU64 {
  __device__ __forceinline__ uint32_t op(uint64_t a, uint64_t b) const { return a == b; }
  __device__ __forceinline__ void acc(uint32_t& c, uint64_t a, uint64_t b) const { acc_eq64(c, a, b); }
  __device__ __forceinline__ int64_t finish(uint32_t c) const { return c; }
};
struct BBitNeq {
  uint64_t L, H;
  int64_t m;
  __device__ __forceinline__ uint32_t op(uint64_t a, uint64_t b) const {
    const uint64_t x = a ^ b;
    return (uint32_t)__popcll((((x & L) + L) | x) & H);
  }
  __device__ __forceinline__ void acc(uint32_t& c, uint64_t a, uint64_t b) const { c += op(a, b); }
  __device__ __forceinline__ int64_t finish(uint32_t c) const { return m - (int64_t)c; }
};
// compile-time masks for the common b (the b = 1 case reduces to popc(a ^ b))
template <int B>
struct BBitNeqT {
  int64_t m;
  __host__ __device__ static constexpr uint64_t mask_h() {
    uint64_t h = 0;
    for (int f = 0; f < 64 / B; f++) h |= 1ULL << (f * B + B - 1);
    return h;
  }
  __host__ __device__ static constexpr uint64_t mask_l() {
    uint64_t l = 0;
    for (int f = 0; f < 64 / B; f++) l |= ((1ULL << (B - 1)) - 1ULL) << (f * B);
    return l;
  }
  __device__ __forceinline__ uint32_t op(uint64_t a, uint64_t b) const {
    const uint64_t x = a ^ b;
    if constexpr (B == 1) {
      return (uint32_t)__popcll(x);
    } else {
      constexpr uint64_t L = mask_l(), H = mask_h();
      return (uint32_t)__popcll((((x & L) + L) | x) & H);
    }
  }
  __device__ __forceinline__ void acc(uint32_t& c, uint64_t a, uint64_t b) const { c += op(a, b); }
  __device__ __forceinline__ int64_t finish(uint32_t c) const { return m - (int64_t)c; }
};

// Tiled all-pairs reduction over rows of `len` words (len = m for EqU64, W
// for BBitNeq): 64x64 pair tiles, words staged through shared memory in
// slices of 32, counts reduced on the fly into a per-CTA histogram (m+1
// bins, flushed once) and the pairs with count >= thr appended as
// (i << 32 | j, count) through a global cursor (dropped beyond `cap`; the
// cursor still counts them).  No dense count matrix is materialised.
template <class Cmp>
__global__ void __launch_bounds__(256) allpairs_reduce_kernel(
    const uint64_t* __restrict__ sigs, int64_t len, int64_t m, Cmp cmp, int64_t r0, int64_t r1,
    int64_t c0, int64_t c1, int32_t thr, unsigned long long* __restrict__ hist,
    unsigned long long* __restrict__ pairs, int64_t cap, unsigned long long* __restrict__ cursor,
    const unsigned long long* __restrict__ gate = nullptr, unsigned long long gate_cap = 0) {
  // gate (two-stage exact path): run only when the candidate list overflowed
  if (gate && *gate <= gate_cap) return;
  extern __shared__ __align__(16) unsigned char smem[];
  uint64_t (*sa)[AP_TILE + 1] = reinterpret_cast<uint64_t (*)[AP_TILE + 1]>(smem);
  uint64_t (*sb)[AP_TILE + 1] =
      reinterpret_cast<uint64_t (*)[AP_TILE + 1]>(smem + sizeof(uint64_t) * AP_KS * (AP_TILE + 1));
  unsigned int* shist =
      reinterpret_cast<unsigned int*>(smem + 2 * sizeof(uint64_t) * AP_KS * (AP_TILE + 1));
  for (int64_t b = threadIdx.x; b <= m; b += blockDim.x) shist[b] = 0;
  __syncthreads();
  const int64_t nti = (r1 - r0 + AP_TILE - 1) / AP_TILE, ntj = (c1 - c0 + AP_TILE - 1) / AP_TILE;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int64_t t = blockIdx.x; t < nti * ntj; t += gridDim.x) {
    const int64_t ti = r0 + (t / ntj) * AP_TILE, tj = c0 + (t % ntj) * AP_TILE;
    if (tj + AP_TILE <= ti + 1) continue;  // entirely on/below the diagonal
    uint32_t cnt[4][4];
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
      for (int v = 0; v < 4; v++) cnt[u][v] = 0;
    for (int64_t k0 = 0; k0 < len; k0 += AP_KS) {
      __syncthreads();
      for (int q = threadIdx.x; q < AP_KS * AP_TILE; q += blockDim.x) {
        const int r = q / AP_KS, kk = q % AP_KS;
        const int64_t gi = ti + r, gj = tj + r, k = k0 + kk;
        // out-of-range words: equal in both operands for every policy, the
        // results of out-of-range rows are discarded
        sa[kk][r] = (gi < r1 && k < len) ? __ldg(&sigs[gi * len + k]) : 0ULL;
        sb[kk][r] = (gj < c1 && k < len) ? __ldg(&sigs[gj * len + k]) : 0ULL;
      }
      __syncthreads();
      const int kn = len - k0 < AP_KS ? (int)(len - k0) : AP_KS;
#pragma unroll 4
      for (int kk = 0; kk < kn; kk++) {
        uint64_t av[4], bv[4];
#pragma unroll
        for (int u = 0; u < 4; u++) av[u] = sa[kk][ty * 4 + u];
#pragma unroll
        for (int v = 0; v < 4; v++) bv[v] = sb[kk][tx * 4 + v];
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int v = 0; v < 4; v++) cmp.acc(cnt[u][v], av[u], bv[v]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t i = ti + ty * 4 + u;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int64_t j = tj + tx * 4 + v;
        if (i < r1 && j < c1 && j > i) {
          const int64_t c = cmp.finish(cnt[u][v]);
          atomicAdd(&shist[c], 1u);
          if (c >= thr) {
            const unsigned long long pos = atomicAdd(cursor, 1ULL);
            if ((int64_t)pos < cap) {
              pairs[2 * pos] = ((unsigned long long)i << 32) | (unsigned long long)j;
              pairs[2 * pos + 1] = (unsigned long long)c;
            }
          }
        }
      }
    }
  }
  __syncthreads();
  for (int64_t b = threadIdx.x; b <= m; b += blockDim.x)
    if (shist[b]) atomicAdd(&hist[b], (unsigned long long)shist[b]);
}

// Two-stage exact all-pairs (EqU64 semantics at about half the ALU work):
// stage 1 compares only the LOW 32 bits of every component pair.  A pair
// whose low words never match has an exact count of 0 (counted into *zeros);
// every other pair is appended to a candidate list (dropped beyond ccap; the
// cursor still counts them).  Stage 2 recounts the candidates exactly (64-bit
// compares, warp per pair) into hist / pairs; stage 3 adds the zeros.  If the
// list overflowed, stages 2-3 do nothing and the gated exact reduction
// (allpairs_reduce_kernel<EqU64>) recomputes the range instead -- all
// decided on the device, no host synchronisation.
constexpr int AP_PAD32 = 4;   // keeps each 4-row group 16-byte aligned (LDS.128)
__global__ void __launch_bounds__(256) allpairs_lo_kernel(
    const uint64_t* __restrict__ sigs, int64_t m, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
    unsigned long long* __restrict__ zeros, unsigned long long* __restrict__ cand, int64_t ccap,
    unsigned long long* __restrict__ ccursor) {
  __shared__ __align__(16) uint32_t sa[AP_KS][AP_TILE + AP_PAD32];
  __shared__ __align__(16) uint32_t sb[AP_KS][AP_TILE + AP_PAD32];
  const int64_t nti = (r1 - r0 + AP_TILE - 1) / AP_TILE, ntj = (c1 - c0 + AP_TILE - 1) / AP_TILE;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  unsigned long long nz = 0;
  for (int64_t t = blockIdx.x; t < nti * ntj; t += gridDim.x) {
    const int64_t ti = r0 + (t / ntj) * AP_TILE, tj = c0 + (t % ntj) * AP_TILE;
    if (tj + AP_TILE <= ti + 1) continue;  // entirely on/below the diagonal
    uint32_t cnt[4][4];
#pragma unroll
    for (int u = 0; u < 4; u++)
#pragma unroll
      for (int v = 0; v < 4; v++) cnt[u][v] = 0;
    for (int64_t k0 = 0; k0 < m; k0 += AP_KS) {
      __syncthreads();
      for (int q = threadIdx.x; q < AP_KS * AP_TILE; q += blockDim.x) {
        const int r = q / AP_KS, kk = q % AP_KS;
        const int64_t gi = ti + r, gj = tj + r, k = k0 + kk;
        // out-of-range words compare equal; those pairs are discarded below
        sa[kk][r] = (gi < r1 && k < m) ? (uint32_t)__ldg(&sigs[gi * m + k]) : 0u;
        sb[kk][r] = (gj < c1 && k < m) ? (uint32_t)__ldg(&sigs[gj * m + k]) : 0u;
      }
      __syncthreads();
      const int kn = m - k0 < AP_KS ? (int)(m - k0) : AP_KS;
#pragma unroll 4
      for (int kk = 0; kk < kn; kk++) {
        const uint4 a4 = *reinterpret_cast<const uint4*>(&sa[kk][ty * 4]);
        const uint4 b4 = *reinterpret_cast<const uint4*>(&sb[kk][tx * 4]);
        const uint32_t av[4] = {a4.x, a4.y, a4.z, a4.w}, bv[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
        for (int u = 0; u < 4; u++)
#pragma unroll
          for (int v = 0; v < 4; v++) acc_eq32(cnt[u][v], av[u], bv[v]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int64_t i = ti + ty * 4 + u;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const int64_t j = tj + tx * 4 + v;
        if (i < r1 && j < c1 && j > i) {
          if (cnt[u][v] == 0) {
            nz++;
          } else {
            const unsigned long long pos = atomicAdd(ccursor, 1ULL);
            if ((int64_t)pos < ccap) cand[pos] = ((unsigned long long)i << 32) | (unsigned long long)j;
          }
        }
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) nz += __shfl_xor_sync(0xffffffffu, nz, o);
  if ((threadIdx.x & 31) == 0 && nz) atomicAdd(zeros, nz);
}

// stage 2: exact count of each candidate pair (warp per pair)
__global__ void __launch_bounds__(256) allpairs_cand_kernel(
    const uint64_t* __restrict__ sigs, int64_t m, const unsigned long long* __restrict__ cand,
    int64_t ccap, const unsigned long long* __restrict__ ccursor, int32_t thr,
    unsigned long long* __restrict__ hist, unsigned long long* __restrict__ pairs, int64_t cap,
    unsigned long long* __restrict__ cursor) {
  const unsigned long long nc = *ccursor;
  if (nc > (unsigned long long)ccap) return;           // overflow: the gated fallback runs
  const int lane = threadIdx.x & 31;
  const int64_t wg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = wg; p < (int64_t)nc; p += nw) {
    const unsigned long long ij = cand[p];
    const int64_t i = (int64_t)(ij >> 32), j = (int64_t)(ij & 0xffffffffULL);
    const uint64_t* a = sigs + i * m;
    const uint64_t* b = sigs + j * m;
    uint32_t c = 0;
    for (int64_t k = lane; k < m; k += 32) c += (__ldg(&a[k]) == __ldg(&b[k]));
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
      atomicAdd(&hist[c], 1ULL);
      if ((int32_t)c >= thr) {
        const unsigned long long pos = atomicAdd(cursor, 1ULL);
        if ((int64_t)pos < cap) {
          pairs[2 * pos] = ij;
          pairs[2 * pos + 1] = (unsigned long long)c;
        }
      }
    }
  }
}

// stage 3: the pairs stage 1 proved to have no equal component (thr >= 1
// only: they are never listed)
__global__ void allpairs_zeros_kernel(const unsigned long long* __restrict__ zeros,
                                      const unsigned long long* __restrict__ ccursor, int64_t ccap,
                                      unsigned long long* __restrict__ hist) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*ccursor > (unsigned long long)ccap) return;
  hist[0] += *zeros;
}

// Fused b-bit reduction + packing (K:851-861 + layout): word w of row s holds
// fields k = w * fpw + f (f < fpw = floor(64 / b)) at bits [f b, f b + b),
// field k = low b bits of mix64(sig_k + GOLDEN (k + 1)); unused fields are 0.
__global__ void bbit_pack_kernel(const uint64_t* __restrict__ sig, int64_t nsets, int64_t m,
                                 int b, int fpw, int64_t W, uint64_t* __restrict__ packed) {
  const uint64_t mask = (1ULL << (uint64_t)b) - 1ULL;
  const int64_t total = nsets * W;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = q / W, wi = q - s * W;
    uint64_t word = 0;
    for (int f = 0; f < fpw; f++) {
      const int64_t k = wi * fpw + f;
      if (k >= m) break;
      const uint64_t h = mix64(sig[s * m + k] + GOLDEN * (uint64_t)(k + 1)) & mask;
      word |= h << (f * b);
    }
    packed[q] = word;
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
