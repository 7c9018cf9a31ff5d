// pmh_flat.cuh -- "flat" point-parallel kernel for ProbMinHash3/3a and the
// unweighted 3/3a (labels with replacement, power-of-two m).
//
// In these variants a point's value and label sit at a STATIC bit offset of
// its element's stream -- point i uses bits [(i-1) P, i P), P = 53 + log2 m
// (K:462-481: TruncExp's fast path draws one 53-bit uniform, the label kb
// bits that never reject for power-of-two m) -- and its lower bound
// winv (i - 1) (K:477) is known before anything is drawn.  So, given the
// threshold t, element e has exactly J_e = floor(t w_e) + 1 candidate points
// and every (element, point) pair can be computed independently:
//   * a CTA takes a set's elements 256 at a time (one per thread, the next
//     chunk's id and weight prefetched), computes J_e and a block-wide prefix;
//   * the chunk's sum_e J_e points are then processed 256 per round, one per
//     thread -- a binary search in the prefix finds the thread's (element,
//     point) -- with one or two splitmix64 words per point, the TruncExp fast
//     path, and the slot offer;
//   * every lane is busy until the chunk's last round, for any set size: a
//     single-element set's ~m ln m points spread over all 256 threads instead
//     of one warp's sequential batches.
// Each round re-evaluates every element's remaining candidates under the
// CURRENT stop limit (which falls as the slots fill), so the total work tracks
// the reference's, not the initial guess's.  TruncExp's slow path (probability
// ~1/(2m) per point) consumes a variable number of bits, so the element's
// later offsets shift: the lowest slow point of an element in a round cuts it
// (its later points of that round are dropped), its owner thread evaluates
// the slow point sequentially from its exact stream position, and the
// element's remaining points restart with static stride P after it.  Threshold guess, verification and retry as in sketch_range
// (retries multiply the guess by 4, always finite: J_e is bounded by the
// coupon cap, K:279-281, which a weighted element can never legitimately
// reach below the final stop limit).
#pragma once
#include "pmh_sketch.cuh"

namespace pmh {

constexpr int FLAT_THREADS = 256;
#ifndef PMH_FLAT_RP
#define PMH_FLAT_RP 4
#endif
constexpr int FLAT_RP = PMH_FLAT_RP;   // points per thread per round
#ifndef PMH_FLAT_NMAX
#define PMH_FLAT_NMAX 1024
#endif

__host__ __device__ inline bool flat_eligible(int family, int64_t m) {
  // power-of-two m (labels never reject) with kb <= 12: a point spans <= 2 words
  return (family == FAM_PMH3 || family == FAM_UW3) && m >= 2 && (m & (m - 1)) == 0 && m <= 4096;
}

struct FlatShared {
  unsigned long long hmax;
  unsigned int filled;
  int retry;
  int32_t wtot[FLAT_THREADS / 32];  // block scan: warp totals
  int32_t pre[FLAT_THREADS + 1];    // exclusive prefix of the round's remaining point counts
  uint64_t id[FLAT_THREADS];        // the chunk's elements (one per thread)
  double winv[FLAT_THREADS];
  int32_t cur[FLAT_THREADS];        // points of the element done
  int32_t bj[FLAT_THREADS];         // point index at which the static offsets restart ...
  uint64_t boff[FLAT_THREADS];      // ... and its bit offset (after a slow point)
  int32_t cut[FLAT_THREADS];        // lowest slow point of the element this round (INT32_MAX: none)
  double red[32];
  long long redl[32];
};

// One slow point: the element's point i at bit offset `bit`, whose TruncExp
// draw fails the fast path (K:133-151), evaluated sequentially from its exact
// stream position; offered if below the threshold; *next_off = the position
// after its label, where the element's later points restart (static stride
// P again).  Returns true on a rejection-cap failure.
template <int F>
__device__ __noinline__ bool flat_slow_point(SetCtx& c, const Tables& T, uint64_t id, double winv,
                                             int64_t e, int64_t i, uint64_t bit,
                                             uint64_t* next_off, double thr) {
  Stream st;
  st.seek(id, bit);
  bool fail = false;
  double x;
  if constexpr (F == FAM_PMH3) {
    const double t = trunc_exp(st, T.c3, &fail);
    x = i == 1 ? winv * t : winv * ((double)i - 1.0) + winv * t;
  } else {
    const double U = st.uniform01();
    x = i == 1 ? U : ((double)i - 1.0) + U;
  }
  const int64_t r = uniform_int_masked(st, (uint64_t)c.m, c.kbits);
  *next_off = st.pos(id);
  if (r < 0 || fail) return true;
  if (x <= thr) ctx_offer(c, r, x, e);
  return false;
}

// The sets of the LPT order's small partition (n <= PMH_FLAT_NMAX:
// order[counts[0], nsets)); the large ones stream through the CTA kernel's
// prefilter, which the per-round scans here cannot match when almost every
// element has a single candidate point.
template <int F>
#ifndef PMH_FLAT_MINB
#define PMH_FLAT_MINB 4   // 64 registers: configs[1] ProbMinHash3 2.50 -> 2.45 ms (2: 2.75; 5-6: see DESIGN)
#endif
__global__ void __launch_bounds__(FLAT_THREADS, PMH_FLAT_MINB) sketch_flat_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ FlatShared sh;
  Slot* slots = reinterpret_cast<Slot*>(smem);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t m = a.m;
  const uint32_t kb = bits_for(m);
  const uint32_t P = 53u + kb;
  const uint64_t kmask = (1ULL << kb) - 1ULL;
  const bool weighted = family_weighted(F) && a.w;
  const double c1 = F == FAM_PMH3 ? a.T.c3.c1 : 0.0;
  const int64_t first = a.counts ? (int64_t)a.counts[0] : 0;
  for (int64_t bs = first + blockIdx.x; bs < a.nsets; bs += gridDim.x) {
    const int64_t s = a.order ? (int64_t)a.order[bs] : bs;
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (tid == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    const uint64_t* ids = a.ids + off;
    const double* w = weighted ? a.w + off : nullptr;
    for (int64_t k = tid; k < m; k += FLAT_THREADS) { slots[k].h = EMPTY_H; slots[k].idx = EMPTY_IDX; }
    double W;
    if (weighted && a.setw && a.setw[s] > 0.0) {
      W = a.setw[s];
    } else if (weighted) {
      double p = 0.0;
      for (int64_t e = tid; e < n; e += FLAT_THREADS) p += __ldg(&w[e]);
      W = block_sum(p, sh.red);
    } else {
      W = (double)n;
    }
    if (tid == 0) { sh.hmax = EMPTY_H; sh.filled = 0; }
    SetCtx c;
    c.slots = slots;
    c.hmax_bits = &sh.hmax;
    c.filled = &sh.filled;
    c.m = (int32_t)m;
    c.kbits = kb;
    c.cap = (int32_t)coupon_cap(m);
    c.points = 0; c.updates = 0; c.multi = 0; c.tprev = -1.0; c.since_refresh = 0;
    c.trig = false;
    c.eoff = 0;
    double tg = (double)m * (log((double)m) + guess_const(a.tconst, n)) / W;
    if (!(tg > 0.0) || !(tg < 1e300)) tg = 1e300;
    bool failed = false;
    __syncthreads();
    for (int attempt = 0;; attempt++) {
      c.tguess = tg;
      // the first chunk's element, prefetched one chunk ahead
      uint64_t id_n = tid < n ? __ldg(&ids[tid]) : 0ULL;
      double w_n = (weighted && tid < n) ? __ldg(&w[tid]) : 1.0;
      for (int64_t base = 0; base < n; base += FLAT_THREADS) {
        const int64_t e = base + tid;
        const bool valid = e < n;
        const uint64_t id = id_n;
        const double wv = w_n;
        if (base + FLAT_THREADS + tid < n) {
          id_n = __ldg(&ids[base + FLAT_THREADS + tid]);
          if (weighted) w_n = __ldg(&w[base + FLAT_THREADS + tid]);
        }
        sh.id[tid] = id;
        sh.winv[tid] = (F == FAM_PMH3 && valid) ? 1.0 / wv : 1.0;
        sh.cur[tid] = 0;
        sh.bj[tid] = 1;
        sh.boff[tid] = 0;
        sh.cut[tid] = INT32_MAX;
        bool multi_counted = false;
        // rounds: every element's remaining candidate points under the CURRENT
        // stop limit, the first FLAT_THREADS of their concatenation processed
        for (;;) {
          const double thr = ctx_thr(c);
          // candidate points: lower bounds winv (i-1) <= thr  <=>  i - 1 <= thr w
          const double lim = F == FAM_PMH3 ? thr * wv : thr;
          int32_t J = 0;
          if (valid) {
            if (lim >= (double)c.cap) { J = c.cap; failed = true; }
            else J = (int32_t)floor(lim) + 1;
          }
          const int32_t cur = sh.cur[tid];
          const int32_t rem = J > cur ? J - cur : 0;
          if (!multi_counted && J >= 2) { c.multi++; multi_counted = true; }
          // block exclusive scan of rem
          int32_t v = rem;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, v, o);
            if (lane >= o) v += t;
          }
          if (lane == 31) sh.wtot[wid] = v;
          __syncthreads();
          int32_t woff = 0, total = 0;
#pragma unroll
          for (int k = 0; k < FLAT_THREADS / 32; k++) {
            const int32_t tk = sh.wtot[k];
            woff += k < wid ? tk : 0;
            total += tk;
          }
          const int32_t mypre = woff + v - rem;
          sh.pre[tid] = mypre;
          if (tid == 0) sh.pre[FLAT_THREADS] = total;
          __syncthreads();
          if (total == 0) break;
          // FLAT_RP points per thread per round (independent chains: ILP, and
          // the round's scan and barriers amortised over more points)
          int el[FLAT_RP];
          int32_t jj[FLAT_RP];
          bool pslow[FLAT_RP];
          double x[FLAT_RP];
          int32_t lab[FLAT_RP];
#pragma unroll
          for (int q = 0; q < FLAT_RP; q++) {
            const int32_t g = tid + q * FLAT_THREADS;
            el[q] = 0; jj[q] = 0; pslow[q] = false; x[q] = 0.0; lab[q] = 0;
            if (g < total) {
              // the element of point g: the largest e with pre[e] <= g
              int lo = 0, hi = FLAT_THREADS;   // pre[lo] <= g < pre[hi]
#pragma unroll
              for (int it = 0; it < 8; it++) {
                const int mid = (lo + hi) >> 1;
                if (sh.pre[mid] <= g) lo = mid; else hi = mid;
              }
              el[q] = lo;
              jj[q] = sh.cur[lo] + (g - sh.pre[lo]) + 1;   // point index
              const uint64_t eid = sh.id[lo];
              const uint64_t bit = sh.boff[lo] + (uint64_t)(jj[q] - sh.bj[lo]) * P;
              const uint64_t wi = bit >> 6;
              const uint32_t shf = (uint32_t)(bit & 63);
              const uint64_t w0 = stream_word(eid, wi + 1);
              const uint64_t w1 = (shf + P > 64) ? stream_word(eid, wi + 2) : 0ULL;
              const uint64_t vv = shf ? (w0 >> shf) | (w1 << (64 - shf)) : w0;
              const uint64_t u = vv & ((1ULL << 53) - 1ULL);
              // the label: bits 53 .. 53 + kb of the point; for kb = 12 its top
              // bit is bit 64 of the point, i.e. bit shf of the second word
              lab[q] = (int32_t)(((vv >> 53) | (P > 64 ? (w1 >> shf) << 11 : 0ULL)) & kmask);
              const double U = (double)u * INV53;
              const int32_t j1 = jj[q];
              if constexpr (F == FAM_PMH3) {
                const double winv = sh.winv[lo];
                const double t = c1 * U;            // TruncExp fast path (K:130-132)
                pslow[q] = !(t < 1.0);
                x[q] = j1 == 1 ? winv * t : winv * ((double)j1 - 1.0) + winv * t;
                c.points += (winv * ((double)j1 - 1.0) > c.tprev) || (j1 == 1 && 0.0 > c.tprev);
              } else {
                x[q] = j1 == 1 ? U : ((double)j1 - 1.0) + U;
                c.points += (((double)j1 - 1.0) > c.tprev) || (j1 == 1 && 0.0 > c.tprev);
              }
              if (pslow[q]) atomicMin(&sh.cut[lo], j1);
            }
          }
          __syncthreads();
          {
            const double thr2 = ctx_thr(c);
#pragma unroll
            for (int q = 0; q < FLAT_RP; q++)
              if (jj[q] > 0 && !pslow[q] && jj[q] < sh.cut[el[q]] && x[q] <= thr2)
                ctx_offer(c, lab[q], x[q], (int64_t)(base + el[q]));
          }
          __syncthreads();   // every lane has read cut[] before the owners update it
          // this element's points of the round: the part of [mypre, mypre + rem)
          // below FLAT_RP * FLAT_THREADS, up to (excluding) a slow point
          int32_t done = FLAT_RP * FLAT_THREADS - mypre;
          done = done < 0 ? 0 : (done > rem ? rem : done);
          const int32_t ct = sh.cut[tid];
          if (ct != INT32_MAX) {
            // the slow point itself, sequentially from its exact stream position;
            // the element's later points restart from the position after it
            if (flat_slow_point<F>(c, a.T, sh.id[tid], sh.winv[tid], base + tid, ct,
                                   sh.boff[tid] + (uint64_t)(ct - sh.bj[tid]) * P, &sh.boff[tid],
                                   ctx_thr(c)))
              failed = true;
            sh.bj[tid] = ct + 1;
            sh.cur[tid] = ct;
            sh.cut[tid] = INT32_MAX;
          } else {
            sh.cur[tid] = cur + done;
          }
          if (__syncthreads_or(c.trig)) {
            c.trig = false;
            if (wid == 0) hmax_refresh_warp(c, lane);
          }
          __syncthreads();
        }
        __syncthreads();
      }
      // verification: every slot non-empty and <= tg
      unsigned long long mx = 0;
      for (int64_t k = tid; k < m; k += FLAT_THREADS) {
        const unsigned long long h = slots[k].h;
        mx = h > mx ? h : mx;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v2 = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v2 > mx ? v2 : mx;
      }
      if (tid == 0) sh.retry = 0;
      __syncthreads();
      if (lane == 0 && __longlong_as_double((long long)mx) > tg) atomicOr(&sh.retry, 1);
      const int any_fail = __syncthreads_or(failed ? 1 : 0);
      if (any_fail) { failed = true; break; }
      if (!sh.retry) break;
      c.tprev = tg;
      tg = tg * 4.0;
      __syncthreads();
    }
    if (failed && tid == 0) {
      atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
      atomicMin(a.err_set, (long long)s);
    }
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = tid; k < m; k += FLAT_THREADS) {
      const unsigned long long ix = slots[k].idx;
      sig[k] = ix < (unsigned long long)n ? ids[ix] : 0ULL;
    }
    if (a.stats) {
      const long long pts = block_sum_ll(c.points, sh.redl);
      const long long mul = block_sum_ll(c.multi, sh.redl);
      const long long upd = block_sum_ll(c.updates, sh.redl);
      if (tid == 0) {
        a.stats[s * 3 + 0] = pts;
        a.stats[s * 3 + 1] = mul;
        a.stats[s * 3 + 2] = upd;
      }
    }
    __syncthreads();
  }
}

}  // namespace pmh
