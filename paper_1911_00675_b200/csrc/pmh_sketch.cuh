// pmh_sketch.cuh -- ProbMinHash signature kernels (sm_100a).
//
// One CTA per set (grid-stride over a cost-ordered set list).  Shared memory
// holds the set's slot table (lexicographic argmin of (h, element index) per
// component, 128-bit CAS) and the stop limit h_max.  Because a signature is
//   sig_k = argmin_d (h_k(d), index(d))
// over per-element point sequences that are fixed functions of (id, w, m,
// variant), and early stopping only skips points above the final stop limit
// H, elements may be processed in ANY order with ANY threshold >= H
// (SURVEY.md §0 facts 4 and 6).  Each CTA therefore:
//   1. computes W = sum(w) and a threshold guess t = m (ln m + 3) / W
//      (a point-process estimate of H; correctness never depends on it);
//   2. streams elements, one per thread, through the variant's exact point
//      recurrence (Appendix A), skipping every point whose value -- or a
//      provable lower bound of it, which avoids log1p -- exceeds
//      thr = min(t, h_max);
//   3. hands elements whose lazy Fisher-Yates state outgrows the lane's map
//      (a per-lane hash table in shared memory, pmh_warp.cuh: HashFY; a small
//      register map in the warp-per-set kernel) to warp-cooperative processing
//      with a dense shared map;
//   4. verifies max_k h_k <= t (else retries with a larger t; re-offering a
//      point is idempotent) and writes sig_k = ids[argmin].
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

// per-m constant tables computed on the host with glibc (K:186-191,
// K:418-420, K:458-459, K:568-579)
struct Tables {
  TruncExpConsts c3;          // PMH3: lam = log1p(1/(m-1))
  const TruncExpConsts* c4;   // PMH4: [m] per interval, index 1..m-1
  const double* gam;          // PMH4: gamma_i, [m]
  const double* dgam;         // PMH4: fl(gamma_i - gamma_{i-1}), [m]
  double delta;               // PMH4: 1/lam_1
  const double* beta;         // PMH2: [m+1], beta_i = m/(m-i+1.0)
};

// 32-bit fields where the ranges allow (m <= 65535, coupon cap < 2^31,
// per-thread counters, in-set element indices < 2^31): the state lives in
// registers across the element loops, and 64-bit fields pushed the 80-register
// kernels into rematerialising and spilling
struct SetCtx {
  Slot* slots;                       // [m] shared
  unsigned long long* hmax_bits;     // shared, current upper bound of H
  unsigned int* filled;              // shared, #non-empty slots
  double tguess;                     // current threshold guess
  int32_t m;
  uint32_t kbits;
  int32_t cap;                       // coupon cap K:279-281
  // counters (per thread)
  uint32_t points;
  double tprev;                      // previous attempt's threshold (-1: none);
                                     // a retry counts only points above it
  uint32_t updates;
  uint32_t multi;                    // elements that produced > 1 point
  int since_refresh;                 // batches since the last h_max refresh
  bool trig;                         // this lane lowered the maximum slot / filled the last
                                     // one: the warp refreshes h_max after the batch
  int32_t eoff;                      // in-set index of element 0 (a split set's part)
  int32_t heavy_pts;                 // expected points above which an element runs warp-cooperatively
};

__device__ __forceinline__ double ctx_thr(const SetCtx& c) {
  const double h = __longlong_as_double((long long)*(volatile unsigned long long*)c.hmax_bits);
  return h < c.tguess ? h : c.tguess;
}

__device__ __forceinline__ void ctx_offer(SetCtx& c, int64_t k0, double x,
                                          int64_t e) {
  PMH_ASSERT(k0 >= 0 && k0 < c.m);
  unsigned long long prev = slot_offer(&c.slots[k0], x, (unsigned long long)(e + c.eoff));
  if (prev == ~0ULL) return;
  c.updates++;
  // h_max stays an upper bound of max_k h_k (a valid, if stale, threshold);
  // the converged warp recomputes it cooperatively after the batch
  // (run_batch) instead of one lane scanning all m slots here
  if (prev == EMPTY_H) {
    unsigned f = atomicAdd(c.filled, 1u) + 1u;
    if (f == (unsigned)c.m) c.trig = true;
  } else if (prev >= *(volatile unsigned long long*)c.hmax_bits) {
    c.trig = true;
  }
}

// warp-cooperative refresh of h_max
__device__ __forceinline__ void hmax_refresh_warp(SetCtx& c, int lane) {
  // warp-uniform decision (lanes may arrive unconverged after divergent work)
  const unsigned f = __shfl_sync(0xffffffffu, *(volatile unsigned*)c.filled, 0);
  if (f < (unsigned)c.m) return;
  unsigned long long mx = 0;
  for (int64_t k = lane; k < c.m; k += 32) {
    unsigned long long h = *(volatile unsigned long long*)&c.slots[k].h;
    mx = h > mx ? h : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = v > mx ? v : mx;
  }
  if (lane == 0) atomicMin(c.hmax_bits, mx);
}

// ---------------------------------------------------------------------------
// Lazy Fisher-Yates (K:222-235).  Positions/values are 1-based; an absent
// entry means perm[p] == p.
// ---------------------------------------------------------------------------
#ifndef PMH_SPARSE_FY_CAP
#define PMH_SPARSE_FY_CAP 16   // measured: 8 / 12 / 16 / 24 tried on config 2
#endif
constexpr int SPARSE_FY_CAP = PMH_SPARSE_FY_CAP;

struct SparseFY {
  int32_t pos[SPARSE_FY_CAP];
  int32_t val[SPARSE_FY_CAP];
  int cnt;
  __device__ __forceinline__ void reset() { cnt = 0; }
  // one lazy Fisher-Yates step (K:222-235) in ONE scan: returns perm[j] and
  // sets perm[j] = perm[i] (both read before the write, as in get/set);
  // 0 on overflow
  __device__ __forceinline__ int32_t swap_step(int32_t i, int32_t j) {
    int32_t vi = i, vj = j;
    int qj = -1;
    for (int q = 0; q < cnt; q++) {
      const int32_t p = pos[q];
      if (p == j) { vj = val[q]; qj = q; }
      if (p == i) vi = val[q];
    }
    if (qj >= 0) {
      val[qj] = vi;
    } else {
      if (cnt == SPARSE_FY_CAP) return 0;
      pos[cnt] = j; val[cnt] = vi; cnt++;
    }
    return vj;
  }
};

// Returns label k (1-based), 0 on FY overflow, -1 on randomness failure.
template <class FY>
__device__ __forceinline__ int64_t perm_next(Stream& st, FY& fy, int64_t i,
                                             int64_t m) {
  int64_t r = uniform_int(st, m - i + 1);
  if (r < 0) return -1;
  return fy.swap_step((int32_t)i, (int32_t)(i + r));
}

// result codes of the element processors
constexpr int EL_DONE = 0;
constexpr int EL_NEED_WARP = 1;
constexpr int EL_FAIL = -1;

// ---------------------------------------------------------------------------
// Element processors: the reference recurrences (Appendix A) with the stop
// test `x >= nodes[root]` replaced by `x > thr` (thr >= H; ties processed).
// ---------------------------------------------------------------------------

// ProbMinHash1 / 1a / unweighted 1, 1a (K:315-333, K:357-400)
__device__ __forceinline__ int el_pmh1(SetCtx& c, int64_t e, uint64_t id,
                                       double winv) {
  Stream st; st.seed(id);
  uint64_t b = st.next53();
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  if (exp1_scaled_lower_bound(winv, b) > ctx_thr(c)) return EL_DONE;
  double x = winv * exp1_from_bits(b);
  int64_t cnt = 1;
  while (x <= ctx_thr(c)) {
    int64_t r = uniform_int_masked(st, (uint64_t)c.m, c.kbits);
    if (r < 0) return EL_FAIL;
    ctx_offer(c, r, x, e);
    b = st.next53();
    c.points += (x > c.tprev);
    if (cnt == 1) c.multi++;
    if (++cnt > c.cap) return EL_FAIL;
    if (x + exp1_scaled_lower_bound(winv, b) > ctx_thr(c)) return EL_DONE;
    x = x + winv * exp1_from_bits(b);
  }
  return EL_DONE;
}

// ProbMinHash2 / unweighted 2 (K:423-441)
template <class FY>
__device__ __forceinline__ int el_pmh2(SetCtx& c, const Tables& T, FY& fy,
                                       int64_t e, uint64_t id, double winv) {
  Stream st; st.seed(id);
  uint64_t b = st.next53();
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  if (exp1_scaled_lower_bound(winv, b) > ctx_thr(c)) return EL_DONE;
  double x = winv * exp1_from_bits(b);
  int64_t i = 1;
  while (x <= ctx_thr(c)) {
    int64_t k = perm_next(st, fy, i, c.m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, x, e);
    i++;
    if (i > c.m) break;
    const double a = winv * __ldg(&T.beta[i]);
    b = st.next53();
    c.points += (x > c.tprev);
    if (i == 2) c.multi++;
    if (x + exp1_scaled_lower_bound(a, b) > ctx_thr(c)) return EL_DONE;
    x = x + a * exp1_from_bits(b);
  }
  return EL_DONE;
}

// ProbMinHash3 / 3a (K:462-481, K:506-547)
__device__ __forceinline__ int el_pmh3(SetCtx& c, const Tables& T, int64_t e,
                                       uint64_t id, double winv) {
  Stream st; st.seed(id);
  bool fail = false;
  double x = winv * trunc_exp(st, T.c3, &fail);
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  int64_t i = 1;
  while (x <= ctx_thr(c)) {
    int64_t r = uniform_int_masked(st, (uint64_t)c.m, c.kbits);
    if (r < 0 || fail) return EL_FAIL;
    ctx_offer(c, r, x, e);
    if (++i > c.cap) return EL_FAIL;
    x = winv * ((double)i - 1.0);
    if (x > ctx_thr(c)) break;
    x = x + winv * trunc_exp(st, T.c3, &fail);
    c.points += (winv * ((double)i - 1.0) > c.tprev);
    if (i == 2) c.multi++;
  }
  return fail ? EL_FAIL : EL_DONE;
}

// ProbMinHash4 (K:582-610)
template <class FY>
__device__ __forceinline__ int el_pmh4(SetCtx& c, const Tables& T, FY& fy,
                                       int64_t e, uint64_t id, double winv) {
  Stream st; st.seed(id);
  bool fail = false;
  double x = winv * trunc_exp(st, T.c4[1], &fail);
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  int64_t i = 1;
  const int64_t m = c.m;
  while (x <= ctx_thr(c)) {
    if (fail) return EL_FAIL;
    int64_t k = perm_next(st, fy, i, m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, x, e);
    i++;
    if (winv * __ldg(&T.gam[i - 1]) > ctx_thr(c)) break;
    if (i == 2) c.multi++;
    if (i < m) {
      const double t = trunc_exp(st, T.c4[i], &fail);
      x = winv * (__ldg(&T.gam[i - 1]) + __ldg(&T.dgam[i]) * t);
      c.points += (winv * __ldg(&T.gam[i - 1]) > c.tprev);
    } else {
      x = winv * (__ldg(&T.gam[m - 1]) + T.delta * exp1_from_bits(st.next53()));
      c.points += (winv * __ldg(&T.gam[i - 1]) > c.tprev);
      if (x <= ctx_thr(c)) {
        k = perm_next(st, fy, m, m);
        if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
        ctx_offer(c, k - 1, x, e);
      }
      break;
    }
  }
  return fail ? EL_FAIL : EL_DONE;
}

// unweighted ProbMinHash3 / 3a (K:631-649, K:674-710)
__device__ __forceinline__ int el_uw3(SetCtx& c, int64_t e, uint64_t id) {
  Stream st; st.seed(id);
  double x = st.uniform01();
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  int64_t i = 1;
  while (x <= ctx_thr(c)) {
    int64_t r = uniform_int_masked(st, (uint64_t)c.m, c.kbits);
    if (r < 0) return EL_FAIL;
    ctx_offer(c, r, x, e);
    if (++i > c.cap) return EL_FAIL;
    x = (double)i - 1.0;
    if (x > ctx_thr(c)) break;
    x = x + st.uniform01();
    c.points += (((double)i - 1.0) > c.tprev);
    if (i == 2) c.multi++;
  }
  return EL_DONE;
}

// unweighted ProbMinHash4 (K:734-759)
template <class FY>
__device__ __forceinline__ int el_uw4(SetCtx& c, FY& fy, int64_t e, uint64_t id) {
  Stream st; st.seed(id);
  double x = st.uniform01();
  c.points += (0.0 > c.tprev);  // first point: LB = 0
  int64_t i = 1;
  const int64_t m = c.m;
  while (x <= ctx_thr(c)) {
    int64_t k = perm_next(st, fy, i, m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, x, e);
    i++;
    if ((double)i - 1.0 > ctx_thr(c)) break;
    if (i == 2) c.multi++;
    if (i < m) {
      x = ((double)i - 1.0) + st.uniform01();
      c.points += (((double)i - 1.0) > c.tprev);
    } else {
      x = ((double)m - 1.0) + st.uniform01();
      c.points += (((double)i - 1.0) > c.tprev);
      if (x <= ctx_thr(c)) {
        k = perm_next(st, fy, m, m);
        if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
        ctx_offer(c, k - 1, x, e);
      }
      break;
    }
  }
  return EL_DONE;
}

// kernel-family selector
enum Family : int { FAM_PMH1 = 1, FAM_PMH2 = 2, FAM_PMH3 = 3, FAM_PMH4 = 4,
                    FAM_UW3 = 5, FAM_UW4 = 6 };

__host__ __device__ constexpr bool family_uses_fy(int f) {
  return f == FAM_PMH2 || f == FAM_PMH4 || f == FAM_UW4;
}
__host__ __device__ constexpr bool family_weighted(int f) {
  return f == FAM_PMH1 || f == FAM_PMH2 || f == FAM_PMH3 || f == FAM_PMH4;
}

template <int F, class FY>
__device__ __forceinline__ int run_element(SetCtx& c, const Tables& T, FY& fy,
                                           int64_t e, uint64_t id, double winv) {
  if constexpr (F == FAM_PMH1) return el_pmh1(c, e, id, winv);
  else if constexpr (F == FAM_PMH2) return el_pmh2(c, T, fy, e, id, winv);
  else if constexpr (F == FAM_PMH3) return el_pmh3(c, T, e, id, winv);
  else if constexpr (F == FAM_PMH4) return el_pmh4(c, T, fy, e, id, winv);
  else if constexpr (F == FAM_UW3) return el_uw3(c, e, id);
  else return el_uw4(c, fy, e, id);
}

struct SketchArgs {
  const uint64_t* ids;
  const double* w;          // nullptr => unit weights
  const int64_t* offsets;
  const int32_t* order;     // set processing order (nullptr => identity)
  int64_t nsets;
  int64_t m;
  uint64_t* sig;            // [nsets, m]
  int64_t* stats;           // [nsets, 3] or nullptr
  unsigned long long* err_flags;  // device, OR of ERRF_*
  long long* err_set;       // device, min failing set index
  Tables T;
  double tconst;            // threshold-guess constant (ln m + tconst)
  const unsigned* counts;   // device: [0] = number of large sets (order prefix)
  const long long* split_info;  // order[0, split_info[0]) are split (pmh_split.cuh)
  const double* setw;       // device [nsets] total weights known in advance, or nullptr
};

// Threshold-guess constant c of t = m (ln m + c) / W for a set (or range) of
// n elements.  A guess below the final limit H costs the set a full retry
// (4t): for a handful of elements (a lone element's coupon collector exceeds
// m (ln m + c) points with probability ~e^-c) that doubles the set's
// latency, and a small batch (one rank's shard) waits on its slowest sets.
// With so few elements the slot table fills from the elements' own long
// point sequences and the stop limit falls to h_max at once, so a larger c
// costs them almost no points.
#ifndef PMH_FEW_N
#define PMH_FEW_N 16
#endif
#ifndef PMH_FEW_BOOST
#define PMH_FEW_BOOST 3.0
#endif
__device__ __forceinline__ double guess_const(double tconst, int64_t n) {
  return n <= PMH_FEW_N ? tconst + PMH_FEW_BOOST : tconst;
}

// Per-set total weights W_s (one CTA per set, grid-stride): computed once per
// batch and shared by every variant of a multi-variant call, or supplied by
// the caller for the non-streaming variants.
__global__ void __launch_bounds__(256) set_weights_kernel(const double* __restrict__ w,
                                                          const int64_t* __restrict__ offsets,
                                                          int64_t nsets, double* __restrict__ out) {
  __shared__ double red[8];
  for (int64_t s = blockIdx.x; s < nsets; s += gridDim.x) {
    const int64_t e0 = offsets[s], e1 = offsets[s + 1];
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    int64_t e = e0 + threadIdx.x;
    for (; e + 768 < e1; e += 1024) {
      p0 += __ldg(&w[e]);
      p1 += __ldg(&w[e + 256]);
      p2 += __ldg(&w[e + 512]);
      p3 += __ldg(&w[e + 768]);
    }
    for (; e < e1; e += 256) p0 += __ldg(&w[e]);
    double v = (p0 + p1) + (p2 + p3);
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < 8; i++) t += red[i];
      out[s] = t;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    v = lane < (int)(blockDim.x >> 5) ? red[lane] : 0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

}  // namespace pmh
