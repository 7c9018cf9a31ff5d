// pmh_lane.cuh -- one ProbMinHash element as a per-lane state machine.
//
// lane_init / lane_step restate the reference recurrences (Appendix A;
// K:318-333, K:428-441, K:462-481, K:582-610, K:631-649, K:734-759) one
// point per call -- value (log1p or TruncExp), stop test, label, slot offer,
// and the NEXT point's lower-bound test fused into the same step -- exactly as
// the lane-per-element processors of pmh_sketch.cuh do, with the same point /
// update / multi-point counters (GPU-schedule statistics).  Used by the lane-
// refill loop of pmh_wps.cuh, where a lane whose element finishes takes the
// next element before the next step.  The lazy Fisher-Yates state
// (K:222-235) is a template: a few entries in registers (RegFY) or a per-lane
// dense map in shared memory (pmh_wps.cuh).  Table reads are generic loads:
// the caller may point Tables at shared-memory copies.
#pragma once
#include "pmh_warp.cuh"

namespace pmh {

#ifndef PMH_RFY_CAP
#define PMH_RFY_CAP 8   // Fisher-Yates swaps a refill lane holds in registers
#endif

// Per-lane lazy Fisher-Yates map (K:222-235) in registers: entry = pos << 16
// | val (1-based, m <= 65535); fully unrolled, never indexed dynamically.
struct RegFY {
  uint32_t ent[PMH_RFY_CAP];
  int cnt;
  __device__ __forceinline__ void reset() { cnt = 0; }
  // perm[j] (returned) and perm[j] = perm[i], both read first; 0 on overflow
  __device__ __forceinline__ int32_t swap_step(int32_t i, int32_t j) {
    int32_t vi = i, vj = j;
    int qj = -1;
#pragma unroll
    for (int q = 0; q < PMH_RFY_CAP; q++) {
      if (q < cnt) {
        const int32_t p = (int32_t)(ent[q] >> 16);
        const int32_t v = (int32_t)(ent[q] & 0xffffu);
        if (p == j) { vj = v; qj = q; }
        if (p == i) vi = v;
      }
    }
    if (qj < 0) {
      if (cnt == PMH_RFY_CAP) return 0;
      qj = cnt++;
    }
    const uint32_t ne = ((uint32_t)j << 16) | (uint32_t)vi;
#pragma unroll
    for (int q = 0; q < PMH_RFY_CAP; q++)
      if (q == qj) ent[q] = ne;
    return vj;
  }
};

constexpr int EL_CONT = 2;   // the element has more points (refill loop)

// the state of one element in a refill lane
template <class FY = RegFY>
struct LaneElT {
  Stream st;
  double winv;
  double x;       // PMH1/2: running sum so far; PMH3/4/uw: the pending point's value
  double a;       // PMH2: the pending point's scale winv * beta_i
  uint64_t b;     // PMH1/2: the pending point's 53 value bits
  int32_t e;      // element index within the range
  int32_t i;      // point index (1-based)
  bool fail;      // TruncExp rejection cap hit (K:150)
  FY fy;
};
using LaneEl = LaneElT<RegFY>;

// Start element e.  Returns false if it is finished at once.
template <int F, class FY>
__device__ __forceinline__ bool lane_init(SetCtx& c, const Tables& T, LaneElT<FY>& s, int32_t e,
                                          uint64_t id, double winv, double thr) {
  s.e = e;
  s.winv = winv;
  s.i = 1;
  s.fail = false;
  s.st.seed(id);
  c.points += (0.0 > c.tprev);   // the first point
  if constexpr (F == FAM_PMH1 || F == FAM_PMH2) {
    s.b = s.st.next53();
    s.x = 0.0;                    // fl(0 + v) == v: the first point is winv E exactly
    s.a = winv;
    if constexpr (F == FAM_PMH2) s.fy.reset();
    return !(exp1_scaled_lower_bound(winv, s.b) > thr);
  } else if constexpr (F == FAM_PMH3) {
    s.x = winv * trunc_exp(s.st, T.c3, &s.fail);
    return true;
  } else if constexpr (F == FAM_PMH4) {
    s.fy.reset();
    s.x = winv * trunc_exp(s.st, T.c4[1], &s.fail);
    return true;
  } else {   // uw3 / uw4
    if constexpr (F == FAM_UW4) s.fy.reset();
    s.x = s.st.uniform01();
    return true;
  }
}

template <class FY>
__device__ __forceinline__ int32_t perm_next_reg(Stream& st, FY& fy, int32_t i, int64_t m) {
  const int64_t r = uniform_int(st, m - i + 1);
  if (r < 0) return -1;
  return fy.swap_step(i, (int32_t)(i + r));
}

// One point of the lane's element: EL_CONT, EL_DONE, EL_FAIL or EL_NEED_WARP.
template <int F, class FY>
__device__ __forceinline__ int lane_step(SetCtx& c, const Tables& T, LaneElT<FY>& s, double thr) {
  const int64_t m = c.m;
  if constexpr (F == FAM_PMH1) {             // K:318-333
    const double xv = s.x + s.winv * exp1_from_bits(s.b);
    if (!(xv <= thr)) return EL_DONE;
    const int64_t r = uniform_int_masked(s.st, (uint64_t)m, c.kbits);
    if (r < 0) return EL_FAIL;
    ctx_offer(c, r, xv, s.e);
    s.b = s.st.next53();
    c.points += (xv > c.tprev);
    if (s.i == 1) c.multi++;
    if (++s.i > c.cap) return EL_FAIL;
    if (xv + exp1_scaled_lower_bound(s.winv, s.b) > thr) return EL_DONE;
    s.x = xv;
    return EL_CONT;
  } else if constexpr (F == FAM_PMH2) {      // K:428-441
    const double xv = s.x + s.a * exp1_from_bits(s.b);
    if (!(xv <= thr)) return EL_DONE;
    const int32_t k = perm_next_reg(s.st, s.fy, s.i, m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, xv, s.e);
    s.i++;
    if (s.i > m) return EL_DONE;
    s.a = s.winv * T.beta[s.i];
    s.b = s.st.next53();
    c.points += (xv > c.tprev);
    if (s.i == 2) c.multi++;
    if (xv + exp1_scaled_lower_bound(s.a, s.b) > thr) return EL_DONE;
    s.x = xv;
    return EL_CONT;
  } else if constexpr (F == FAM_PMH3) {      // K:462-481
    if (!(s.x <= thr)) return s.fail ? EL_FAIL : EL_DONE;
    const int64_t r = uniform_int_masked(s.st, (uint64_t)m, c.kbits);
    if (r < 0 || s.fail) return EL_FAIL;
    ctx_offer(c, r, s.x, s.e);
    if (++s.i > c.cap) return EL_FAIL;
    const double xl = s.winv * ((double)s.i - 1.0);
    if (xl > thr) return EL_DONE;
    s.x = xl + s.winv * trunc_exp(s.st, T.c3, &s.fail);
    c.points += (xl > c.tprev);
    if (s.i == 2) c.multi++;
    return EL_CONT;
  } else if constexpr (F == FAM_PMH4) {      // K:582-610
    if (!(s.x <= thr)) return s.fail ? EL_FAIL : EL_DONE;
    if (s.fail) return EL_FAIL;
    int32_t k = perm_next_reg(s.st, s.fy, s.i, m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, s.x, s.e);
    s.i++;
    const double gl = T.gam[s.i - 1];
    if (s.winv * gl > thr) return EL_DONE;
    if (s.i == 2) c.multi++;
    c.points += (s.winv * gl > c.tprev);
    if (s.i < m) {
      const double t = trunc_exp(s.st, T.c4[s.i], &s.fail);
      s.x = s.winv * (gl + T.dgam[s.i] * t);
      return EL_CONT;
    }
    const double x = s.winv * (T.gam[m - 1] + T.delta * exp1_from_bits(s.st.next53()));
    if (x <= thr) {
      k = perm_next_reg(s.st, s.fy, (int32_t)m, m);
      if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
      ctx_offer(c, k - 1, x, s.e);
    }
    return EL_DONE;
  } else if constexpr (F == FAM_UW3) {       // K:631-649
    if (!(s.x <= thr)) return EL_DONE;
    const int64_t r = uniform_int_masked(s.st, (uint64_t)m, c.kbits);
    if (r < 0) return EL_FAIL;
    ctx_offer(c, r, s.x, s.e);
    if (++s.i > c.cap) return EL_FAIL;
    const double xl = (double)s.i - 1.0;
    if (xl > thr) return EL_DONE;
    s.x = xl + s.st.uniform01();
    c.points += (xl > c.tprev);
    if (s.i == 2) c.multi++;
    return EL_CONT;
  } else {                                   // uw4, K:734-759
    if (!(s.x <= thr)) return EL_DONE;
    int32_t k = perm_next_reg(s.st, s.fy, s.i, m);
    if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
    ctx_offer(c, k - 1, s.x, s.e);
    s.i++;
    const double xl = (double)s.i - 1.0;
    if (xl > thr) return EL_DONE;
    if (s.i == 2) c.multi++;
    c.points += (xl > c.tprev);
    if (s.i < m) {
      s.x = xl + s.st.uniform01();
      return EL_CONT;
    }
    const double x = ((double)m - 1.0) + s.st.uniform01();
    if (x <= thr) {
      k = perm_next_reg(s.st, s.fy, (int32_t)m, m);
      if (k <= 0) return k == 0 ? EL_NEED_WARP : EL_FAIL;
      ctx_offer(c, k - 1, x, s.e);
    }
    return EL_DONE;
  }
}

}  // namespace pmh
