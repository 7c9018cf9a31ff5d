// pmh_kernel.cuh -- the set-level ProbMinHash kernel (one CTA per set).
//
// Per set: slot table + h_max in shared memory; warps pull chunks of
// elements from a shared counter.  Within a chunk each lane takes one
// element; elements whose expected point count w * thr is small are run
// lane-per-element through the reference recurrence (pmh_sketch.cuh, "mode
// A"); long elements (small sets, heavy weights) and Fisher-Yates elements
// that outgrow the lane's hash map are run warp-cooperatively (pmh_warp.cuh,
// "mode B"); unweighted sets of >= 256 elements keep their equal-length
// elements on the lanes (heavy_points_for).  The final verification
// max_k h_k <= t makes the threshold guess t exact-safe (retry with a larger
// t otherwise).
#pragma once
#include "pmh_warp.cuh"
#include "pmh_split.cuh"

namespace pmh {

#ifndef PMH_CHUNK_DIV
#define PMH_CHUNK_DIV 2       // element chunks per warp and set (at least)
#endif
#ifndef PMH_REFRESH_EVERY
#define PMH_REFRESH_EVERY 16  // batches between forced h_max refreshes (4 / 8 / 16: equal within 1%)
#endif
#ifndef PMH_HEAVY_POINTS
#define PMH_HEAVY_POINTS 16.0   // measured best on config 2 (4 / 6 / 8 / 12 / 16 / 24 / 32 / 48 tried)
#endif
constexpr double HEAVY_POINTS = PMH_HEAVY_POINTS;   // expected points above which mode B runs
// Sets that fill every lane of the CTA (n >= 256) with elements of EQUAL
// weight (the unweighted families) run lane-per-element up to a much longer
// sequence: their lanes stay in step (point counts differ only by the points'
// own randomness), while a warp-cooperative element of 36 points (configs[2]:
// m = 4096, n = 1000) fills 36 of 64 lane slots (unweighted 1 there: 139 ->
// 84 ms).  Below 256 elements the lanes are too few and the warp path wins
// (measured at n = 32 ... 8192, tools/uw_sweep.py).
#ifndef PMH_HEAVY_POINTS_UW
#define PMH_HEAVY_POINTS_UW 256
#endif
#ifndef PMH_HEAVY_UW_MIN_N
#define PMH_HEAVY_UW_MIN_N 256
#endif
#ifndef PMH_HEAVY_POINTS_BIGN
#define PMH_HEAVY_POINTS_BIGN PMH_HEAVY_POINTS
#endif


// Division-free prefilter for the common case of large sets: decide from the
// element's first stream word whether its FIRST point exceeds thr and the
// SECOND point's lower bound does too, in which case the element contributes
// nothing (exactly what the recurrence would conclude).  Weighted families
// compare against thr * w with 2^-40 margins, which dominate every rounding in
// x = fl(fl(1/w) * E) (E >= U for PMH1/2; T exact for PMH3/4), so a rejection
// here is always a rejection there.  Returns false when unsure.
template <int F>
__device__ __forceinline__ bool first_point_rejects(const Tables& T, uint64_t id, double w,
                                                    double thr) {
  const uint64_t b53 = mix64(id + GOLDEN) & ((1ULL << 53) - 1ULL);  // bits 0..52 = word 1
  const double U = (double)b53 * INV53;
  const double lo = 0.99999999999909051, hi = 1.0000000000009095;  // 1 -/+ 2^-40
  if constexpr (F == FAM_UW3 || F == FAM_UW4) {
    return U > thr && 1.0 > thr;                 // x = U, next lower bound 1
  } else if constexpr (F == FAM_PMH1 || F == FAM_PMH2) {
    // next point's lower bound is x itself (x_2 = x + winv E_2 >= x)
    return U * lo > thr * w * hi;
  } else {
    const double c1 = (F == FAM_PMH3) ? T.c3.c1 : T.c4[1].c1;
    const double t = c1 * U;                     // TruncExp fast path (K:130-132)
    if (!(t < 1.0)) return false;
    // x = winv t; next lower bound winv * 1 (PMH3: winv * (2 - 1); PMH4: winv * gamma_1 = winv)
    return t * lo > thr * w * hi && 1.0 * lo > thr * w * hi;
  }
}
// K:279-281 (or a test's lowered cap, pmh_device.cuh)
__device__ __forceinline__ int64_t coupon_cap(int64_t m) {
  if (g_coupon_cap_override > 0) return (int64_t)g_coupon_cap_override;
  return (int64_t)(64.0 * (double)m * (1.0 + log((double)m)) + 64.0);
}


}  // namespace pmh
#include "pmh_wps.cuh"
namespace pmh {

constexpr int SKETCH_THREADS = 256;
// dynamic shared memory per CTA: the 227 KB opt-in limit counts the kernels'
// static __shared__ state too (SetShared and friends, < 1 KB)
constexpr size_t SMEM_DYN_MAX = 227 * 1024 - 1024;

// bytes of one warp's scratch in the CTA kernels (16-byte multiple)
__host__ __device__ inline size_t scratch_bytes(int family) {
  const size_t b = family_uses_fy(family)
                       ? sizeof(WarpScratch)
                       : offsetof(WarpScratch, words) + sizeof(uint64_t) * WIN_STATIC_WORDS;
  return (b + 15) & ~(size_t)15;
}

__host__ __device__ inline size_t sketch_smem_bytes(int family, int64_t m, int threads,
                                                    bool fy16 = false) {
  const int nw = threads / 32;
  size_t b = sizeof(Slot) * (size_t)m;
  b += scratch_bytes(family) * (size_t)nw;
  if (family_uses_fy(family)) b += fy_region_bytes(m, fy16) * (size_t)nw;
  return (b + 15) & ~(size_t)15;
}

// 256-thread CTAs keep 32-bit Fisher-Yates maps while they fit; beyond that
// (m > 4516) the maps are 16-bit (m < 8192 required by the 13-bit values),
// which extends the Fisher-Yates families from m = 4516 to m = 6775.
__host__ __device__ inline bool sketch_fy16_256(int family, int64_t m) {
  return family_uses_fy(family) && sketch_smem_bytes(family, m, SKETCH_THREADS, false) > SMEM_DYN_MAX;
}

// Large m: the slot table alone is 16 m bytes, so the CTA kernel runs ONE set
// per SM; the Fisher-Yates families then run 16 warps per CTA on 16-bit maps
// (2x the warps of the 256-thread layout in the same shared memory).
constexpr int SKETCH_THREADS_BIG = 512;
__host__ __device__ inline bool sketch_use_big(int family, int64_t m) {
  return family_uses_fy(family) && m > 2048 && m < 8192 &&
         sketch_smem_bytes(family, m, SKETCH_THREADS_BIG, true) <= SMEM_DYN_MAX;
}

// Expected points of an element above which it runs warp-cooperatively, for
// a set of n elements in the CTA kernels.  The Fisher-Yates families stay
// within what a lane's hash map holds.
template <int F, bool FY16>
__device__ __forceinline__ int32_t heavy_points_for(bool weighted, int64_t n, int64_t m) {
  double h = HEAVY_POINTS;
  if (n >= PMH_HEAVY_UW_MIN_N) h = weighted ? (double)PMH_HEAVY_POINTS_BIGN : (double)PMH_HEAVY_POINTS_UW;
  if constexpr (family_uses_fy(F)) {
    const uint32_t s = hashfy_slots(fy_region_bytes(m, FY16));
    const double cap = (double)hashfy_room(s) - 4.0;   // HashFY::room less a margin
    if (h > cap) h = cap;
  }
  return (int32_t)h;
}

// Per-warp element loop shared by the CTA-per-set and warp-per-set kernels:
// chunks of up to 32 elements come from `grab` (a shared counter or a private
// cursor); the next chunk's ids/weights are loaded before the current one is
// processed (global-load latency overlaps the work).  Every element first runs
// the division-free first-point prefilter; SURVIVORS are compacted into a
// per-warp queue and run through the full recurrence 32 at a time, so the
// expensive path executes with full warps instead of the few lanes that
// survive in any one chunk (large sets keep only ~1-15%); elements expected
// to be long (or whose Fisher-Yates state outgrows the lane map) run
// warp-cooperatively.
struct SharedGrab {
  static constexpr bool shared = true;
  unsigned* ctr;
  unsigned chunk;
  __device__ __forceinline__ unsigned next(int lane) {
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(ctr, chunk);
    return __shfl_sync(0xffffffffu, b, 0);
  }
};
struct LocalGrab {
  static constexpr bool shared = false;
  unsigned cur;
  unsigned chunk;
  __device__ __forceinline__ unsigned next(int) { const unsigned b = cur; cur += chunk; return b; }
};

// One batch of up to 32 queued survivors, one per lane (mode A), then the
// batch's warp-cooperative elements (mode B) and the h_max refresh.  Kept out
// of line so the register budget of the heavy recurrences does not spill the
// streaming prefilter loop around it (one call per batch, i.e. per ~4-32
// prefilter iterations).  Returns true if an element hit a loop cap.
template <int F, bool FY16, bool HASHFY>
__device__ __forceinline__ bool run_batch(SetCtx& c, const Tables& T, const uint64_t* ids,
                                       const double* w, WarpScratch* wscr, uint32_t* fy_dense,
                                       bool warp_ok, int lane, int take, int qn) {
  bool failed = false;
  const bool act = lane < take;
  const int64_t e = act ? (int64_t)wscr->sq[qn - take + lane] : 0;   // LIFO: the queue's tail
  __syncwarp();
  const int64_t upd0 = c.updates;
  bool heavy = false;
  int status = EL_DONE;
  if (act) {
    const uint64_t id = __ldg(&ids[e]);
    double winv = 1.0;
    if (family_weighted(F) && w) winv = 1.0 / __ldg(&w[e]);
    heavy = warp_ok && ctx_thr(c) > (double)c.heavy_pts * winv;
    if (!heavy) {
      if constexpr (HASHFY && family_uses_fy(F)) {
        HashFY<FY16> fy; fy.reset(fy_dense, lane, hashfy_slots(fy_region_bytes(c.m, FY16)));
        status = run_element<F>(c, T, fy, e, id, winv);
      } else {
        SparseFY fy; fy.reset();
        status = run_element<F>(c, T, fy, e, id, winv);
      }
    }
  }
  if constexpr (HASHFY && family_uses_fy(F)) {
    if (lane == 0) wscr->fy_dirty = 1u;
    __syncwarp();
  }
  if (status == EL_FAIL) failed = true;
  unsigned hm = __ballot_sync(0xffffffffu, act && (heavy || status == EL_NEED_WARP));
  // warp-cooperative elements of this batch, one at a time
  while (hm) {
    const int l = __ffs(hm) - 1;
    hm &= hm - 1;
    const int64_t eh = __shfl_sync(0xffffffffu, e, l);
    const uint64_t idh = __ldg(&ids[eh]);
    const double winvh = (family_weighted(F) && w) ? 1.0 / __ldg(&w[eh]) : 1.0;
    const int st = warp_element<F, FY16>(c, T, *wscr, fy_dense, lane, eh, idh, winvh);
    if (st == EL_FAIL) failed = true;
    if (lane == 0) c.multi++;
    __syncwarp();
  }
  // periodic h_max refresh (every PMH_REFRESH_EVERY batches)
// h_max is kept exact where it matters -- a lowered maximum slot or the last
// slot filling triggers a recompute (ctx_offer, offer_trig) -- so the warp
// scan of all m slots after every batch that lowered ANY slot was redundant
// (configs[1]: PMH1 -7%, PMH2/PMH4 -3%, PMH3 -4% without it); only the
// periodic safety refresh remains
#ifndef PMH_REFRESH_ON_CHANGE
#define PMH_REFRESH_ON_CHANGE 0
#endif
  const bool changed = PMH_REFRESH_ON_CHANGE && __any_sync(0xffffffffu, c.updates != upd0);
  // ... and, for unweighted sets, the FIRST refresh: their table fills only at
  // ~93% of the work (every element contributes equally), in the middle of
  // long lane batches, and the lane whose offer filled the last slot may be
  // deep inside another warp's batch.  The first warp that ends a batch with
  // the table full and no stop limit yet computes it; the other warps' lanes
  // read h_max at every step (configs[2] uw2 158 -> 150 ms, uw1 / uw4 -0.5 /
  // -0.8%, uw3 +0.6%; on weighted sets the check cost the configs[1] step 0.2%)
#ifndef PMH_FIRST_REFRESH
#define PMH_FIRST_REFRESH 1
#endif
  bool first = false;
  if (PMH_FIRST_REFRESH && !w && lane == 0 &&
      *(volatile unsigned long long*)c.hmax_bits == EMPTY_H &&
      *(volatile unsigned*)c.filled >= (unsigned)c.m)
    // one warp only: EMPTY_H - 1 is still an upper bound of every slot
    first = atomicCAS(c.hmax_bits, EMPTY_H, EMPTY_H - 1ULL) == EMPTY_H;
  const bool trig = __any_sync(0xffffffffu, c.trig || first);
  c.trig = false;
  if (changed || trig || ++c.since_refresh >= PMH_REFRESH_EVERY) {
    hmax_refresh_warp(c, lane);
    c.since_refresh = 0;
  }
  return failed;
}

// The streaming loop: each lane takes PMH_EPL elements per chunk (chunk =
// 32 * PMH_EPL, coalesced per j), so the per-chunk costs (grab, stop-limit
// read, ballots, queue append, loop control) are amortised and PMH_EPL
// independent loads and prefilters are in flight per lane.  The ids are in
// L2 (prefetched per set) and the weights too (the weight sum), so no
// register prefetch is kept across the heavy batch.  32-bit element indices
// (sets hold < 2^31 elements); rejections counted in a register (stats only).
// (PMH_EPL is defined in pmh_warp.cuh next to the queue it sizes)
template <int F, bool FY16, bool HASHFY, class Grab>
__device__ __forceinline__ void warp_elements(SetCtx& c, const Tables& T, const uint64_t* ids,
                                           const double* w, int64_t n, int64_t chunk, Grab& grab,
                                           WarpScratch* wscr, uint32_t* fy_dense, bool warp_ok,
                                           bool& failed, int lane) {
  const volatile unsigned long long* hb = c.hmax_bits;
  const double tg = c.tguess;
  const uint32_t n32 = (uint32_t)n, ch = (uint32_t)chunk;   // ch <= 32 * PMH_EPL
  uint32_t rej = 0;                            // prefilter rejections (stats)
  int qn = 0;                                  // queued survivors (warp-uniform)
  for (;;) {
    const uint32_t base = grab.next(lane);
    const bool more = base < n32;
#ifndef PMH_ROLL_PREFETCH
#define PMH_ROLL_PREFETCH 8   // chunks ahead (0: off)
#endif
    if constexpr (Grab::shared && PMH_ROLL_PREFETCH > 0) {
      // rolling L2 prefetch: the chunk some warp of the CTA will grab
      // PMH_ROLL_PREFETCH grabs from now (lanes 0-7: its ids lines, 16-23: its
      // weights), so the element loads below find L2 instead of HBM latency
      const uint32_t o = 16u * (uint32_t)(lane & 15);
      const uint32_t pe = base + ch * PMH_ROLL_PREFETCH + o;
      if (o < ch && pe < n32) {
        if (lane < 16) asm volatile("prefetch.global.L2 [%0];" ::"l"(ids + pe));
        else if (family_weighted(F) && w) asm volatile("prefetch.global.L2 [%0];" ::"l"(w + pe));
      }
    }
    if (more) {
      uint64_t id[PMH_EPL];
      double wv[PMH_EPL];
      bool act[PMH_EPL];
#pragma unroll
      for (int j = 0; j < PMH_EPL; j++) {
        const uint32_t o = (uint32_t)lane + 32u * j;
        const uint32_t e = base + o;
        act[j] = o < ch && e < n32;
        id[j] = act[j] ? __ldg(&ids[e]) : 0ULL;
        wv[j] = (family_weighted(F) && w && act[j]) ? __ldg(&w[e]) : 1.0;
      }
      const double hm = __longlong_as_double((long long)*hb);
      const double thr = hm < tg ? hm : tg;
#pragma unroll
      for (int j = 0; j < PMH_EPL; j++) {
        const bool surv = act[j] && !first_point_rejects<F>(T, id[j], wv[j], thr);
        rej += act[j] && !surv;
        const unsigned sm = __ballot_sync(0xffffffffu, surv);
        PMH_ASSERT(qn + __popc(sm) <= SQ_CAP);
        if (surv) wscr->sq[qn + __popc(sm & ((1u << lane) - 1u))] = (int32_t)(base + (uint32_t)lane + 32u * j);
        qn += __popc(sm);
      }
      __syncwarp();
    }
    while (qn >= 32 || (!more && qn > 0)) {
      const int take = qn < 32 ? qn : 32;
      if (run_batch<F, FY16, HASHFY>(c, T, ids, w, wscr, fy_dense, warp_ok, lane, take, qn)) failed = true;
      qn -= take;
      __syncwarp();
    }
    if (!more) break;
  }
  if (0.0 > c.tprev) c.points += rej;          // rejected first points
}

// per-CTA shared state of one set (or one part of a split set)
struct SetShared {
  unsigned long long hmax;
  unsigned int filled;
  unsigned int next;
  int retry;
  double red[32];
  long long redl[32];
};

// The verified minima of elements [e0, e1) of the set at `off` in the shared
// slot table (in-set element indices); the threshold guess uses the range's
// own total weight.  Returns true if an element hit a loop cap.  Counters of
// the range in pts/mul/upd (CTA-reduced, valid in every thread).
template <int F, bool FY16>
__device__ __forceinline__ bool sketch_range(const SketchArgs& a, int64_t off, int64_t e0,
                                             int64_t e1, Slot* slots, WarpScratch* wscr,
                                             uint32_t* fy_dense, bool warp_ok, SetShared& sh,
                                             long long* pts, long long* mul, long long* upd,
                                             double w_given) {
  const int lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const int64_t m = a.m;
  const int64_t n = e1 - e0;
  const uint64_t* ids = a.ids + off + e0;
  const double* w = a.w ? a.w + off + e0 : nullptr;
  for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
    slots[k].h = EMPTY_H;
    slots[k].idx = EMPTY_IDX;
  }
  // Pull the range's ids into L2 while the weights are summed (the weights
  // arrive there by the sum itself): the element loop then reads its chunks
  // from L2 instead of HBM.
  // (not for weighted sets whose W is known, where the element loop is the
  // first and only reader of the weights too: with ~440 sets in flight
  // the prefetched lines of the large ones were evicted before their use --
  // ncu showed the ids read twice from DRAM, at no gain in time)
  if (!(family_weighted(F) && w && w_given > 0.0))
    for (int64_t L = threadIdx.x; L * 16 < n; L += blockDim.x)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(ids + L * 16));
  double W;
  if (family_weighted(F) && w && w_given > 0.0) {
    // total weight known in advance (computed once per batch, or the caller's
    // for the non-streaming variants): no weight pre-pass, the element loop
    // reads the weights once.  Any W > 0 is exact-safe (it only sizes the
    // threshold guess that the final verification checks).
    __syncthreads();
    W = w_given;
  } else if (family_weighted(F) && w) {
    // four independent loads in flight per thread (latency-bound otherwise)
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
    const int64_t B = blockDim.x;
    int64_t e = threadIdx.x;
    for (; e + 3 * B < n; e += 4 * B) {
      p0 += __ldg(&w[e]);
      p1 += __ldg(&w[e + B]);
      p2 += __ldg(&w[e + 2 * B]);
      p3 += __ldg(&w[e + 3 * B]);
    }
    for (; e < n; e += B) p0 += __ldg(&w[e]);
    W = block_sum((p0 + p1) + (p2 + p3), sh.red);
  } else {
    W = (double)n;
  }
  if (threadIdx.x == 0) { sh.hmax = EMPTY_H; sh.filled = 0; }

  SetCtx c;
  c.slots = slots;
  c.hmax_bits = &sh.hmax;
  c.filled = &sh.filled;
  c.m = (int32_t)m;
  c.kbits = bits_for(m);
  c.cap = (int32_t)coupon_cap(m);
  c.points = 0; c.updates = 0; c.multi = 0; c.tprev = -1.0; c.since_refresh = 0;
  c.trig = false;
  c.eoff = (int32_t)e0;
  c.heavy_pts = heavy_points_for<F, FY16>(w != nullptr, n, m);
  double tg = (double)m * (log((double)m) + guess_const(a.tconst, n)) / W;
  if (!(tg > 0.0)) tg = __longlong_as_double(0x7FF0000000000000LL);
  bool failed = false;
  int64_t chunk = (n + PMH_CHUNK_DIV * nwarps - 1) / (PMH_CHUNK_DIV * nwarps);
  chunk = chunk < 1 ? 1 : (chunk > 32 * PMH_EPL ? 32 * PMH_EPL : chunk);

  for (int attempt = 0;; attempt++) {
    c.tguess = tg;
    if (threadIdx.x == 0) sh.next = 0;
    __syncthreads();
    SharedGrab grab{&sh.next, (unsigned)chunk};
    warp_elements<F, FY16, true>(c, a.T, ids, w, n, chunk, grab, wscr, fy_dense, warp_ok, failed, lane);
    __syncthreads();
    // verification: every slot non-empty and <= tguess
    unsigned long long mx = 0;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      unsigned long long h = slots[k].h;
      mx = h > mx ? h : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
      mx = v > mx ? v : mx;
    }
    if (threadIdx.x == 0) sh.retry = 0;
    __syncthreads();
    if (lane == 0 && __longlong_as_double((long long)mx) > tg) atomicOr(&sh.retry, 1);
    const int any_fail = __syncthreads_or(failed ? 1 : 0);
    if (any_fail) { failed = true; break; }
    if (!sh.retry) break;
    c.tprev = tg;
    tg = attempt >= 2 ? __longlong_as_double(0x7FF0000000000000LL) : tg * 4.0;
    __syncthreads();
  }
  if (a.stats) {
    *pts = block_sum_ll(c.points, sh.redl);
    *mul = block_sum_ll(c.multi, sh.redl);
    *upd = block_sum_ll(c.updates, sh.redl);
  }
  return failed;
}

// Dynamic shared memory: Slot[m] | WarpScratch[nwarps] | int32 FY[nwarps][m+1]
#ifndef SKETCH_MINBLOCKS
#define SKETCH_MINBLOCKS 3   // 80 registers, 3 CTAs/SM: measured 3-12% faster than 2
#endif
// ProbMinHash1 (labels with replacement, log1p points: the smallest per-lane
// state) gains from a fourth CTA per SM even at 64 registers with ~220 bytes
// of spills (configs[1]: 3.49 -> 3.18 ms); ProbMinHash2 / 4 lose 5-10% there
// (and their shared memory holds three CTAs anyway), ProbMinHash3 is unchanged.
#ifndef PMH_MINBLOCKS_PMH1
#define PMH_MINBLOCKS_PMH1 4
#endif
template <int F>
constexpr int sketch_minblocks() { return F == FAM_PMH1 ? PMH_MINBLOCKS_PMH1 : SKETCH_MINBLOCKS; }

template <int F, bool FY16>
__device__ __forceinline__ void sketch_cta_setup(unsigned char* smem, int64_t m, Slot** slots,
                                                 WarpScratch** wscr, uint32_t** fy_dense) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  *slots = reinterpret_cast<Slot*>(smem);
  *wscr = reinterpret_cast<WarpScratch*>(smem + sizeof(Slot) * m + scratch_bytes(F) * (size_t)wid);
  *fy_dense = reinterpret_cast<uint32_t*>(smem + sizeof(Slot) * m + scratch_bytes(F) * (size_t)nwarps +
                                          fy_region_bytes(m, FY16) * (size_t)wid);
  if (family_uses_fy(F)) {  // epoch 0 never matches: the map starts empty
    fy_clear<FY16>(*fy_dense, m, lane);
    if (lane == 0) { (*wscr)->epoch = 0; (*wscr)->fy_dirty = 0u; }
  }
}

// FY16: 16-bit dense Fisher-Yates maps (EpochFY<true>), a compile-time choice
// so the other instantiations carry no trace of it (these kernels are
// instruction-cache bound)
template <int F, int NT = SKETCH_THREADS, bool FY16 = false>
__global__ void __launch_bounds__(NT, (NT == SKETCH_THREADS ? sketch_minblocks<F>() : 1))
    sketch_sets_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SetShared sh;
  const int64_t m = a.m;
  Slot* slots;
  WarpScratch* wscr;
  uint32_t* fy_dense;
  sketch_cta_setup<F, FY16>(smem, m, &slots, &wscr, &fy_dense);
  // mode B needs static point offsets (power-of-two m) unless the family
  // parses its bit offsets (Fisher-Yates families)
  const bool warp_ok = family_uses_fy(F) || ((m & (m - 1)) == 0);

  // with a small-set kernel running beside it, this kernel takes the large
  // sets only: the prefix order[0, counts[0]) of the LPT order, minus the
  // split sets at its front
  const int64_t n_mine = a.counts ? (int64_t)a.counts[0] : a.nsets;
  const int64_t first = a.split_info ? (int64_t)a.split_info[0] : 0;
  for (int64_t bs = first + blockIdx.x; bs < n_mine; bs += gridDim.x) {
    const int64_t s = a.order ? (int64_t)a.order[bs] : bs;
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (threadIdx.x == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    long long pts = 0, mul = 0, upd = 0;
    const bool failed = sketch_range<F, FY16>(a, off, 0, n, slots, wscr, fy_dense, warp_ok, sh, &pts,
                                        &mul, &upd, a.setw ? a.setw[s] : -1.0);
    if (failed && threadIdx.x == 0) {
      atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
      atomicMin(a.err_set, (long long)s);
    }
    uint64_t* sig = a.sig + (size_t)s * m;
    const uint64_t* ids = a.ids + off;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const unsigned long long ix = slots[k].idx;
      sig[k] = ix < (unsigned long long)n ? ids[ix] : 0ULL;
    }
    if (a.stats && threadIdx.x == 0) {
      a.stats[s * 3 + 0] = pts;
      a.stats[s * 3 + 1] = mul;
      a.stats[s * 3 + 2] = upd;
    }
    __syncthreads();
  }
}

// Parts of the split sets (pmh_split.cuh): persistent CTAs, each part's
// verified minima merged into the set's global table.
template <int F, bool FY16 = false>
__global__ void __launch_bounds__(SKETCH_THREADS, sketch_minblocks<F>())
    sketch_split_kernel(SketchArgs a, SplitArgs sp) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ SetShared sh;
  __shared__ long long s_t;
  const int64_t m = a.m;
  Slot* slots;
  WarpScratch* wscr;
  uint32_t* fy_dense;
  sketch_cta_setup<F, FY16>(smem, m, &slots, &wscr, &fy_dense);
  const bool warp_ok = family_uses_fy(F) || ((m & (m - 1)) == 0);
  SplitPart p;
  while (split_next_part(sp, &s_t, &p)) {
    long long pts = 0, mul = 0, upd = 0;
    const bool failed = sketch_range<F, FY16>(a, p.off, p.e0, p.e1, slots, wscr, fy_dense, warp_ok, sh,
                                        &pts, &mul, &upd, -1.0);
    if (failed && threadIdx.x == 0) {
      atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
      atomicMin(a.err_set, (long long)p.s);
    }
    Slot* gt = sp.gtab + (size_t)p.i * m;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
      const Slot v = slots[k];
      if (v.idx != EMPTY_IDX) slot_offer_global(&gt[k], v.h, v.idx);
    }
    if (a.stats && threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&a.stats[p.s * 3 + 0], (unsigned long long)pts);
      atomicAdd((unsigned long long*)&a.stats[p.s * 3 + 1], (unsigned long long)mul);
      atomicAdd((unsigned long long*)&a.stats[p.s * 3 + 2], (unsigned long long)upd);
    }
    __syncthreads();
  }
}

}  // namespace pmh

namespace pmh {

// ---------------------------------------------------------------------------
// Small sets (n <= small_n(m)): one WARP per set, with a private slot table,
// scratch and Fisher-Yates map in shared memory, running the same element
// loop as the CTA kernel (warp_elements) over a private cursor.  For m = 1024
// this is the tiny sets (n <= 3: their coupon-collector phase keeps one warp
// busy and a CTA-per-set layout would idle 7 of 8 warps); for small m
// (configs[3]: m = 64, n = 100) whole sets are cheap and the CTA kernel's
// per-set barriers dominate, so they all run warp-per-set.
// ---------------------------------------------------------------------------
#ifndef PMH_SMALL_N
#define PMH_SMALL_N 1
#endif
#ifndef PMH_SMALL_N_STATIC
#define PMH_SMALL_N_STATIC 7
#endif
// sets up to this size run warp-per-set at large m (measured on configs[1]
// in round 1: cutoff 7 vs 3 is 2% / 6% faster for ProbMinHash 1 / 3 and 4%
// slower for the Fisher-Yates families 2 / 4, whose warp-per-set map costs
// more; ProbMinHash1 has its own cutoff since, small_n_for below).  The
// Fisher-Yates families send only singletons there: a warp runs a set's long
// elements one after another, and 2-3 elements of ~m points each made those
// sets the latency floor of a small batch (1/8 shard of configs[1]: the
// n < 4 class 0.89 -> 0.38 ms for ProbMinHash2, 0.53 -> 0.25 for 4; the
// whole batch unchanged)
#ifndef PMH_SMALL_N_PMH1
#define PMH_SMALL_N_PMH1 3
#endif
constexpr int64_t SMALL_N = PMH_SMALL_N;
constexpr int64_t SMALL_N_STATIC = PMH_SMALL_N_STATIC;
// warp-per-set cutoff: for large m only tiny sets; for m <= 256 whole sets are
// cheap enough for one warp up to a few hundred elements (configs[3]: the
// m <= 64 kernel of pmh_wps.cuh takes them all).  Above that the CTA kernel
// wins, earlier for the Fisher-Yates families since their lanes got hash maps
// (tools/uw_sweep.py, weighted sets at m = 128 / 256, n = 20 ... 500; configs[4],
// m = 256, n = 500: ProbMinHash4 19.2 -> 17.5 ms)
__host__ __device__ inline int64_t small_n_for(int family, int64_t m) {
  if (wps_eligible(family, m)) return (int64_t)WPS_NMAX;   // pmh_wps.cuh
  if (m <= 256) {
    if (family_uses_fy(family)) return m <= 128 ? 384 : 128;
    return m <= 128 ? 512 : 384;
  }
  if (family_uses_fy(family)) return SMALL_N;
  // ProbMinHash1 since its CTA kernel runs four CTAs per SM: 3 (configs[1]:
  // 3.19 -> 3.09 ms; 1: 3.30, 2: 3.10, 5: 3.15, 7: 3.19, 15: 3.23)
  return family == FAM_PMH1 ? (int64_t)PMH_SMALL_N_PMH1 : SMALL_N_STATIC;
}

struct WarpSetVars {
  unsigned long long hmax;
  unsigned int filled;
  unsigned int pad;
};

__host__ __device__ inline size_t small_warp_bytes(int family, int64_t m) {
  size_t b = sizeof(Slot) * (size_t)m + sizeof(WarpScratch) + sizeof(WarpSetVars);
  if (family_uses_fy(family)) b += sizeof(uint32_t) * (size_t)(m + 1);
  return (b + 15) & ~(size_t)15;
}

template <int F>
__global__ void __launch_bounds__(128) sketch_small_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpc = blockDim.x >> 5;
  const int64_t m = a.m;
  unsigned char* base = smem + small_warp_bytes(F, m) * (size_t)wid;
  Slot* slots = reinterpret_cast<Slot*>(base);
  WarpScratch* ws = reinterpret_cast<WarpScratch*>(base + sizeof(Slot) * m);
  WarpSetVars* wv = reinterpret_cast<WarpSetVars*>(base + sizeof(Slot) * m + sizeof(WarpScratch));
  uint32_t* fy = reinterpret_cast<uint32_t*>(base + sizeof(Slot) * m + sizeof(WarpScratch) +
                                             sizeof(WarpSetVars));
  if (family_uses_fy(F)) {
    for (int64_t p = lane; p <= m; p += 32) fy[p] = 0;
    if (lane == 0) { ws->epoch = 0; ws->fy_dirty = 0u; }
  }
  const int64_t n_large = (int64_t)a.counts[0];
  const int64_t n_small = a.nsets - n_large;
  const bool warp_ok = family_uses_fy(F) || ((m & (m - 1)) == 0);
  for (int64_t bs = (int64_t)blockIdx.x * wpc + wid; bs < n_small; bs += (int64_t)gridDim.x * wpc) {
    const int64_t s = (int64_t)a.order[n_large + bs];
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    if (n <= 0) {
      if (lane == 0) atomicMin(a.err_set, (long long)s);
      continue;
    }
    const uint64_t* ids = a.ids + off;
    const double* w = a.w ? a.w + off : nullptr;
    for (int64_t k = lane; k < m; k += 32) { slots[k].h = EMPTY_H; slots[k].idx = EMPTY_IDX; }
    double W = 0.0;
    if (family_weighted(F) && w && a.setw && a.setw[s] > 0.0) {
      W = a.setw[s];
    } else if (family_weighted(F) && w) {
      for (int64_t e = lane; e < n; e += 32) W += w[e];
      for (int o = 16; o > 0; o >>= 1) W += __shfl_xor_sync(0xffffffffu, W, o);
    } else {
      W = (double)n;
    }
    if (lane == 0) { wv->hmax = EMPTY_H; wv->filled = 0; }
    __syncwarp();
    SetCtx c;
    c.slots = slots;
    c.hmax_bits = &wv->hmax;
    c.filled = &wv->filled;
    c.m = (int32_t)m;
    c.kbits = bits_for(m);
    c.cap = (int32_t)coupon_cap(m);
    c.points = 0; c.updates = 0; c.multi = 0; c.tprev = -1.0; c.since_refresh = 0;
  c.trig = false;
    c.eoff = 0;
    c.heavy_pts = (int32_t)HEAVY_POINTS;
    double tg = (double)m * (log((double)m) + guess_const(a.tconst, n)) / W;
    if (!(tg > 0.0)) tg = __longlong_as_double(0x7FF0000000000000LL);
    bool failed = false;
    for (int attempt = 0;; attempt++) {
      c.tguess = tg;
      LocalGrab grab{0u, 32u * PMH_EPL};
      warp_elements<F, false, false>(c, a.T, ids, w, n, 32 * PMH_EPL, grab, ws, fy, warp_ok, failed, lane);
      unsigned long long mx = 0;
      for (int64_t k = lane; k < m; k += 32) {
        const unsigned long long h = slots[k].h;
        mx = h > mx ? h : mx;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = v > mx ? v : mx;
      }
      if (failed || !(__longlong_as_double((long long)mx) > tg)) break;
      c.tprev = tg;
      tg = attempt >= 2 ? __longlong_as_double(0x7FF0000000000000LL) : tg * 4.0;
    }
    if (failed && lane == 0) {
      atomicOr(a.err_flags, (unsigned long long)ERRF_RANDOMNESS);
      atomicMin(a.err_set, (long long)s);
    }
    uint64_t* sig = a.sig + (size_t)s * m;
    for (int64_t k = lane; k < m; k += 32) {
      const unsigned long long ix = slots[k].idx;
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
}

}  // namespace pmh
