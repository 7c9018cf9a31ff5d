// pmh_warp.cuh -- warp-cooperative ("lane = point") element processing.
//
// An element whose point sequence is long (small sets: the coupon-collector
// phase needs ~m(ln m + c) points per set, SURVEY.md §7 hard parts) is
// processed by a whole warp in batches of up to 32 consecutive points:
//   * the 32 stream words covering the batch are generated once, one mix64
//     per lane, into a per-warp shared-memory window (2048 bits);
//   * point bit offsets are static for labels with replacement and power-of-
//     two m (53 + log2 m bits per point, K:97-110 never rejects), so lanes
//     decode their point directly; TruncExp's fast path (K:130-132) is
//     speculated and the first slow-path lane ends the batch after finishing
//     its draw sequentially;
//   * labels without replacement (PMH2/PMH4/uw4, K:222-235) have data-
//     dependent widths: lane 0 parses the batch's bit offsets and runs the
//     lazy Fisher-Yates steps on a dense per-warp shared map, then all lanes
//     evaluate the floating-point work in parallel;
//   * PMH1/PMH2's running sum x_i = fl(x_{i-1} + d_i) is an ordered fold: lane
//     p adds d_0..d_p in order, which is exactly the reference's sequence of
//     roundings (K:328, K:440);
//   * points are valid while x <= thr (x is increasing along an element); the
//     valid prefix is offered to the slot table.
#pragma once
#include "pmh_sketch.cuh"

namespace pmh {

constexpr uint32_t WIN_BITS = 2048;  // 32 words

// elements per lane per chunk of the streaming loop (pmh_kernel.cuh); the
// survivor queue holds < 32 leftovers plus one chunk: 32 * (PMH_EPL + 1)
#ifndef PMH_EPL
#define PMH_EPL 4
#endif
constexpr int SQ_CAP = 32 * (PMH_EPL + 1);

// The fields the static families (labels with replacement) use come first:
// their kernels allocate only that prefix per warp (scratch_bytes), which is
// what lets three m = 4096 sets (64 KB slot tables) share an SM.
struct WarpScratch {
  double dbuf[32];      // per-point increments of the ordered fold
  uint32_t q;           // points parsed
  uint32_t flags;       // bit0: batch ended by a slow path; bit1: fail
  uint64_t next_off;    // absolute bit offset after the batch
  uint32_t epoch;       // Fisher-Yates map epoch (one per warp-processed element)
  uint32_t fy_dirty;    // the map region last held the lanes' hash maps (HashFY): clear before use
  int32_t sq[SQ_CAP];   // survivor queue of the large-set path (element indices, LIFO)
  uint64_t words[65];   // window: 33-38 words for static offsets; 64 for the parallel
                        // Fisher-Yates parse, +1 guard
  // ---- Fisher-Yates families only ----
  uint32_t eoff[32];    // window-relative bit offset of each point's first draw
  int32_t lab[32];      // 1-based labels
  uint32_t gm[32];      // parallel Fisher-Yates: lanes whose target is i0 + k
};
constexpr int WIN_STATIC_WORDS = 40;   // words[] entries the static families touch (<= 38)

// Dense per-warp Fisher-Yates map with O(1) reset: entry = epoch << 16 | value
// (the versioned lazy permutation of K:222-235 / lazyperm.py, one epoch per
// element).  Requires m < 65536.  With h16 the entries are 16-bit, epoch << 13
// | value (m < 8192, epochs 1..7, the map cleared when they wrap): half the
// shared memory, so large-m sets run 16 warps per CTA (FY_EPOCHS16).
constexpr uint32_t FY_EPOCHS32 = 0x10000u, FY_EPOCHS16 = 8u;
template <bool H16>
struct EpochFY {
  static constexpr bool h16 = H16;
  uint32_t* a;
  uint32_t ep;
  __device__ __forceinline__ int32_t get(int32_t p) const {
    PMH_ASSERT(p >= 0 && p < (h16 ? 8192 : 65536));
    if constexpr (H16) {
      const uint32_t v = reinterpret_cast<const uint16_t*>(a)[p];
      return (v >> 13) == ep ? (int32_t)(v & 0x1fffu) : p;
    }
    const uint32_t v = a[p];
    return (v >> 16) == ep ? (int32_t)(v & 0xffffu) : p;
  }
  __device__ __forceinline__ void set(int32_t p, int32_t v) {
    PMH_ASSERT(p >= 0 && v >= 0 && (h16 ? (p < 8192 && v < 8192 && ep < 8) : (p < 65536 && v < 65536)));
    if constexpr (H16) reinterpret_cast<uint16_t*>(a)[p] = (uint16_t)((ep << 13) | (uint32_t)v);
    else a[p] = (ep << 16) | (uint32_t)v;
  }
};

// bytes of one warp's dense Fisher-Yates map (16-byte multiple)
__host__ __device__ inline size_t fy_map_bytes(int64_t m, bool fy16) {
  return ((fy16 ? 2 : 4) * (size_t)(m + 1) + 15) & ~(size_t)15;
}
// bytes of one warp's map REGION in the CTA kernels: the dense map or the
// lanes' hash maps (HashFY below; at least 32 slots per lane), whichever is larger
constexpr size_t HASHFY_MIN_BYTES = 32 * 128;
__host__ __device__ inline size_t fy_region_bytes(int64_t m, bool fy16) {
  const size_t d = fy_map_bytes(m, fy16);
  return d > HASHFY_MIN_BYTES ? d : HASHFY_MIN_BYTES;
}

// clear a dense map (entries 0..m) -- epoch 0 never matches
template <bool H16>
__device__ __forceinline__ void fy_clear(uint32_t* fy, int64_t m, int lane) {
  if constexpr (H16) {
    uint16_t* f = reinterpret_cast<uint16_t*>(fy);
    for (int64_t p = lane; p <= m; p += 32) f[p] = 0;
  } else {
    for (int64_t p = lane; p <= m; p += 32) fy[p] = 0;
  }
}

// Per-LANE lazy Fisher-Yates maps for the lane-per-element path, in the SAME
// shared-memory region as the warp's dense map (a warp runs its lanes'
// elements first, then the batch's warp-cooperative ones; WarpScratch.fy_dirty
// tells warp_el_fy to clear the region before the dense map uses it again).
// Lane l owns words l, l + 32, l + 64, ... (its own bank: conflict-free), an
// open-addressing table of S = 2^k <= 64 slots, entry = pos << 16 | value
// (m < 65536), linear probing from pos & (S - 1); which slots are in use is a
// 64-bit register mask, so a new element starts with an O(1) reset.  The
// register-resident SparseFY it replaces held 16 entries in 32 registers and
// scanned all of them per step.
// BLOOM (the large-m layout: 64 slots per lane, filled to 0.7-0.9 by the 36-60
// steps of a configs[2] element): register filters end most lookups -- nearly
// all of them are of positions never stored, since m >> steps -- without a
// probe: a 128-bit Bloom filter (one hashed bit per stored position) and an
// exact mask of the stored positions < 64.  Insertion is a bit scan of `used`.
// configs[2] uw4 113 -> 92 ms, uw2 200 -> 158 ms in all (a
// triangular probe sequence was better only before the filters).  At
// m = 1024 (32 slots, <= 0.6 full) the filters' registers cost the
// 80-register kernels more than the probes (PMH4 +4%): plain probes there.
#ifndef PMH_HASHFY_ROOM_SHIFT
#define PMH_HASHFY_ROOM_SHIFT 4
#endif
// entries a lane's table of `slots` takes (15/16 of it: 7/8 sent three times as many
// long unweighted-2 elements to the warp path, configs[2] uw2 +4%)
__host__ __device__ inline uint32_t hashfy_room(uint32_t slots) {
  return slots - (slots >> PMH_HASHFY_ROOM_SHIFT);
}
template <bool BLOOM>
struct HashFY {
  uint32_t* a;        // region + lane
  uint64_t used;      // slots in use
  uint64_t bloom, bloom1;   // BLOOM: 128-bit filter, one hashed bit per stored position >= 64
  uint64_t low;       // BLOOM: exactly which positions < 64 are stored.  Step i looks up
                      // position i (< 64 for the first 63 steps), stored only if an
                      // earlier target fell that low: this lookup then never probes
  uint32_t mask;      // S - 1
  uint32_t room;      // entries left before the element goes to the warp path
  __device__ __forceinline__ void reset(uint32_t* region, int lane, uint32_t slots) {
    a = region + lane;
    used = 0ULL;
    bloom = 0ULL;
    bloom1 = 0ULL;
    low = 0ULL;
    mask = slots - 1u;
    room = hashfy_room(slots);
  }
  static __device__ __forceinline__ uint32_t bloom_bit(uint32_t p) { return (p * 0x9E3779B1u) >> 25; }
  // value stored for position p (p itself if absent); *slot = its slot, or -1
  __device__ __forceinline__ int32_t lookup(uint32_t p, int* slot) const {
    *slot = -1;
    if (BLOOM) {
      if (p < 64u) { if (!((low >> p) & 1ULL)) return (int32_t)p; }
      else {
        const uint32_t bb = bloom_bit(p);
        if (!((((bb & 64u) ? bloom1 : bloom) >> (bb & 63u)) & 1ULL)) return (int32_t)p;
      }
    }
    uint32_t s = p & mask;
    while ((used >> s) & 1ULL) {
      const uint32_t en = a[s << 5];
      if ((en >> 16) == p) { *slot = (int)s; return (int32_t)(en & 0xffffu); }
      s = (s + 1u) & mask;
    }
    return (int32_t)p;
  }
  // first free slot at or (cyclically) after p's home slot: where linear
  // probing inserts an absent position (a bit scan of `used`, no memory access)
  __device__ __forceinline__ uint32_t free_slot(uint32_t p) const {
    const uint32_t s0 = p & mask;
    const uint64_t all = mask == 63u ? ~0ULL : ((1ULL << (mask + 1u)) - 1ULL);
    const uint64_t fr = ~used & all;
    const uint64_t hi = fr & (~0ULL << s0);
    PMH_ASSERT(fr != 0ULL);   // room < slots: a free slot always exists
    return (uint32_t)(__ffsll((long long)(hi ? hi : fr)) - 1);
  }
  // one lazy Fisher-Yates step (K:222-235): returns perm[j] and sets
  // perm[j] = perm[i] (both read before the write); 0 when the table is full
  __device__ __forceinline__ int32_t swap_step(int32_t i, int32_t j) {
    if constexpr (!BLOOM) {   // plain probes: the search for j ends on its insertion slot
      int32_t vj = j, vi = i;
      uint32_t s = (uint32_t)j & mask;
      bool found = false;
      while ((used >> s) & 1ULL) {
        const uint32_t en = a[s << 5];
        if ((en >> 16) == (uint32_t)j) { vj = (int32_t)(en & 0xffffu); found = true; break; }
        s = (s + 1u) & mask;
      }
      if (i == j) {
        vi = vj;
      } else {
        uint32_t t = (uint32_t)i & mask;
        while ((used >> t) & 1ULL) {
          const uint32_t en = a[t << 5];
          if ((en >> 16) == (uint32_t)i) { vi = (int32_t)(en & 0xffffu); break; }
          t = (t + 1u) & mask;
        }
      }
      if (!found) {
        if (room == 0u) return 0;
        room--;
        used |= 1ULL << s;
      }
      a[s << 5] = ((uint32_t)j << 16) | (uint32_t)vi;
      return vj;
    }
    int sj, si;
    const int32_t vj = lookup((uint32_t)j, &sj);
    const int32_t vi = i == j ? vj : lookup((uint32_t)i, &si);
    uint32_t s = (uint32_t)sj;
    if (sj < 0) {
      if (room == 0u) return 0;
      room--;
      s = free_slot((uint32_t)j);
      used |= 1ULL << s;
      if (BLOOM) {
        if ((uint32_t)j < 64u) low |= 1ULL << j;
        else {
          const uint32_t bb = bloom_bit((uint32_t)j);
          if (bb & 64u) bloom1 |= 1ULL << (bb & 63u); else bloom |= 1ULL << bb;
        }
      }
    }
    PMH_ASSERT(s <= mask && j > 0 && j < 65536 && vi > 0 && vi < 65536);
    a[s << 5] = ((uint32_t)j << 16) | (uint32_t)vi;
    return vj;
  }
};

// slots per lane of the HashFY tables that fit a per-warp region of `bytes`
__host__ __device__ inline uint32_t hashfy_slots(size_t bytes) {
  uint32_t s = 64;
  while (s > 1 && (size_t)s * 128 > bytes) s >>= 1;
  return s;
}

// clear a whole map region (16-byte stores)
__device__ __forceinline__ void fy_clear_region(uint32_t* fy, size_t bytes, int lane) {
  uint4* p = reinterpret_cast<uint4*>(fy);
  for (size_t k = lane; k < bytes / 16; k += 32) p[k] = make_uint4(0u, 0u, 0u, 0u);
}

__device__ __forceinline__ uint64_t win_bits(const uint64_t* w, uint32_t rel, uint32_t k) {
  const uint32_t i = rel >> 6, sh = rel & 63;
  PMH_ASSERT(i < 65 && !(sh && sh + k > 64 && i + 1 >= 65));
  uint64_t v = w[i] >> sh;
  if (sh && sh + k > 64) v |= w[i + 1] << (64 - sh);
  return k == 64 ? v : (v & ((1ULL << k) - 1ULL));
}

constexpr uint32_t WIN2_BITS = 4096;  // 64 words

__device__ __forceinline__ void win_load64(WarpScratch& ws, uint64_t id, uint64_t wb, int lane) {
  ws.words[lane] = stream_word(id, wb + 1 + (uint64_t)lane);
  ws.words[lane + 32] = stream_word(id, wb + 33 + (uint64_t)lane);
  if (lane == 0) ws.words[64] = stream_word(id, wb + 65);
  __syncwarp();
}

__device__ __forceinline__ void win_load(WarpScratch& ws, uint64_t id, uint64_t wb, int lane) {
  ws.words[lane] = stream_word(id, wb + 1 + (uint64_t)lane);
  if (lane == 0) ws.words[32] = stream_word(id, wb + 33);
  __syncwarp();
}

// offer with a refresh trigger instead of an inline serial recompute
__device__ __forceinline__ bool offer_trig(SetCtx& c, int64_t k0, double x, int64_t e) {
  PMH_ASSERT(k0 >= 0 && k0 < c.m);
  unsigned long long prev = slot_offer(&c.slots[k0], x, (unsigned long long)(e + c.eoff));
  if (prev == ~0ULL) return false;
  c.updates++;
  if (prev == EMPTY_H) {
    unsigned f = atomicAdd(c.filled, 1u) + 1u;
    return f == (unsigned)c.m;
  }
  return prev >= *(volatile unsigned long long*)c.hmax_bits;
}

__device__ __forceinline__ double warp_thr(const SetCtx& c) {
  return __shfl_sync(0xffffffffu, ctx_thr(c), 0);
}

// inclusive ordered fold: lane p returns fl(...fl(fl(x0 + d_0) + d_1)... + d_p)
// (lanes >= q: the fold of all q).  The increments go through shared memory
// and every lane runs the same sequential chain from broadcast loads, writing
// each prefix back in place (all lanes store the same value: one broadcast
// store); lane p then reads prefix p.  Per step: a DADD and a store, the
// loads vectorised.
__device__ __forceinline__ double ordered_fold(WarpScratch& ws, double x0, double d, int lane,
                                               uint32_t q) {
  ws.dbuf[lane] = d;
  __syncwarp();
  double acc = x0;
#pragma unroll 8
  for (uint32_t j = 0; j < q; j++) {
    acc = acc + ws.dbuf[j];
    ws.dbuf[j] = acc;
  }
  __syncwarp();
  const double mine = (uint32_t)lane < q ? ws.dbuf[lane] : acc;
  __syncwarp();
  return mine;
}

// ---- labels with replacement, power-of-two m: PMH1, PMH3, uw3 -------------

// F = FAM_PMH1 | FAM_PMH3 | FAM_UW3
template <int F>
__device__ int warp_el_static(SetCtx& c, const Tables& T, WarpScratch& ws, int lane,
                              int64_t e, uint64_t id, double winv) {
  const uint32_t kb = c.kbits;
  const uint32_t P = 53 + kb;
  uint64_t off = 0;     // absolute bit offset of the next point
  int64_t i = 1;        // next point index (1-based)
  double x = 0.0;       // PMH1 running sum
  for (;;) {
    const uint64_t wb = off >> 6;
    win_load(ws, id, wb, lane);
    const uint32_t rel0 = (uint32_t)(off - (wb << 6));
    uint32_t q = (WIN_BITS - rel0) / P;
    q = q > 32 ? 32 : q;
    const double thr = warp_thr(c);
    const int64_t pt = i + lane;
    const bool in = (uint32_t)lane < q;
    uint64_t u = 0;
    int32_t lab = 0;
    if (in) {
      const uint32_t ro = rel0 + (uint32_t)lane * P;
      u = win_bits(ws.words, ro, 53);
      lab = (int32_t)win_bits(ws.words, ro + 53, kb) + 1;
    }
    double xv = 0.0;
    uint32_t ncand = q;
    bool had_slow = false;
    if constexpr (F == FAM_PMH1) {
      const double d = in ? winv * exp1_from_bits(u) : 0.0;
      xv = ordered_fold(ws, x, d, lane, q);
    } else if constexpr (F == FAM_UW3) {
      const double U = (double)u * INV53;
      xv = pt == 1 ? U : ((double)pt - 1.0) + U;
    } else {  // PMH3: speculate on TruncExp's fast path
      double t = T.c3.c1 * ((double)u * INV53);
      const unsigned slow = __ballot_sync(0xffffffffu, in && !(t < 1.0));
      if (slow) {
        const int f = __ffs(slow) - 1;
        ncand = (uint32_t)f + 1;
        had_slow = true;
        if (lane == f) {
          Stream st;
          st.seek(id, off + (uint64_t)f * P + 53);
          bool fail = false;
          t = trunc_exp_slow(st, T.c3, &fail);
          lab = (int32_t)st.next_bits(kb) + 1;
          ws.next_off = st.pos(id);
          ws.flags = fail ? 2u : 0u;
        }
        __syncwarp();
        if (ws.flags & 2u) return EL_FAIL;
      }
      xv = pt == 1 ? winv * t : winv * ((double)pt - 1.0) + winv * t;
    }
    const bool cand = (uint32_t)lane < ncand;
    const bool valid = cand && xv <= thr;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const bool trig = valid ? offer_trig(c, lab - 1, xv, e) : false;
    if (__any_sync(0xffffffffu, trig)) hmax_refresh_warp(c, lane);
    const uint32_t nv = __popc(vm);
    // a retry attempt only counts points above the previous threshold
    const uint32_t nn = __popc(__ballot_sync(0xffffffffu, cand && !(xv <= c.tprev)));
    if (lane == 0) c.points += (c.tprev < 0.0 ? nv + (nv < ncand ? 1 : 0) : nn);
    if (nv < ncand) return EL_DONE;
    i += ncand;
    if (i > c.cap) return EL_FAIL;
    if constexpr (F == FAM_PMH1) x = __shfl_sync(0xffffffffu, xv, ncand - 1);
    if (had_slow) off = ws.next_off;
    else off += (uint64_t)ncand * P;
    __syncwarp();
  }
}

// Exact warp-parallel version of the ordered fold x_j = fl(x_{j-1} + d_j)
// (K:328, K:440): lane j returns x_j, x_{-1} = x0.  While the running sum
// stays in one binade [2^e, 2^(e+1)) every rounding is onto the same grid
// u = 2^(e-52), so with x_{j-1} on the grid
//     fl(x_{j-1} + d_j) = x_{j-1} + u * rint(d_j / u)
// except on an exact tie (d_j / u = k + 1/2, where IEEE rounds to the EVEN
// result, which depends on x_{j-1}).  The grid increments g_j = u rint(d_j/u)
// are multiples of u, so their prefix sums below 2^(e+1) are exact in
// floating point in any association: a Kogge-Stone scan reproduces the
// sequential chain bit for bit.  Lanes from the first tie or binade exit on
// are redone from the last exact value (one sequential add, then a new scan
// on the new binade); a batch normally needs one scan, rarely two.  x0 == 0
// (the element's first point): fl(0 + d_0) = d_0.
__device__ __forceinline__ double grid_fold(double x0, double d, int lane) {
  double base = x0;
  int start = 0;
  double res = 0.0;
  if (x0 == 0.0) {
    base = __shfl_sync(0xffffffffu, d, 0);
    res = base;
    start = 1;
  }
  while (start < 32) {
    const uint64_t bb = dbl_bits(base);
    const uint64_t ex = bb >> 52;            // base >= 0: the biased exponent
    if (ex < 53 || ex > 2044) {
      // zero / tiny / huge running sum (never seen in practice): sequential
      double acc = base;
      for (int j = start; j < 32; j++) {
        acc = acc + __shfl_sync(0xffffffffu, d, j);
        if (lane == j) res = acc;
      }
      return res;
    }
    const double inv_u = bits_dbl((2098ULL - ex) << 52);   // 2^(52 - e)
    const double u = bits_dbl((ex - 52ULL) << 52);          // 2^(e - 52)
    const double lim = bits_dbl((ex + 1ULL) << 52);         // 2^(e + 1)
    const bool mine = lane >= start;
    const double k = mine ? d * inv_u : 0.0;
    const double r = rint(k);
    const double fr = k - r;
    const bool tie = mine && (fr == 0.5 || fr == -0.5);
    double S = r * u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(0xffffffffu, S, o);
      if (lane >= o) S = S + t;
    }
    const double cand = base + S;
    const bool bad = mine && (tie || !(cand < lim));
    const unsigned bm = __ballot_sync(0xffffffffu, bad);
    const int f = bm ? __ffs(bm) - 1 : 32;
    if (mine && lane < f) res = cand;
    if (f == 32) break;
    const double prev = f == start ? base : __shfl_sync(0xffffffffu, cand, f - 1);
    const double xf = prev + __shfl_sync(0xffffffffu, d, f);   // the sequential step
    if (lane == f) res = xf;
    base = xf;
    start = f + 1;
  }
  return res;
}

#ifndef PMH_GRIDFOLD_FROM
#define PMH_GRIDFOLD_FROM 64   // grid_fold for batches starting beyond this point index
#endif

// Mode B for labels with replacement at label widths kb <= 16 (points of
// 53 + kb <= 69 bits): a window of 33 (kb <= 11) or 37 stream words always
// holds 32 whole points, so every batch is 32 points with static offsets;
// each lane's value bits come from one funnel shift of two adjacent words
// (the label from the same one when kb <= 11, else from a second), and
// ProbMinHash1's running sum folds with grid_fold after its first batches.
// Same results and counters as warp_el_static.
template <int F>
__device__ int warp_el_static2(SetCtx& c, const Tables& T, WarpScratch& ws, int lane,
                               int64_t e, uint64_t id, double winv) {
  const uint32_t kb = c.kbits;
  const uint32_t P = 53 + kb;
  const uint64_t kmask = (1ULL << kb) - 1ULL;
  // window words beyond the first 32: 32 points of P <= 64 bits need 33; of
  // P <= 69 bits (kb <= 16) 37 (63 + 32 P bits, plus the label funnel's guard)
  const int nx = kb <= 11 ? 1 : 5;
  uint64_t off = 0;     // absolute bit offset of the next point
  int64_t i = 1;        // next point index (1-based)
  double x = 0.0;       // PMH1 running sum
  for (;;) {
    const uint64_t wb = off >> 6;
    ws.words[lane] = stream_word(id, wb + 1 + (uint64_t)lane);
    if (lane < nx) ws.words[32 + lane] = stream_word(id, wb + 33 + (uint64_t)lane);
    __syncwarp();
    const uint32_t rel0 = (uint32_t)(off & 63);
    const double thr = warp_thr(c);
    const int64_t pt = i + lane;
    const uint32_t ro = rel0 + (uint32_t)lane * P;
    const uint32_t wi = ro >> 6, sh = ro & 63;
    const uint64_t w0 = ws.words[wi];
    const uint64_t v = sh ? (w0 >> sh) | (ws.words[wi + 1] << (64 - sh)) : w0;
    const uint64_t u = v & ((1ULL << 53) - 1ULL);
    int32_t lab;
    if (kb <= 11) {   // the label is in the same 64 bits
      lab = (int32_t)((v >> 53) & kmask) + 1;
    } else {
      const uint32_t rl = ro + 53, wl = rl >> 6, sl = rl & 63;
      const uint64_t l0 = ws.words[wl];
      lab = (int32_t)(((sl ? (l0 >> sl) | (ws.words[wl + 1] << (64 - sl)) : l0)) & kmask) + 1;
    }
    double xv = 0.0;
    uint32_t ncand = 32;
    bool had_slow = false;
    if constexpr (F == FAM_PMH1) {
      // the first batches cross binades at almost every doubling of x
      // (many grid_fold rounds): the sequential fold there
      const double d = winv * exp1_from_bits(u);
      xv = i <= PMH_GRIDFOLD_FROM ? ordered_fold(ws, x, d, lane, 32) : grid_fold(x, d, lane);
    } else if constexpr (F == FAM_UW3) {
      const double U = (double)u * INV53;
      xv = pt == 1 ? U : ((double)pt - 1.0) + U;
    } else {  // PMH3: speculate on TruncExp's fast path
      double t = T.c3.c1 * ((double)u * INV53);
      const unsigned slow = __ballot_sync(0xffffffffu, !(t < 1.0));
      if (slow) {
        const int f = __ffs(slow) - 1;
        ncand = (uint32_t)f + 1;
        had_slow = true;
        if (lane == f) {
          Stream st;
          st.seek(id, off + (uint64_t)f * P + 53);
          bool fail = false;
          t = trunc_exp_slow(st, T.c3, &fail);
          lab = (int32_t)st.next_bits(kb) + 1;
          ws.next_off = st.pos(id);
          ws.flags = fail ? 2u : 0u;
        }
        __syncwarp();
        if (ws.flags & 2u) return EL_FAIL;
      }
      xv = pt == 1 ? winv * t : winv * ((double)pt - 1.0) + winv * t;
    }
    const bool cand = (uint32_t)lane < ncand;
    const bool valid = cand && xv <= thr;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const bool trig = valid ? offer_trig(c, lab - 1, xv, e) : false;
    if (__any_sync(0xffffffffu, trig)) hmax_refresh_warp(c, lane);
    const uint32_t nv = __popc(vm);
    // a retry attempt only counts points above the previous threshold
    const uint32_t nn = __popc(__ballot_sync(0xffffffffu, cand && !(xv <= c.tprev)));
    if (lane == 0) c.points += (c.tprev < 0.0 ? nv + (nv < ncand ? 1 : 0) : nn);
    if (nv < ncand) return EL_DONE;
    i += ncand;
    if (i > c.cap) return EL_FAIL;
    if constexpr (F == FAM_PMH1) x = __shfl_sync(0xffffffffu, xv, ncand - 1);
    if (had_slow) off = ws.next_off;
    else off += (uint64_t)ncand * P;
    __syncwarp();
  }
}

// ---- labels without replacement: PMH2, PMH4, uw4 -------------------------

// Lane 0 parses up to 32 points of the window: the bit offset of each point's
// value draw (53 bits) and its Fisher-Yates index r = uniform_int(m-pt+1)
// (kbits-wide rejection rounds, K:97-117, K:225), assuming TruncExp's fast
// path.  Only integer work is on this serial chain; the fast-path test, the
// Fisher-Yates map steps and all floating point run afterwards.
__device__ __forceinline__ uint32_t bits_for_fast(int64_t R) {  // == bits_for(R), R >= 2
  return 64u - (uint32_t)__clzll((long long)(R - 1));
}

__device__ void parse_fy_cursor(const SetCtx& c, WarpScratch& ws, uint64_t id, uint64_t off,
                                int64_t i0) {
  const int64_t m = c.m;
  const uint64_t wb = off >> 6;
  uint32_t cur = (uint32_t)(off - (wb << 6));
  uint32_t q = 0;
  uint32_t flags = 0;
  uint64_t next_off = 0;
  while (q < 32) {
    const int64_t pt = i0 + q;
    if (pt > m || cur + 53 > WIN_BITS) break;
    const uint32_t eo = cur;
    uint32_t c2 = cur + 53;
    const int64_t R = m - pt + 1;
    int64_t r = 0;
    if (R > 1) {
      const uint32_t kb = bits_for_fast(R);
      int rounds = 0;
      bool fits = true;
      for (;;) {
        if (c2 + kb > WIN_BITS) { fits = false; break; }
        const uint64_t v = win_bits(ws.words, c2, kb);
        c2 += kb;
        if (v < (uint64_t)R) { r = (int64_t)v; break; }
        if (++rounds > g_reject_cap) { flags = 2u; break; }
      }
      if (flags) break;
      if (!fits) {
        if (q > 0) break;
        // the first point of the batch does not fit the window: finish it
        // with a sequential cursor and end the batch after it
        Stream st;
        st.seek(id, (wb << 6) + eo + 53);
        r = uniform_int_masked(st, (uint64_t)R, kb);
        if (r < 0) { flags = 2u; break; }
        ws.eoff[q] = eo;
        ws.lab[q] = (int32_t)r;
        q++;
        flags = 1u;
        next_off = st.pos(id);
        break;
      }
    }
    ws.eoff[q] = eo;
    ws.lab[q] = (int32_t)r;       // the FY index for now; the label after fy_steps
    q++;
    cur = c2;
  }
  ws.q = q;
  ws.flags = flags;
  ws.next_off = (flags & 1u) ? next_off : (wb << 6) + cur;
}

// Bit t (t0 <= t < t1) set iff label round t (the kb-bit field at pos + kb t)
// is accepted (< R).  Rounds are contiguous fields, so one 64-bit funnel load
// serves fpw = 64 / kb of them.
constexpr uint32_t ACC_ROUNDS0 = 8;
__device__ __forceinline__ uint32_t accept_mask(const uint64_t* w, uint32_t pos, uint32_t kb,
                                                uint64_t R, uint32_t t0, uint32_t t1,
                                                uint32_t fpw) {
  const uint64_t mask = (1ULL << kb) - 1ULL;
  uint32_t acc = 0;
  for (uint32_t t = t0; t < t1;) {
    const uint32_t p = pos + kb * t, i = p >> 6, sh = p & 63;
    const uint64_t win = sh ? (w[i] >> sh) | (w[i + 1] << (64 - sh)) : w[i];
    const uint32_t te = t + fpw < t1 ? t + fpw : t1;
    uint32_t fo = 0;
    for (; t < te; t++, fo += kb) acc |= (((win >> fo) & mask) < R ? 1u : 0u) << t;
  }
  return acc;
}

// accept_mask for a compile-time label width and round range: the field
// shifts, masks and bit positions become immediates and the compares 32-bit
// (fields and R < 2^KB <= 2^32).  Rounds [T0, T1) start at window loads
// aligned to T0, so the fields of one load are u = 0 .. FPW-1.
template <uint32_t KB, uint32_t T0, uint32_t T1>
__device__ __forceinline__ uint32_t accept_mask_k(const uint64_t* w, uint32_t pos, uint32_t R) {
  constexpr uint32_t FPW = 64u / KB;
  constexpr uint64_t MASK = (1ULL << KB) - 1ULL;
  uint32_t acc = 0;
#pragma unroll
  for (uint32_t t = T0; t < T1; t += FPW) {
    const uint32_t p = pos + KB * t, i = p >> 6, sh = p & 63;
    const uint64_t win = sh ? (w[i] >> sh) | (w[i + 1] << (64 - sh)) : w[i];
#pragma unroll
    for (uint32_t u = 0; u < FPW; u++)
      if (t + u < T1) acc |= ((uint32_t)((win >> (KB * u)) & MASK) < R ? 1u : 0u) << (t + u);
  }
  return acc;
}

// the label widths of the configured m (64, 256, 1024, 4096: kb = 6, 8, 10,
// 12 for the first half of the ranges) specialised, the rest generic
template <uint32_t T0, uint32_t T1>
__device__ __forceinline__ uint32_t accept_mask_sel(const uint64_t* w, uint32_t pos, uint32_t kb,
                                                    uint64_t R, uint32_t fpw) {
// PMH_ACC_SPEC 2: kb = 6/8/10/12 specialised; 1: 10/12 only; 0: none.
// Measured (configs[1] PMH2/PMH4 ms, configs[3] PMH2/PMH4, configs[4]):
// 2: 7.81/5.87, 108.5/83.4, 24.4;  1: 8.06/6.24, 112.6/83.9, 25.8;
// 0: 7.99/6.22, 93.8/84.2, 26.4 -- the warp-per-set kernel of configs[3] is
// instruction-cache bound, so results follow code layout more than op counts
#ifndef PMH_ACC_SPEC
#define PMH_ACC_SPEC 2
#endif
  switch (kb) {
#if PMH_ACC_SPEC >= 2
    case 6: return accept_mask_k<6, T0, T1>(w, pos, (uint32_t)R);
    case 8: return accept_mask_k<8, T0, T1>(w, pos, (uint32_t)R);
#endif
#if PMH_ACC_SPEC >= 1
    case 10: return accept_mask_k<10, T0, T1>(w, pos, (uint32_t)R);
    case 12: return accept_mask_k<12, T0, T1>(w, pos, (uint32_t)R);
#endif
    default: return accept_mask(w, pos, kb, R, T0, T1, fpw);
  }
}

// Warp-parallel version of parse_fy_cursor.  For a run of points whose
// Fisher-Yates range R = m - pt + 1 shares the label width kb, point k starts
// at base_k + kb * Y_k, where base_k = rel0 + k (53 + kb) and Y_k is the number
// of REJECTED label rounds of points 0..k-1.  Lane k records in a 24-bit mask
// which of its candidate label draws (base_k + 53 + kb t, t = 0..23) would be
// accepted (< R_k); the recurrence Y_{k+1} = Y_k + ctz(acc_k >> Y_k) then
// fixes every offset (K:97-117 rejection semantics exactly).  Falls back to the
// serial parse when the run is empty or a point rejects beyond the window.
__device__ void parse_fy_parallel(const SetCtx& c, WarpScratch& ws, uint64_t id, uint64_t off,
                                  int64_t i0, int lane) {
  const int64_t m = c.m;
  const uint64_t wb = off >> 6;
  const uint32_t rel0 = (uint32_t)(off - (wb << 6));
  const int64_t R0 = m - i0 + 1;
  if (R0 <= 1) {  // the last point (pt = m) draws no label bits
    if (lane == 0) {
      ws.eoff[0] = rel0;
      ws.lab[0] = 0;
      ws.q = 1;
      ws.flags = 0;
      ws.next_off = off + 53;
    }
    __syncwarp();
    return;
  }
  const uint32_t kb = bits_for_fast(R0);
  const int64_t pt = i0 + lane;
  const int64_t R = m - pt + 1;
  // lanes of the same-width run (R > 1 and bits_for(R) == kb)
  const bool inrun = R > 1 && bits_for_fast(R) == kb;
  const unsigned runmask = __ballot_sync(0xffffffffu, inrun);
  const uint32_t qmax = runmask == 0xffffffffu ? 32u : (uint32_t)(__ffs(~runmask) - 1);
  const uint32_t base = rel0 + (uint32_t)lane * (53u + kb);
  // rounds [0, 8) first: rejections are rare for most ranges, so the later
  // rounds are only decoded when the scan runs past them
  const uint32_t fpw = 64u / kb;   // label fields per 64-bit window load
  const bool mine = (uint32_t)lane < qmax;
  uint32_t acc = mine ? accept_mask_sel<0u, ACC_ROUNDS0>(ws.words, base + 53u, kb, (uint64_t)R, fpw)
                      : 0u;
  bool full = false;
  // Y_{k+1} = first accepted round >= Y_k of point k.  Y only moves at points
  // whose round Y is rejected, so jump between those with a ballot: one
  // iteration per rejection instead of one per point.
  uint32_t Y = 0, myY = 0, mye = 0, q = qmax, start = 0;
  for (;;) {
    const bool rej = (uint32_t)lane >= start && mine && !((acc >> Y) & 1u);
    const unsigned bad = __ballot_sync(0xffffffffu, rej);
    const uint32_t j = bad ? (uint32_t)(__ffs(bad) - 1) : qmax;
    if ((uint32_t)lane >= start && (uint32_t)lane < j) { myY = Y; mye = 0; }
    if (j >= qmax) break;
    const uint32_t am = __shfl_sync(0xffffffffu, acc, (int)j) >> Y;
    if (am == 0 && !full) {  // decode the remaining rounds and retry this point
      if (mine) acc |= accept_mask_sel<ACC_ROUNDS0, 24u>(ws.words, base + 53u, kb, (uint64_t)R, fpw);
      full = true;
      continue;
    }
    if (am == 0) { q = j; break; }
    const uint32_t e = (uint32_t)(__ffs(am) - 1);
    if ((uint32_t)lane == j) { myY = Y; mye = e; }
    Y += e;
    start = j + 1;
  }
  if (q == 0) {  // the first point's label needs more rounds than the window: serial
    if (lane == 0) parse_fy_cursor(c, ws, id, off, i0);
    __syncwarp();
    return;
  }
  if ((uint32_t)lane < q) {
    ws.eoff[lane] = base + kb * myY;
    ws.lab[lane] = (int32_t)win_bits(ws.words, base + 53u + kb * (myY + mye), kb);
  }
  if (lane == (int)q - 1) {
    ws.q = q;
    ws.flags = 0;
    ws.next_off = (wb << 6) + base + 53u + kb * (myY + mye + 1u);
  }
  __syncwarp();
}

// The common case of a Fisher-Yates batch: no label draw of the batch's run
// is rejected, so every point sits at its static offset rel0 + k (53 + kb).
// Loads the window's first 37 words (enough for 32 static points of <= 69
// bits), checks each lane's first label field against its range R (K:97-110)
// and, if all accept, writes the parse result.  Returns false -- the caller
// then loads the rest of the 64-word window and runs parse_fy_parallel -- on
// any rejection, for the last point (R = 1) or for kb > 16.  (At m = 4096
// the first ~40 ranges reject with probability < 1%.)
__device__ __forceinline__ bool parse_fy_fast(const SetCtx& c, WarpScratch& ws, uint64_t id,
                                              uint64_t off, int64_t i0, int lane) {
  const int64_t m = c.m;
  const uint64_t wb = off >> 6;
  ws.words[lane] = stream_word(id, wb + 1 + (uint64_t)lane);
  if (lane < 5) ws.words[32 + lane] = stream_word(id, wb + 33 + (uint64_t)lane);
  __syncwarp();
  const int64_t R0 = m - i0 + 1;
  if (R0 <= 1) return false;
  const uint32_t kb = bits_for_fast(R0);
  if (kb > 16) return false;
  const uint32_t P = 53u + kb;
  const uint32_t rel0 = (uint32_t)(off - (wb << 6));
  const int64_t R = m - (i0 + lane) + 1;
  const bool inrun = R > 1 && bits_for_fast(R) == kb;
  const unsigned runmask = __ballot_sync(0xffffffffu, inrun);
  const uint32_t qmax = runmask == 0xffffffffu ? 32u : (uint32_t)(__ffs(~runmask) - 1);
  const uint32_t ro = rel0 + (uint32_t)lane * P;
  const bool mine = (uint32_t)lane < qmax;
  uint32_t field = 0;
  if (mine) field = (uint32_t)win_bits(ws.words, ro + 53u, kb);
  if (__ballot_sync(0xffffffffu, mine && !((int64_t)field < R))) return false;
  if (mine) {
    ws.eoff[lane] = ro;
    ws.lab[lane] = (int32_t)field;   // the FY index; the label after fy_steps
  }
  if (lane == 0) {
    ws.q = qmax;
    ws.flags = 0;
    ws.next_off = (wb << 6) + rel0 + (uint64_t)qmax * P;
  }
  __syncwarp();
  return true;
}

// Warp-parallel lazy Fisher-Yates for the q points of a batch (lane k =
// point pt_k = i0 + k with index j_k = pt_k + r_k, K:222-235).  Sequentially:
//   out_k = P[j_k];  P[j_k] = P[pt_k]
// so with v_k = P_{k-1}[pt_k]: v_k is the v of the latest earlier lane whose
// target j equals pt_k (else the map before the batch), out_k is the v of the
// latest earlier lane with the same target j_k (else the map before the batch),
// and each distinct target finally holds the v of its last writer.  Earlier
// writers come from __match_any_sync; the (short) v chains resolve by shuffle
// pointer chasing.
template <class FYMap>
__device__ __forceinline__ void fy_steps_parallel(WarpScratch& ws, FYMap fy, int64_t i0,
                                                  uint32_t q, int lane) {
  const bool valid = (uint32_t)lane < q;
  const int32_t pt = (int32_t)(i0 + lane);
  const int32_t j = valid ? pt + ws.lab[lane] : -1 - lane;
  ws.gm[lane] = 0u;
  __syncwarp();
  const unsigned vmask = __ballot_sync(0xffffffffu, valid);
  unsigned grp = 0u;
  if (valid) grp = __match_any_sync(vmask, j);
  const int last = valid ? 31 - __clz((int)grp) : -1;   // last writer of target j
  if (valid && lane == last && j - (int32_t)i0 < 32) ws.gm[j - (int32_t)i0] = grp;
  const int32_t pb_pt = valid ? fy.get(pt) : 0;         // map before the batch
  const int32_t pb_j = valid ? fy.get(j) : 0;
  __syncwarp();
  const unsigned below = (1u << lane) - 1u;
  const unsigned pm = valid ? (ws.gm[lane] & below) : 0u;
  const int prevp = pm ? 31 - __clz((int)pm) : lane;
  const unsigned jm = grp & below;
  const int prevj = jm ? 31 - __clz((int)jm) : lane;
  int32_t v = pb_pt;
  bool pend = valid && prevp != lane;
  while (__any_sync(0xffffffffu, pend)) {
    const int32_t vs = __shfl_sync(0xffffffffu, v, prevp);
    const bool ps = __shfl_sync(0xffffffffu, pend, prevp);
    if (pend && !ps) { v = vs; pend = false; }
  }
  const int32_t vj = __shfl_sync(0xffffffffu, v, prevj);
  __syncwarp();
  if (valid && lane == last) fy.set(j, v);
  if (valid) ws.lab[lane] = prevj != lane ? vj : pb_j;
  __syncwarp();
}

template <int F, bool FY16>
__device__ int warp_el_fy(SetCtx& c, const Tables& T, WarpScratch& ws, uint32_t* fy, int lane,
                          int64_t e, uint64_t id, double winv) {
  const int64_t m = c.m;
  uint32_t ep = ws.epoch + 1;
  if (ws.fy_dirty) {   // the lanes' hash maps were here (CTA kernels only): start over
    fy_clear_region(fy, fy_region_bytes(m, FY16), lane);
    ep = 1;
  } else if (ep >= (FY16 ? FY_EPOCHS16 : FY_EPOCHS32)) {  // epoch wrap: clear the map
    fy_clear<FY16>(fy, m, lane);
    ep = 1;
  }
  __syncwarp();
  if (lane == 0) { ws.epoch = ep; ws.fy_dirty = 0u; }
  EpochFY<FY16> efy{fy, ep};
  uint64_t off = 0;
  int64_t i = 1;
  double x = 0.0;
  for (;;) {
    const uint64_t wb = off >> 6;
    if (!parse_fy_fast(c, ws, id, off, i, lane)) {
      // a rejection in the batch: the rest of the 64-word window, full parse
      if (lane < 28) ws.words[37 + lane] = stream_word(id, wb + 38 + (uint64_t)lane);
      __syncwarp();
      parse_fy_parallel(c, ws, id, off, i, lane);
    }
    if (ws.flags & 2u) return EL_FAIL;
    uint32_t q = ws.q;
    const int64_t pt = i + lane;
    const bool in0 = (uint32_t)lane < q;
    // value draw of this lane's point (fast path assumed by the parse)
    const uint64_t u = in0 ? win_bits(ws.words, ws.eoff[lane], 53) : 0;
    double tv = 0.0;
    if constexpr (F == FAM_PMH4) {
      bool slow = false;
      if (in0 && pt < m) {
        tv = __ldg(&T.c4[pt].c1) * ((double)u * INV53);
        slow = !(tv < 1.0);
      }
      const unsigned sm = __ballot_sync(0xffffffffu, slow);
      if (sm) {
        const int f = __ffs(sm) - 1;
        q = (uint32_t)f + 1;   // points after a slow draw have unknown offsets
        if (lane == f) {
          Stream st;
          st.seek(id, (wb << 6) + ws.eoff[f] + 53);
          bool fail = false;
          tv = trunc_exp_slow(st, T.c4[pt], &fail);
          const int64_t R = m - pt + 1;
          const int64_t r = uniform_int_masked(st, (uint64_t)R, bits_for_fast(R));
          ws.lab[f] = (int32_t)r;
          ws.next_off = st.pos(id);
          if (fail || r < 0) ws.flags = 2u;
        }
        __syncwarp();
        if (ws.flags & 2u) return EL_FAIL;
      }
    } else if constexpr (F == FAM_UW4) {
      tv = (double)u * INV53;  // the uniform itself
    }
    fy_steps_parallel(ws, efy, i, q, lane);
    const double thr = warp_thr(c);
    const bool in = (uint32_t)lane < q;
    double xv = 0.0;
    if constexpr (F == FAM_PMH2) {
      double d = 0.0;
      if (in) {
        const double E = exp1_from_bits(u);
        d = pt == 1 ? winv * E : (winv * __ldg(&T.beta[pt])) * E;
      }
      xv = ordered_fold(ws, x, d, lane, q);
    } else if constexpr (F == FAM_PMH4) {
      if (in) {
        if (pt == 1) {
          xv = winv * tv;
        } else if (pt < m) {
          xv = winv * (__ldg(&T.gam[pt - 1]) + __ldg(&T.dgam[pt]) * tv);
        } else {
          xv = winv * (__ldg(&T.gam[m - 1]) + T.delta * exp1_from_bits(u));
        }
      }
    } else {  // uw4
      if (in) xv = pt == 1 ? tv : ((double)pt - 1.0) + tv;
    }
    const bool valid = in && xv <= thr;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    const bool trig = valid ? offer_trig(c, ws.lab[lane] - 1, xv, e) : false;
    if (__any_sync(0xffffffffu, trig)) hmax_refresh_warp(c, lane);
    const uint32_t nv = __popc(vm);
    const uint32_t nn = __popc(__ballot_sync(0xffffffffu, in && !(xv <= c.tprev)));
    if (lane == 0) c.points += (c.tprev < 0.0 ? nv + (nv < q ? 1 : 0) : nn);
    if (nv < q) return EL_DONE;
    i += q;
    if (i > m) return EL_DONE;
    if constexpr (F == FAM_PMH2) x = __shfl_sync(0xffffffffu, xv, q - 1);
    off = ws.next_off;
    __syncwarp();
  }
}

template <int F, bool FY16>
__device__ __forceinline__ int warp_element(SetCtx& c, const Tables& T, WarpScratch& ws,
                                            uint32_t* fy, int lane, int64_t e, uint64_t id,
                                            double winv) {
  if constexpr (F == FAM_PMH1 || F == FAM_PMH3 || F == FAM_UW3) {
#ifndef PMH_STATIC2
#define PMH_STATIC2 1
#endif
    if (PMH_STATIC2 && c.kbits <= 16) return warp_el_static2<F>(c, T, ws, lane, e, id, winv);
    return warp_el_static<F>(c, T, ws, lane, e, id, winv);
  }
  else
    return warp_el_fy<F, FY16>(c, T, ws, fy, lane, e, id, winv);
}

}  // namespace pmh
