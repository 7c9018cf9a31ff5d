// pmh_split.cuh -- splitting the largest sets of a batch across CTAs.
//
// Every sketch kernel runs one CTA per set, which caps one set at one SM: a
// single 10^6-element set (P-MinHash, m = 1024) or 10^7-element set
// (ProbMinHash) takes tens to hundreds of ms where the whole GPU would take
// one.  Sets larger than both `split_n` and the batch's fair share per CTA
// slot (total cost / CTA slots, rounded down to a power of two) are cut into
// parts of <= split_n elements.  A part's CTA computes the exact minima of
// its element range in shared memory -- its own threshold guess, verified, so
// any range is exact-safe -- and merges them into the set's global slot table
// with 128-bit CAS on (h, in-set index): lexicographic, hence
// order-independent.  A final
// pass writes the ids.  Which sets are split is decided on the device (no
// host sync): the LPT order is by bit length of (n + c), so the sets with
// n + c >= 2^k form an order prefix, found by binary search.
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

struct SplitArgs {
  const int64_t* offsets;
  const int32_t* order;
  int64_t nsets;
  int64_t c_off;          // the order's cost offset (0 for P-MinHash, 7m otherwise)
  int64_t split_n;        // part size; only sets with n >= split_n are split
  int64_t split_cap;      // at most this many sets are split (gtab rows)
  int64_t m;
  Slot* gtab;             // [split_cap, m]
  int64_t* part_base;     // [split_cap + 1]
  long long* info;        // [0] nsplit, [1] total parts, [2] work counter
  int64_t* stats;         // [nsets, 3] or nullptr: zeroed for the split sets
};

// Lexicographic (h, idx) minimum into a global slot.
__device__ __forceinline__ void slot_offer_global(Slot* p, unsigned long long h,
                                                  unsigned long long idx) {
  unsigned long long ch, ci;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(ch), "=l"(ci) : "l"(p)
               : "memory");
  while (h < ch || (h == ch && idx < ci)) {
    unsigned long long oh, oi;
    asm volatile(
        "{\n\t.reg .b128 c, n, d;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 n, {%4, %5};\n\t"
        "atom.global.cas.b128 d, [%6], c, n;\n\t"
        "mov.b128 {%0, %1}, d;\n\t}"
        : "=l"(oh), "=l"(oi)
        : "l"(ch), "l"(ci), "l"(h), "l"(idx), "l"(p)
        : "memory");
    if (oh == ch && oi == ci) return;
    ch = oh;
    ci = oi;
  }
}

#ifndef PMH_SPLIT_SMALL_FAIR
#define PMH_SPLIT_SMALL_FAIR 65536
#endif
// single CTA: which sets are split, the parts per set, their prefix
__global__ void split_prep_kernel(SplitArgs a, long long cta_slots) {
  __shared__ long long s_run;
  __shared__ long long s_warp[32];
  __shared__ long long s_nsplit;
  if (threadIdx.x == 0) {
    // threshold: the largest power of two not above the fair share (total
    // cost / CTA slots), but at least the smallest power of two >= one part
    const long long total = (a.offsets[a.nsets] - a.offsets[0]) + a.c_off * a.nsets;
    long long fair = total / (cta_slots > 0 ? cta_slots : 1);
    // a small batch (one rank's shard): a quarter of the fair share, so the
    // LPT tail is a few short parts instead of one unsplit set near the
    // fair share (large batches keep whole sets: a part prunes with its own
    // minima only, so splitting costs work there)
    if (fair < PMH_SPLIT_SMALL_FAIR) fair /= 4;
    long long floor_p2 = 1;
    while (floor_p2 < a.split_n + a.c_off) floor_p2 <<= 1;
    long long p2 = floor_p2;
    while (p2 * 2 <= fair) p2 <<= 1;
    long long lo = 0, hi = a.nsets;                 // first order index with n + c < p2
    while (lo < hi) {
      const long long mid = (lo + hi) / 2;
      const int64_t sm = a.order[mid];
      if (a.offsets[sm + 1] - a.offsets[sm] + a.c_off >= p2) lo = mid + 1; else hi = mid;
    }
    s_nsplit = lo < a.split_cap ? lo : a.split_cap;
    s_run = 0;
  }
  __syncthreads();
  const long long nsplit = s_nsplit;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long i0 = 0; i0 < nsplit; i0 += blockDim.x) {
    const long long i = i0 + threadIdx.x;
    long long parts = 0;
    if (i < nsplit) {
      const int64_t s = a.order[i];
      const int64_t n = a.offsets[s + 1] - a.offsets[s];
      parts = (n + a.split_n - 1) / a.split_n;
    }
    long long x = parts;                            // inclusive block scan
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    long long before = 0, chunk_total = 0;
    for (int k = 0; k < nw; k++) {
      if (k < wid) before += s_warp[k];
      chunk_total += s_warp[k];
    }
    if (i < nsplit) a.part_base[i] = s_run + before + x - parts;
    __syncthreads();
    if (threadIdx.x == 0) s_run += chunk_total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    a.part_base[nsplit] = s_run;
    a.info[0] = nsplit;
    a.info[1] = s_run;
    a.info[2] = 0;
  }
}

__global__ void split_init_kernel(SplitArgs a) {
  const int64_t nsplit = a.info[0];
  const int64_t total = nsplit * a.m;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    a.gtab[q].h = EMPTY_H;
    a.gtab[q].idx = EMPTY_IDX;
  }
  if (a.stats)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nsplit;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t s = a.order[i];
      a.stats[s * 3 + 0] = 0;
      a.stats[s * 3 + 1] = 0;
      a.stats[s * 3 + 2] = 0;
    }
}

// next part for a persistent CTA (all threads; -1 when none is left):
// (order index i, element range [e0, e1) within the set)
struct SplitPart {
  int64_t i, s, off, n, e0, e1;
};
__device__ __forceinline__ bool split_next_part(const SplitArgs& a, long long* s_t, SplitPart* p) {
  if (threadIdx.x == 0) *s_t = (long long)atomicAdd((unsigned long long*)&a.info[2], 1ULL);
  __syncthreads();
  const long long t = *s_t;
  __syncthreads();
  if (t >= a.info[1]) return false;
  int64_t lo = 0, hi = a.info[0] - 1;               // last i with part_base[i] <= t
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    if (a.part_base[mid] <= t) lo = mid; else hi = mid - 1;
  }
  p->i = lo;
  p->s = a.order[lo];
  p->off = a.offsets[p->s];
  p->n = a.offsets[p->s + 1] - p->off;
  const int64_t parts = a.part_base[lo + 1] - a.part_base[lo];
  const int64_t k = t - a.part_base[lo];
  p->e0 = p->n * k / parts;
  p->e1 = p->n * (k + 1) / parts;
  PMH_ASSERT(lo < a.info[0] && lo < a.split_cap && k < parts && p->e1 <= p->n && p->e0 < p->e1);
  return true;
}

// ids of the split sets from their merged tables
__global__ void split_finalize_kernel(SplitArgs a, const uint64_t* __restrict__ ids,
                                      uint64_t* __restrict__ sig) {
  const int64_t nsplit = a.info[0];
  const int64_t total = nsplit * a.m;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / a.m, k = q - i * a.m;
    const int64_t s = a.order[i];
    const int64_t off = a.offsets[s];
    const int64_t n = a.offsets[s + 1] - off;
    const unsigned long long bi = a.gtab[q].idx;
    sig[s * a.m + k] = bi < (unsigned long long)n ? ids[off + bi] : 0ULL;
  }
}

}  // namespace pmh
