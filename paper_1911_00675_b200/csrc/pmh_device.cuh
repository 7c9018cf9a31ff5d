// pmh_device.cuh -- device primitives of the ProbMinHash signature engine.
//
// Bit-level contract (reference /root/reference/pkg/src/probminhash/_kernels.py,
// cited as K:<line>):
//   * element stream = splitmix64 seeded with the element id (K:47-60, K:291):
//     word j (j >= 1) = mix64(id + j * GOLDEN mod 2^64);
//   * bits are consumed as one LSB-first bit stream over those words
//     (K:63-78), so a draw of k bits at absolute bit offset b is
//     (words >> b) & (2^k - 1) -- random access by offset;
//   * U = bits53 * 2^-53 (K:81-83); E = -log1p(-U) with glibc log1p
//     (K:120-122, pmh_math.cuh); TruncExp = Alg. 7 (K:125-151);
//   * labels with replacement = 1 + kbits-wide rejection draws (K:97-110);
//     labels without replacement = lazy Fisher-Yates (K:222-235).
// All arithmetic is one IEEE double rounding per operation in the
// reference's order; this file is compiled with -fmad=false.
#pragma once
#include <stdint.h>

#include "pmh_math.cuh"

namespace pmh {

// Bounds checks of a debug build (-DPMH_DEBUG_BOUNDS): trap on a violated
// index invariant so a test run fails loudly instead of corrupting memory.
#ifdef PMH_DEBUG_BOUNDS
#define PMH_ASSERT(c) do { if (!(c)) __trap(); } while (0)
#else
#define PMH_ASSERT(c) do { } while (0)
#endif


constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;  // K:20
constexpr uint64_t MIX1 = 0xBF58476D1CE4E5B9ULL;    // K:21
constexpr uint64_t MIX2 = 0x94D049BB133111EBULL;    // K:22
constexpr double INV53 = 1.1102230246251565e-16;    // K:30
constexpr uint64_t OPH_SALT = 0xA24BAED4963EE407ULL;  // K:33
constexpr int REJECT_CAP = 4096;                    // K:37

// The loop caps the device code enforces: the reference's REJECT_CAP (K:37)
// and coupon cap (K:279-281).  Always these values, except that a TEST may
// lower them through the environment (PMH_TEST_REJECT_CAP /
// PMH_TEST_COUPON_CAP, read once per device by the host, pmh_capi.cu) to
// drive the RandomnessFailureError path on the device.
__constant__ int g_reject_cap = REJECT_CAP;
__constant__ long long g_coupon_cap_override = 0;   // > 0: replaces the K:279-281 cap

// algorithm ids = K:866-881
enum Algo : int {
  ALG_PMINHASH = 0, ALG_PMH1 = 1, ALG_PMH1A = 2, ALG_PMH2 = 3, ALG_PMH3 = 4,
  ALG_PMH3A = 5, ALG_PMH4 = 6, ALG_MINHASH = 10, ALG_SUPERMINHASH = 11,
  ALG_OPH = 12, ALG_UW1 = 13, ALG_UW1A = 14, ALG_UW2 = 15, ALG_UW3 = 16,
  ALG_UW3A = 17, ALG_UW4 = 18
};

// device error flags (per call, OR-ed)
constexpr int ERRF_RANDOMNESS = 1;
constexpr int ERRF_CAPACITY = 2;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // K:40-44
  uint64_t z = (x ^ (x >> 30)) * MIX1;
  z = (z ^ (z >> 27)) * MIX2;
  return z ^ (z >> 31);
}

// mix64 without its final xorshift (out = z ^ (z >> 31)); bits 33..63 of z
// and of mix64's output agree (the P-MinHash body tests those on z directly)
__device__ __forceinline__ uint64_t mix64_z(uint64_t x) {
  uint64_t z = (x ^ (x >> 30)) * MIX1;
  return (z ^ (z >> 27)) * MIX2;
}


// word j (1-based) of the stream seeded with `seed`
__device__ __forceinline__ uint64_t stream_word(uint64_t seed, uint64_t j) {
  return mix64(seed + j * GOLDEN);
}

// Sequential bit cursor, the reference's 4-word state (K:47-78).
struct Stream {
  uint64_t s;    // generator state (id + words * GOLDEN)
  uint64_t buf;  // buffered bits, LSB first
  uint32_t nb;   // number of buffered bits
  __device__ __forceinline__ void seed(uint64_t id) { s = id; buf = 0; nb = 0; }
  // position the cursor at absolute bit offset `off` of the stream of `id`
  __device__ __forceinline__ void seek(uint64_t id, uint64_t off) {
    s = id + (off >> 6) * GOLDEN;
    const uint32_t r = (uint32_t)(off & 63);
    if (r) { const uint64_t w = next_u64(); buf = w >> r; nb = 64 - r; }
    else { buf = 0; nb = 0; }
  }
  // absolute bit offset of the cursor (words generated * 64 - buffered)
  __device__ __forceinline__ uint64_t pos(uint64_t id) const {
    return ((s - id) * 0xF1DE83E19937733DULL) * 64ULL - nb;  // (s-id)/GOLDEN: inverse of GOLDEN mod 2^64
  }
  __device__ __forceinline__ uint64_t next_u64() { s += GOLDEN; return mix64(s); }
  // consumes exactly k bits, 1 <= k <= 63 (K:63-78)
  __device__ __forceinline__ uint64_t next_bits(uint32_t k) {
    if (nb >= k) {
      uint64_t out = buf & ((1ULL << k) - 1ULL);
      buf >>= k;
      nb -= k;
      return out;
    }
    uint64_t out = buf;
    uint64_t w = next_u64();
    uint32_t need = k - nb;
    out |= (w & ((1ULL << need) - 1ULL)) << nb;
    buf = w >> need;
    nb = 64 - need;
    return out;
  }
  __device__ __forceinline__ uint64_t next53() { return next_bits(53); }
  __device__ __forceinline__ double uniform01() {  // K:81-83
    return (double)next53() * INV53;
  }
};

__host__ __device__ __forceinline__ uint32_t bits_for(int64_t n) {  // K:86-94
#ifdef __CUDA_ARCH__
  return n <= 1 ? 0u : 64u - (uint32_t)__clzll((long long)(n - 1));
#else
  uint32_t k = 0;
  int64_t v = n - 1;
  while (v > 0) { v >>= 1; k++; }
  return k;
#endif
}

// K:97-110: uniform on {0..n-1}; returns -1 when the rejection cap is hit
__device__ __forceinline__ int64_t uniform_int_masked(Stream& st, uint64_t n,
                                                      uint32_t kbits) {
  if (n <= 1) return 0;
  for (int rounds = 0;; ) {
    uint64_t r = st.next_bits(kbits);
    if (r < n) return (int64_t)r;
    if (++rounds > g_reject_cap) return -1;
  }
}
__device__ __forceinline__ int64_t uniform_int(Stream& st, int64_t n) {  // K:113-117
  if (n <= 1) return 0;
  return uniform_int_masked(st, (uint64_t)n, bits_for(n));
}

// E = -log1p(-U) given the 53 raw bits (K:120-122)
__device__ __forceinline__ double exp1_from_bits(uint64_t b53) {
  return -g_log1p_negu(-((double)b53 * INV53));
}

// Conservative lower bound of fl(a * E(b53)) used ONLY to skip evaluating
// log1p for points that provably exceed a threshold.  -log(1-U) >= U, glibc
// log1p is within 1 ulp, and the margin (1 - 2^-40) covers the roundings, so
// lb <= fl(a * E) always; skipping x whenever lb > thr is exact.
__device__ __forceinline__ double exp1_scaled_lower_bound(double a, uint64_t b53) {
  return (a * ((double)b53 * INV53)) * 0.99999999999909051;
}

struct TruncExpConsts { double lam, c1, c2, c3; };

// K:125-151, continuing from the first uniform u0 (already drawn); returns the
// value and sets *fail if the rejection cap is exceeded.
__device__ __noinline__ double trunc_exp_slow(Stream& st, const TruncExpConsts& c,
                                              bool* fail) {
  for (int rounds = 0;; ) {
    double x = st.uniform01();
    if (x < c.c2) return x;
    double y = 0.5 * st.uniform01();
    if (y > 1.0 - x) { x = 1.0 - x; y = 1.0 - y; }
    if (x <= c.c3 * (1.0 - y)) return x;
    if (y * c.c1 <= 1.0 - x) return x;
    bool ok;
    double e = g_expm1(c.lam * (1.0 - x), &ok);
    if (!ok) { *fail = true; return 0.0; }
    if (y * c.c1 * c.lam <= e) return x;
    if (++rounds > g_reject_cap) { *fail = true; return 0.0; }
  }
}
__device__ __forceinline__ double trunc_exp(Stream& st, const TruncExpConsts& c,
                                            bool* fail) {
  double x = c.c1 * st.uniform01();
  if (x < 1.0) return x;
  return trunc_exp_slow(st, c, fail);
}

// Asynchronous 8-byte global -> shared copies (cp.async): element chunks and
// sets stream into shared memory while the warp works on the previous ones.
// 8-byte granularity because set offsets are arbitrary.
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_group1() {
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}

// ---------------------------------------------------------------------------
// Slot table: per component k the lexicographic minimum of (h, element index)
// over all generated points -- the exact semantics of the reference's strict
// `<` updates in input order.  16-byte entries updated
// with a 128-bit shared-memory CAS (ATOMS.CAS.128 on sm_100a).
// h >= 0 always, so its IEEE bit pattern orders like u64.
// ---------------------------------------------------------------------------
struct __align__(16) Slot { unsigned long long h; unsigned long long idx; };

constexpr unsigned long long EMPTY_H = 0x7FF0000000000000ULL;  // +inf
constexpr unsigned long long EMPTY_IDX = ~0ULL;

__device__ __forceinline__ void slot_load(const Slot* p, unsigned long long& h,
                                          unsigned long long& idx) {
  unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(h), "=l"(idx) : "r"(addr) : "memory");
}

__device__ __forceinline__ void cas128_shared(Slot* p, unsigned long long cmp_h,
                                              unsigned long long cmp_i,
                                              unsigned long long new_h,
                                              unsigned long long new_i,
                                              unsigned long long& out_h,
                                              unsigned long long& out_i) {
  unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  asm volatile(
      "{\n\t.reg .b128 c, n, d;\n\t"
      "mov.b128 c, {%2, %3};\n\t"
      "mov.b128 n, {%4, %5};\n\t"
      "atom.shared.cas.b128 d, [%6], c, n;\n\t"
      "mov.b128 {%0, %1}, d;\n\t}"
      : "=l"(out_h), "=l"(out_i)
      : "l"(cmp_h), "l"(cmp_i), "l"(new_h), "l"(new_i), "r"(addr)
      : "memory");
}

// Offer (h, idx) to slot p.  Returns the previous h bits if the slot was
// lowered, or ~0 if the offer lost.
__device__ __forceinline__ unsigned long long slot_offer(Slot* p, double hv,
                                                         unsigned long long idx) {
  const unsigned long long h = dbl_bits(hv);
  unsigned long long ch, ci;
  slot_load(p, ch, ci);
  while (h < ch || (h == ch && idx < ci)) {
    unsigned long long oh, oi;
    cas128_shared(p, ch, ci, h, idx, oh, oi);
    if (oh == ch && oi == ci) return ch;
    ch = oh; ci = oi;
  }
  return ~0ULL;
}

}  // namespace pmh
