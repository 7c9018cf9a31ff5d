// pmh_join.cuh -- exact all-pairs equal-component histogram by a hash join
// on (component, value), for signature batches whose sets rarely share
// components (BASELINE configs[4]: 100,000 signatures, 5e9 pairs, ~50,000
// pairs with any equal component).
//
// The dense path (pmh_pminhash.cuh: allpairs_lo / cand / zeros) compares
// every component of every pair: n^2 m / 2 compares, ~145 ms for configs[4].
// Two signatures agree in component k iff they hold the same value there, so
// the pairs with a NON-zero count are exactly the pairs that share a
// (k, value) key.  The join:
//   1. inserts every (i, k) into a per-component open-addressing table keyed
//      by the value (128-bit CAS on {value, occupied}); the slot's head index
//      is swapped in atomically and the previous head linked behind i, so
//      each value's sets form a list;
//   2. walks, for every (i, k), the list behind i: each pair sharing the key
//      is visited exactly once (by its later-inserted member) -- first only
//      counted (the work bound: sum over keys of K(K-1)/2), then inserted
//      into a pair hash map that accumulates the number of shared
//      components;
//   3. scans the map: hist[c] += 1 per pair with count c >= 1, pairs with
//      c >= thr listed; hist[0] += (pairs in range) - (pairs in the map).
// The result equals the dense path's bit for bit (same histogram, same pair
// set).  The host entry declines (returns 1) when the key lists are long
// (sum K(K-1)/2 above a budget: e.g. many duplicate sets) so the caller
// falls back to the dense path.
#pragma once
#include <stdint.h>

#include "pmh_device.cuh"

namespace pmh {

struct JoinSlot { unsigned long long key, occ; };   // occ: 0 empty, 1 taken

__device__ __forceinline__ uint64_t join_hash(uint64_t v) {
  return mix64(v ^ 0x5851F42D4C957F2DULL);
}

// 1. insert (i, k) for i < n, k in [k0, k0 + G): table of component k0 + kk
// at tab + kk * C, heads parallel; next[i * G + kk] = previous head (-1)
__global__ void __launch_bounds__(256) join_insert_kernel(
    const uint64_t* __restrict__ sigs, int64_t n, int64_t m, int64_t k0, int64_t G, JoinSlot* tab,
    int32_t* head, int32_t* next, int logC) {
  const uint64_t mask = (1ULL << logC) - 1ULL;
  const int64_t total = n * G;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / G, kk = idx - i * G;
    const uint64_t v = sigs[i * m + k0 + kk];
    JoinSlot* t = tab + (kk << logC);
    uint64_t h = join_hash(v) & mask;
    for (;;) {
      unsigned long long oh, oo;
      asm volatile(
          "{\n\t.reg .b128 c, nv, d;\n\t"
          "mov.b128 c, {%2, %3};\n\t"
          "mov.b128 nv, {%4, %5};\n\t"
          "atom.global.cas.b128 d, [%6], c, nv;\n\t"
          "mov.b128 {%0, %1}, d;\n\t}"
          : "=l"(oh), "=l"(oo)
          : "l"(0ULL), "l"(0ULL), "l"((unsigned long long)v), "l"(1ULL), "l"(&t[h])
          : "memory");
      if (oo == 0ULL || oh == v) break;   // claimed it, or the key is already there
      h = (h + 1) & mask;
    }
    const int32_t prev = atomicExch(&head[(kk << logC) + h], (int32_t)i);
    next[idx] = prev;
  }
}

__device__ __forceinline__ bool join_in_range(int64_t a, int64_t b, int64_t r0, int64_t r1,
                                              int64_t c0, int64_t c1) {
  return a >= r0 && a < r1 && b >= c0 && b < c1;
}

// pair map: key (i << 32) | j (i < j < 2^31: never ~0), count
struct PairSlot { unsigned long long key; unsigned long long cnt; };
constexpr unsigned long long PAIR_EMPTY = ~0ULL;

// 2. walk the key lists: COUNT (map == nullptr) adds the number of in-range
// pair visits to *visits; otherwise each visit adds 1 to the pair's count
__global__ void __launch_bounds__(256) join_emit_kernel(
    const int32_t* __restrict__ next, int64_t n, int64_t G, int64_t r0, int64_t r1, int64_t c0,
    int64_t c1, unsigned long long* visits, PairSlot* map, int logM) {
  const uint64_t mask = (1ULL << logM) - 1ULL;
  const int64_t total = n * G;
  unsigned long long local = 0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / G, kk = idx - i * G;
    for (int32_t p = next[idx]; p >= 0; p = next[(int64_t)p * G + kk]) {
      const int64_t a = p < i ? p : i, b = p < i ? i : p;
      if (a == b || !join_in_range(a, b, r0, r1, c0, c1)) continue;
      if (!map) { local++; continue; }
      const unsigned long long key = ((unsigned long long)a << 32) | (unsigned long long)b;
      uint64_t h = join_hash(key) & mask;
      for (;;) {
        const unsigned long long cur = atomicCAS(&map[h].key, PAIR_EMPTY, key);
        if (cur == PAIR_EMPTY || cur == key) { atomicAdd(&map[h].cnt, 1ULL); break; }
        h = (h + 1) & mask;
      }
    }
  }
  if (!map) {
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(visits, local);
  }
}

// 3. the map into the histogram and the pair list; *occ counts the pairs
__global__ void __launch_bounds__(256) join_scan_kernel(
    const PairSlot* __restrict__ map, int64_t slots, int64_t m, int32_t thr, unsigned long long* hist,
    unsigned long long* pairs, int64_t cap, unsigned long long* cursor, unsigned long long* occ) {
  unsigned long long local = 0;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = map[s].key;
    if (key == PAIR_EMPTY) continue;
    const unsigned long long c = map[s].cnt;
    local++;
    atomicAdd(&hist[c <= (unsigned long long)m ? c : m], 1ULL);
    if ((long long)c >= (long long)thr) {
      const unsigned long long slot = atomicAdd(cursor, 1ULL);
      if ((long long)slot < cap) {
        pairs[2 * slot] = key;
        pairs[2 * slot + 1] = c;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(occ, local);
}

// hist[0] += pairs in range - pairs with a shared component; with thr <= 0
// the zero-count pairs would have to be listed too: not supported here
__global__ void join_zeros_kernel(unsigned long long* hist, const unsigned long long* occ,
                                  unsigned long long in_range) {
  hist[0] += in_range - *occ;
}

}  // namespace pmh
