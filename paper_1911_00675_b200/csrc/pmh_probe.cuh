// pmh_probe.cuh -- ALU-pipe peak microbenchmark (the roofline denominator of
// the integer-bound signature kernels; MEASURED_PEAKS.json only carries HBM
// and bf16 peaks).  Every thread runs 8 independent LOP3 chains; one LOP3 is
// one 32-bit ALU-pipe operation.
#pragma once
#include <stdint.h>

namespace pmh {

__global__ void __launch_bounds__(256) alu_probe_kernel(int iters, uint32_t* out) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u, a4 = a0 * 11u,
           a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
  const uint32_t b = blockIdx.x | 1u, c = 0x9E3779B9u;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++) {
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a0) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a1) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a2) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a3) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a4) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a5) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a6) : "r"(b), "r"(c));
      asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a7) : "r"(b), "r"(c));
    }
  }
  if ((a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7) == 0x12345678u) out[0] = 1;
}

}  // namespace pmh
