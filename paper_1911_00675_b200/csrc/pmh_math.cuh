// pmh_math.cuh -- bit-exact device equivalents of the host libm calls the
// reference reaches through numba.
//
// The reference evaluates  E = -log1p(-U)  (K:120-122) and, on TruncExp's slow
// path, expm1(lam*(1-x)) (K:146) with glibc 2.39 libm.  On x86-64 hosts with
// FMA+AVX2 glibc's ifunc resolver selects the FMA builds of the fdlibm-derived
// sysdeps/ieee754/dbl-64/s_log1p.c and s_expm1.c (verified by disassembling
// this image's libm.so.6: resolver at log1p -> 0x7aff0, expm1 -> 0x7ac30, both
// using vfmadd/vfnmadd/vfmsub).  The functions below restate that published
// algorithm with the contractions placed exactly where the compiled glibc
// places them (explicit fma(), everything else one IEEE rounding), so that
//   g_log1p(x) == glibc log1p(x)   and   g_expm1(x) == glibc expm1(x)
// bit-for-bit.  tests/test_math_host.py compiles this header with gcc and
// checks it against the host glibc on millions of inputs of the sampled
// domain; tests/test_gpu_math.py evaluates the DEVICE build (pmh_math_eval)
// on 2^21 inputs per function and compares it with the host glibc bit for bit.
//
// Compile device code with -fmad=false: nothing here relies on contraction.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PMH_HD __host__ __device__ __forceinline__
#define PMH_FMA(a, b, c) fma((a), (b), (c))
#else
#include <math.h>
#include <string.h>
#define PMH_HD static inline
#define PMH_FMA(a, b, c) fma((a), (b), (c))
#endif

namespace pmh {

PMH_HD uint64_t dbl_bits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t u; memcpy(&u, &x, 8); return u;
#endif
}
PMH_HD double bits_dbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  double x; memcpy(&x, &u, 8); return x;
#endif
}
PMH_HD int32_t hi_word(double x) { return (int32_t)(dbl_bits(x) >> 32); }
PMH_HD double with_hi_word(double x, uint32_t hi) {
  return bits_dbl(((uint64_t)hi << 32) | (dbl_bits(x) & 0xffffffffULL));
}

// fdlibm constants (s_log1p.c)
#define PMH_LN2_HI 6.93147180369123816490e-01 /* 3fe62e42 fee00000 */
#define PMH_LN2_LO 1.90821492927058770002e-10 /* 3dea39ef 35793c76 */
#define PMH_LP1 6.666666666666735130e-01      /* 3FE55555 55555593 */
#define PMH_LP2 3.999999999940941908e-01      /* 3FD99999 9997FA04 */
#define PMH_LP3 2.857142874366239149e-01      /* 3FD24924 94229359 */
#define PMH_LP4 2.222219843214978396e-01      /* 3FCC71C5 1D8E78AF */
#define PMH_LP5 1.818357216161805012e-01      /* 3FC74664 96CB03DE */
#define PMH_LP6 1.531383769920937332e-01      /* 3FC39A09 D078C69F */
#define PMH_LP7 1.479819860511658591e-01      /* 3FC2F112 DF3E5244 */

// glibc log1p, FMA build.  Valid for every finite x > -1 (the sampled domain
// is x = -k*2^-53, k in [0, 2^53)); x <= -1, inf and NaN follow fdlibm.
PMH_HD double g_log1p(double x) {
  const int32_t hx = hi_word(x);
  const int32_t ax = hx & 0x7fffffff;
  int32_t k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {
    if (ax >= 0x3ff00000) {
      if (x == -1.0) return -__builtin_inf();
      return (x - x) / (x - x);
    }
    if (ax < 0x3e200000) {
      if (ax < 0x3c900000) return x;
      return PMH_FMA(-(x * x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec4) { k = 0; f = x; hu = 1; }
  } else if (hx >= 0x7ff00000) {
    return x + x;
  }
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = 1.0 + x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
      c = c / u;
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {
      u = with_hi_word(u, (uint32_t)hu | 0x3ff00000u);
    } else {
      k += 1;
      u = with_hi_word(u, (uint32_t)hu | 0x3fe00000u);
      hu = (0x00100000 - hu) >> 2;
    }
    f = u - 1.0;
  }
  const double hfsq = (f * 0.5) * f;
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return PMH_FMA(dk, PMH_LN2_HI, PMH_FMA(dk, PMH_LN2_LO, c));
    }
    const double R = PMH_FMA(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    return PMH_FMA(dk, PMH_LN2_HI, -((R - PMH_FMA(dk, PMH_LN2_LO, c)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = PMH_FMA(z, PMH_LP3, PMH_LP2);
  const double R3 = PMH_FMA(z, PMH_LP5, PMH_LP4);
  const double R4 = PMH_FMA(z, PMH_LP7, PMH_LP6);
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = PMH_FMA(z, PMH_LP1, z2 * R2);
  R = PMH_FMA(z4, R3, R);
  R = PMH_FMA(z6, R4, R);
  const double t = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - t);
  return PMH_FMA(dk, PMH_LN2_HI, -((hfsq - (PMH_FMA(dk, PMH_LN2_LO, c) + t)) - f));
}

// g_log1p restricted to the SAMPLED domain x = -U, U = b 2^-53 in [0, 1)
// (E = -log1p(-U), K:120-122): the same algorithm and roundings with the
// branches that domain never takes removed, and the one it always takes
// simplified:
//   * x > -1, finite and non-positive: no NaN / inf / x >= 2^53 branches;
//   * |x| > 0.2929 (k != 0): u = 1 + x is EXACT (x is a multiple of 2^-53
//     and 0 < u < 0.71), so u - 1 == x exactly and glibc's correction
//     c = x - (u - 1.0) (u < 1: k <= 0) is exactly +0 -- its division c / u
//     (a full IEEE double division) is dropped;
//   * the k = 0 and k != 0 results share one formula: with k = 0 and c = 0,
//     fma(0, ln2_hi, -((hfsq - (fma(0, ln2_lo, 0) + t)) - f)) rounds exactly
//     like f - (hfsq - t) (round-to-nearest is sign-symmetric, the result is
//     never zero here), so the two argument reductions are selected and the
//     polynomial runs once, without divergence.
// Bit-identical to g_log1p (and glibc) on that domain: tests/native/
// math_check.cpp (host) and tests/test_gpu_math.py (device) check it.
// Device: the polynomial and ln2 constants come from the constant bank (an
// FP64 instruction reads a c[][] operand directly; full 64-bit literals would
// be rebuilt in registers by two moves each, every point).
#if defined(__CUDACC__)
__constant__ double g_log1p_k[9] = {PMH_LP1, PMH_LP2, PMH_LP3, PMH_LP4, PMH_LP5, PMH_LP6,
                                    PMH_LP7, PMH_LN2_HI, PMH_LN2_LO};
#endif
#if defined(__CUDA_ARCH__)
#define PMH_KC(i, lit) g_log1p_k[i]
#else
#define PMH_KC(i, lit) (lit)
#endif

PMH_HD double g_log1p_negu(double x) {
  const int32_t hx = hi_word(x);
  const int32_t ax = hx & 0x7fffffff;
  if (ax < 0x3e200000) {           // |x| < 2^-29
    if (ax < 0x3c900000) return x;
    return PMH_FMA(-(x * x), 0.5, x);
  }
  // k != 0 reduction (u = 1 + x exact, c = 0)
  const double u = 1.0 + x;
  int32_t hu = hi_word(u);
  int32_t k = (hu >> 20) - 1023;
  hu &= 0x000fffff;
  double un;
  if (hu < 0x6a09e) {
    un = with_hi_word(u, (uint32_t)hu | 0x3ff00000u);
  } else {
    k += 1;
    un = with_hi_word(u, (uint32_t)hu | 0x3fe00000u);
    hu = (0x00100000 - hu) >> 2;
  }
  double f = un - 1.0;
  if (hx <= (int32_t)0xbfd2bec4) { k = 0; f = x; hu = 1; }   // |x| <= 0.2929: k = 0
  const double hfsq = (f * 0.5) * f;
  const double dk = (double)k;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      return PMH_FMA(dk, PMH_KC(7, PMH_LN2_HI), PMH_FMA(dk, PMH_KC(8, PMH_LN2_LO), 0.0));
    }
    const double R = PMH_FMA(-f, 0.66666666666666666, 1.0) * hfsq;
    if (k == 0) return f - R;
    return PMH_FMA(dk, PMH_KC(7, PMH_LN2_HI), -((R - PMH_FMA(dk, PMH_KC(8, PMH_LN2_LO), 0.0)) - f));
  }
  const double s = f / (2.0 + f);
  const double z = s * s;
  const double R2 = PMH_FMA(z, PMH_KC(2, PMH_LP3), PMH_KC(1, PMH_LP2));
  const double R3 = PMH_FMA(z, PMH_KC(4, PMH_LP5), PMH_KC(3, PMH_LP4));
  const double R4 = PMH_FMA(z, PMH_KC(6, PMH_LP7), PMH_KC(5, PMH_LP6));
  const double z2 = z * z;
  const double z4 = z2 * z2;
  const double z6 = z2 * z4;
  double R = PMH_FMA(z, PMH_KC(0, PMH_LP1), z2 * R2);
  R = PMH_FMA(z4, R3, R);
  R = PMH_FMA(z6, R4, R);
  const double t = (R + hfsq) * s;
  return PMH_FMA(dk, PMH_KC(7, PMH_LN2_HI), -((hfsq - (PMH_FMA(dk, PMH_KC(8, PMH_LN2_LO), 0.0) + t)) - f));
}

// fdlibm constants (s_expm1.c)
#define PMH_Q1 -3.33333333333331316428e-02 /* BFA11111 111110F4 */
#define PMH_Q2 1.58730158725481460165e-03  /* 3F5A01A0 19FE5585 */
#define PMH_Q3 -7.93650757867487942473e-05 /* BF14CE19 9EAADBB7 */
#define PMH_Q4 4.00821782732936239552e-06  /* 3ED0CFCA 86E65239 */
#define PMH_Q5 -2.01099218183624371326e-07 /* BE8AFDB7 6E09C32D */

// glibc expm1, FMA build, for |x| < 1.5*ln2 (the TruncExp slow path evaluates
// expm1(lam*(1-x)) with 0 <= lam*(1-x) <= lam <= ln 2, K:146).  Arguments
// outside that range never reach it; `ok` reports it for the caller.
PMH_HD double g_expm1(double x, bool* ok) {
  const uint32_t hx_full = (uint32_t)hi_word(x);
  const uint32_t xsb = hx_full & 0x80000000u;
  const uint32_t hx = hx_full & 0x7fffffffu;
  *ok = true;
  int k;
  double hi, lo, c = 0.0;
  if (hx > 0x3fd62e42u) {          // |x| > 0.5 ln2
    if (hx < 0x3FF0A2B2u) {        // |x| < 1.5 ln2
      if (xsb == 0) { hi = x - PMH_LN2_HI; lo = PMH_LN2_LO; k = 1; }
      else { hi = x + PMH_LN2_HI; lo = -PMH_LN2_LO; k = -1; }
      x = hi - lo;
      c = (hi - x) - lo;
    } else {
      *ok = false;
      return 0.0;
    }
  } else if (hx < 0x3c900000u) {   // |x| < 2^-54
    return x;
  } else {
    k = 0;
  }
  const double hfx = x * 0.5;
  const double hxs = x * hfx;
  const double R2 = PMH_FMA(hxs, PMH_Q3, PMH_Q2);
  const double R3 = PMH_FMA(hxs, PMH_Q5, PMH_Q4);
  const double h2 = hxs * hxs;
  const double R1 = PMH_FMA(hxs, PMH_Q1, 1.0);
  const double h4 = h2 * h2;
  double r1 = PMH_FMA(h2, R2, R1);
  r1 = PMH_FMA(h4, R3, r1);
  const double t = PMH_FMA(-r1, hfx, 3.0);
  double e = ((r1 - t) / PMH_FMA(-x, t, 6.0)) * hxs;
  if (k == 0) return x - PMH_FMA(e, x, -hxs);
  e = PMH_FMA(e - c, x, -c);
  e = e - hxs;
  if (k == -1) return PMH_FMA(x - e, 0.5, -0.5);
  if (x < -0.25) return (e - (x + 0.5)) * -2.0;
  return PMH_FMA(x - e, 2.0, 1.0);
}

}  // namespace pmh
