// Host check: pmh_math.cuh (compiled by g++, -ffp-contract=off) vs glibc libm.
// Usage: math_check <n_samples> ; prints "log1p_dom <mism> log1p_negu <mism> log1p_wide <mism>
// expm1 <mism> total <n>" and exits 0.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1911_00675_b200/csrc/pmh_math.cuh"

static uint64_t mix64(uint64_t x) {
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  long n = argc > 1 ? atol(argv[1]) : 1000000;
  long m_dom = 0, m_negu = 0, m_wide = 0, m_exp = 0, m_ok = 0;
  for (long i = 0; i < n; i++) {
    uint64_t w = mix64(0x1234ULL + (uint64_t)i * 0x9E3779B97F4A7C15ULL);
    uint64_t w2 = mix64(0x777ULL + (uint64_t)i * 0x9E3779B97F4A7C15ULL);
    // sampled domain: x = -U, U = k 2^-53 (K:81-83,120-122); also stress
    // small U (k < 2^20) and U near 1
    uint64_t k = w >> 11;
    if ((i & 7) == 1) k >>= (w2 & 63);
    if ((i & 7) == 2) k = (1ULL << 53) - 1 - (k >> (w2 & 63));
    double x = -((double)k * 1.1102230246251565e-16);
    if (pmh::dbl_bits(pmh::g_log1p(x)) != pmh::dbl_bits(log1p(x))) m_dom++;
    if (pmh::dbl_bits(pmh::g_log1p_negu(x)) != pmh::dbl_bits(log1p(x))) m_negu++;
    // wide: any finite double > -1
    double y = pmh::bits_dbl(w2 & 0x7fefffffffffffffULL);
    if (w & 1) y = -(double)(w2 >> 11) * 1.1102230246251565e-16 * ((w >> 1) & 1 ? 1.0 : 0.5);
    if (y > -1.0) {
      double a = pmh::g_log1p(y), b = log1p(y);
      if (pmh::dbl_bits(a) != pmh::dbl_bits(b)) m_wide++;
    }
    // expm1 on [0, ln2] (TruncExp argument) and on (-1.5ln2, 1.5ln2)
    double t = (double)(w2 >> 11) * 1.1102230246251565e-16;
    double arg = (i & 1) ? t * 0.6931471805599453 : (t - 0.5) * 2.0 * 1.0397;
    if ((i & 15) == 3) arg = t * pow(2.0, -(double)(w & 63));
    bool ok;
    double e = pmh::g_expm1(arg, &ok);
    if (!ok) m_ok++;
    else if (pmh::dbl_bits(e) != pmh::dbl_bits(expm1(arg))) m_exp++;
  }
  printf("log1p_dom %ld log1p_negu %ld log1p_wide %ld expm1 %ld expm1_outofrange %ld total %ld\n",
         m_dom, m_negu, m_wide, m_exp, m_ok, n);
  return 0;
}
