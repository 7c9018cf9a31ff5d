/* Host glibc log1p / expm1 over arrays (test helper, compiled by the GPU math
 * test): the reference reaches exactly these libm symbols through numba
 * (K:120-122, K:146). */
#include <math.h>

void glibc_log1p(const double *x, double *y, long n) {
    for (long i = 0; i < n; i++) y[i] = log1p(x[i]);
}

void glibc_expm1(const double *x, double *y, long n) {
    for (long i = 0; i < n; i++) y[i] = expm1(x[i]);
}
