/* One-off exhaustive check: spl_expf (csrc/spl_expf.cuh, the GPU encoder's
 * exp) == glibc expf for all 2^32 float bit patterns (NaN payload compared
 * as "both NaN"). Build: g++ -O2 -std=c++17 -ffp-contract=off -fopenmp ... -lm */
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include "../paper_2508_19740_b200/csrc/spl_expf.cuh"
int main(void) {
    unsigned long long bad = 0;
#pragma omp parallel for reduction(+:bad) schedule(static)
    for (long long i = 0; i <= 0xffffffffLL; ++i) {
        uint32_t u = (uint32_t)i; float x; memcpy(&x, &u, 4);
        float a = expf(x), b = spl_expf(x);
        uint32_t ua, ub; memcpy(&ua, &a, 4); memcpy(&ub, &b, 4);
        if (ua != ub && !(isnan(a) && isnan(b))) { if (bad < 5) printf("mismatch x=%a glibc=%a port=%a\n", x, a, b); ++bad; }
    }
    printf("exhaustive: %llu mismatches over 2^32 inputs\n", bad);
    return bad != 0;
}
