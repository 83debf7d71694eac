/* tests/tools/gelu_fwd_sweep.c -- TEST TOOL.
 *
 * Exhaustive accuracy sweep of the In-Place GELU forward fast path
 * (paper_2210_10246_b200/csrc/gelu_math.h, compiled here for the host; every
 * op there is an explicitly rounded IEEE fp32 op, so the host build computes
 * the same bits as the device) against the reference's formula
 * float(x * 0.5 * erfc(-x / sqrt2)) in double (proj/include/tempo/math.hpp:
 * 17-28, rounded once by tensor.hpp:114-116).
 *
 * Usage: gelu_fwd_sweep [stride]   -- stride 1 visits every fp32 bit pattern
 * in the fast-path domain [-13, +inf) outside the slow-path window.
 * Prints: inputs checked, max ulp error, histogram of ulp errors.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "../../paper_2210_10246_b200/csrc/gelu_math.h"

static float as_f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static int64_t ord(float f) {
    int32_t i; memcpy(&i, &f, 4);
    return i < 0 ? -(int64_t)(i & 0x7fffffff) : (int64_t)i;
}

int main(int argc, char** argv) {
    uint64_t stride = argc > 1 ? strtoull(argv[1], 0, 10) : 1;
    const double x_star = -0.75179152469399924;
    int64_t maxd = 0; uint64_t n = 0; uint64_t hist[8] = {0};
    float worst = 0.f;
#pragma omp parallel for reduction(+:n) schedule(dynamic, 65536)
    for (int64_t u = 0; u < (int64_t)0x100000000LL; u += stride) {
        float x = as_f((uint32_t)u);
        if (!isfinite(x) || x < TM_GELU_FAST_XMIN) continue;
        if (fabs((double)x - x_star) < TM_GELU_WINDOW) continue;
        float ref = (float)((double)x * (0.5 * erfc(-(double)x * 0.70710678118654752440)));
        float got = tm_gelu_fast(x);
        int64_t d = llabs(ord(ref) - ord(got));
        ++n;
        int b = d > 7 ? 7 : (int)d;
#pragma omp atomic
        hist[b]++;
        if (d > maxd) {
#pragma omp critical
            if (d > maxd) { maxd = d; worst = x; }
        }
    }
    printf("checked %llu max_ulp %lld worst_x %.9g hist", (unsigned long long)n, (long long)maxd, worst);
    for (int i = 0; i < 8; ++i) printf(" %llu", (unsigned long long)hist[i]);
    printf("\n");
    return maxd > 4;
}
