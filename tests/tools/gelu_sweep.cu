// tests/tools/gelu_sweep.cu -- TEST TOOL (run on the GPU by tests/test_gpu_sweep.py).
//
// Exhaustive accuracy sweep of the In-Place GELU forward value as the
// product computes it (paper_2210_10246_b200/csrc/gelu_math.h +
// gelu_fwd_slow.h: the fp32 fast path plus the fp64 fix-ups) over EVERY
// fp32 bit pattern, against the reference's formula
// float(x * 0.5 * erfc(-x / sqrt2)) evaluated in fp64 (proj/include/tempo/
// math.hpp:17-28; CUDA's fp64 erfc stands in for glibc's, both within ~1
// double ulp, so they round to the same float except at ~2^-28 odds).
//
// Prints one JSON line: inputs checked, max ulp error, ulp histogram, the
// worst input, and how many inputs of the fp64 window |x - x*| < 1/64 differ.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2210_10246_b200/csrc/gelu_fwd_slow.h"

__device__ unsigned long long g_hist[8];
__device__ unsigned long long g_count, g_window, g_window_bad, g_nan_bad;
__device__ unsigned int g_max, g_worst, g_band[8];

__device__ __forceinline__ long long ordinal(float f) {
    int i = __float_as_int(f);
    return i < 0 ? -(long long)(i & 0x7fffffff) : (long long)i;
}

__global__ void sweep(unsigned long long begin, unsigned long long end) {
    unsigned long long hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long cnt = 0, win = 0, winbad = 0, nanbad = 0;
    unsigned int mx = 0, worst = 0;
    for (unsigned long long u = begin + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
         u < end; u += (unsigned long long)gridDim.x * blockDim.x) {
        float x = __uint_as_float((unsigned int)u);
        // exactly the kernel's per-element logic: the packed fp32x2 fast path
        // (lane .x of a pair), fp64 where tm_gelu_needs_fix says so
        float got = tm_gelu_fast2(make_float2(x, 1.0f)).x;
        if (tm_gelu_needs_fix(x, TM_GELU_XSTAR_F)) got = tm_gelu_fix(x);
        const float sc = tm_gelu_fwd(x, TM_GELU_XSTAR_F);
        if (got != sc && !(isnan(got) && isnan(sc))) ++nanbad;  // scalar path must agree
        float ref = (float)tm_gelu_exact(x);
        if (isnan(ref) || isnan(got)) {
            nanbad += (isnan(ref) != isnan(got));
            continue;
        }
        long long d = ordinal(ref) - ordinal(got);
        unsigned int ad = (unsigned int)(d < 0 ? -d : d);
        hist[ad > 7 ? 7 : ad]++;
        ++cnt;
        if (ad > mx) { mx = ad; worst = (unsigned int)u; }
        if (fabsf(x - TM_GELU_XSTAR_F) < TM_GELU_TAYLOR_WINDOW) { ++win; winbad += (ad != 0); }
        // fast-path error inside the window, by distance band 2^-(6+b)
        const float dist = fabsf(x - TM_GELU_XSTAR_F);
        if (dist < 0.015625f) {
            const float fy = tm_gelu_fast2(make_float2(x, 1.0f)).x;
            long long fd = ordinal(ref) - ordinal(fy);
            unsigned int fad = (unsigned int)(fd < 0 ? -fd : fd);
            int b = 0;
            float lim = 0.0078125f;
            while (b < 7 && dist < lim) { ++b; lim *= 0.5f; }
            atomicMax(&g_band[b], fad);
        }
    }
    for (int i = 0; i < 8; ++i) if (hist[i]) atomicAdd(&g_hist[i], hist[i]);
    atomicAdd(&g_count, cnt);
    atomicAdd(&g_window, win);
    atomicAdd(&g_window_bad, winbad);
    atomicAdd(&g_nan_bad, nanbad);
    unsigned int old = atomicMax(&g_max, mx);
    if (mx > old) g_worst = worst;  // racy but only diagnostic
}

int main(int argc, char** argv) {
    unsigned long long stride = argc > 1 ? strtoull(argv[1], 0, 10) : 1;
    unsigned long long total = 1ULL << 32;
    unsigned long long chunk = (1ULL << 30);
    for (unsigned long long b = 0; b < total; b += chunk) {
        if (stride == 1) {
            sweep<<<148 * 16, 256>>>(b, b + chunk);
        } else {
            sweep<<<148 * 16, 256>>>(b, b + chunk / stride);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e)); return 2; }
    unsigned long long hist[8], cnt, win, winbad, nanbad;
    unsigned int mx, worst;
    cudaMemcpyFromSymbol(hist, g_hist, sizeof(hist));
    cudaMemcpyFromSymbol(&cnt, g_count, 8);
    cudaMemcpyFromSymbol(&win, g_window, 8);
    cudaMemcpyFromSymbol(&winbad, g_window_bad, 8);
    cudaMemcpyFromSymbol(&nanbad, g_nan_bad, 8);
    cudaMemcpyFromSymbol(&mx, g_max, 4);
    cudaMemcpyFromSymbol(&worst, g_worst, 4);
    float wx;
    memcpy(&wx, &worst, 4);
    printf("{\"checked\": %llu, \"max_ulp\": %u, \"worst_x\": %.9g, \"hist\": [", cnt, mx, wx);
    for (int i = 0; i < 8; ++i) printf("%llu%s", hist[i], i < 7 ? ", " : "");
    unsigned int band[8];
    cudaMemcpyFromSymbol(band, g_band, sizeof(band));
    printf("], \"window_checked\": %llu, \"window_mismatch\": %llu, \"nan_mismatch\": %llu, "
           "\"fast_path_max_ulp_by_band\": [", win, winbad, nanbad);
    for (int i = 0; i < 8; ++i) printf("%u%s", band[i], i < 7 ? ", " : "");
    printf("]}\n");
    return 0;
}
