// gelu_math.h -- the fp32 fast path of the In-Place GELU forward.
//
// Computes y = x * Phi(x) (the erfc form of proj/include/tempo/math.hpp:17-28,
// which the reference evaluates in double and rounds to float once,
// tensor.hpp:114-116) with fp32 arithmetic only, so the forward stays on the
// HBM roofline instead of the FP64 pipe.
//
// Every operation is an explicitly rounded IEEE fp32 op (no contraction, no
// MUFU approximation), so this header compiled for the HOST reproduces the
// device results bit for bit.  tests/tools/gelu_fwd_sweep.c uses that to
// check the fast path against the reference's double formula on EVERY fp32
// input of its domain.
//
// Q(a) = 1 - Phi(a) = Phi(-a), a >= 0, is factored as
//     Q(a) = exp(-a^2/2) * P(t) / (a + K),   t = (a - K) / (a + K)
// where P ~ (a + K) Q(a) e^{a^2/2} is smooth (1.25 .. 0.40 on [0, 13]) and
// is a degree-10 polynomial in t fitted offline (fp32 coefficients, least
// squares in relative error, K = 2.5; the fit script is
// tests/tools/fit_gelu_q.py).
// a^2 is split exactly (h + l) with an FMA so the exponential does not
// amplify the rounding of a^2.
//
// Domain of the fast path: -13 <= x (finite).  Callers route x < -13,
// non-finite x, and the window around the GELU minimum (where the
// derivative-from-output is ill conditioned, SURVEY section 7 hard part 2)
// to the fp64 slow path.
#pragma once

#if defined(__CUDACC__)
#define TM_HD __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define TM_FMA(a, b, c) __fmaf_rn((a), (b), (c))
#define TM_MUL(a, b) __fmul_rn((a), (b))
#define TM_ADD(a, b) __fadd_rn((a), (b))
#define TM_DIV(a, b) __fdiv_rn((a), (b))
#define TM_RINT(a) rintf(a)
#define TM_AS_FLOAT(i) __int_as_float(i)
#else
#include <math.h>
#include <string.h>
static inline float tm_as_float_host(int i) { float f; memcpy(&f, &i, 4); return f; }
#define TM_FMA(a, b, c) fmaf((a), (b), (c))
#define TM_MUL(a, b) ((a) * (b))
#define TM_ADD(a, b) ((a) + (b))
#define TM_DIV(a, b) ((a) / (b))
#define TM_RINT(a) rintf(a)
#define TM_AS_FLOAT(i) tm_as_float_host(i)
#endif
#else
#include <math.h>
#include <string.h>
#define TM_HD static inline
static inline float tm_as_float_host(int i) { float f; memcpy(&f, &i, 4); return f; }
#define TM_FMA(a, b, c) fmaf((a), (b), (c))
#define TM_MUL(a, b) ((a) * (b))
#define TM_ADD(a, b) ((a) + (b))
#define TM_DIV(a, b) ((a) / (b))
#define TM_RINT(a) rintf(a)
#define TM_AS_FLOAT(i) tm_as_float_host(i)
#endif

// Fast-path domain and the slow-path window around the minimum.
#define TM_GELU_FAST_XMIN (-13.0f)
#define TM_GELU_WINDOW (0.03125f)

// exp(v) for v in [-88, 0]: Cody-Waite reduction by ln2 (hi part has zero
// low bits so n*ln2_hi is exact), degree-7 Taylor on |r| <= ln2/2
// (truncation 5.5e-9 relative), exact scaling by 2^n (n >= -126 here).
TM_HD float tm_exp_nonpos(float v) {
    const float log2e = 1.44269504088896341f;
    const float ln2_hi = 0.693145751953125f;      // 0x3f317200
    const float ln2_lo = 1.428606765330187e-06f;  // 0x35bfbe8e
    float n = TM_RINT(TM_MUL(v, log2e));
    float r = TM_FMA(n, -ln2_hi, v);
    r = TM_FMA(n, -ln2_lo, r);
    float p = 1.98412698e-04f;          // 1/5040
    p = TM_FMA(p, r, 1.38888889e-03f);  // 1/720
    p = TM_FMA(p, r, 8.33333377e-03f);  // 1/120
    p = TM_FMA(p, r, 4.16666679e-02f);  // 1/24
    p = TM_FMA(p, r, 1.66666672e-01f);  // 1/6
    p = TM_FMA(p, r, 0.5f);
    p = TM_FMA(p, r, 1.0f);
    p = TM_FMA(p, r, 1.0f);
    int e = (int)n + 127;
    return TM_MUL(p, TM_AS_FLOAT(e << 23));
}

// Q(a) = Phi(-a) for a in [0, 13]:  Q = exp(-a^2/2) * P(t) * r,
// r = 1 / (a + K), t = (a - K) * r, P(t) ~ (a + K) * Q(a) * e^{a^2/2}
// (degree 10, fp32 coefficients, 3.1e-8 relative fit error, K = 2.5).
// One IEEE division serves both the variable map and the 1/(a+K) factor.
TM_HD float tm_gelu_q(float a) {
    const float K = 2.5f;
    float h = TM_MUL(a, a);
    float l = TM_FMA(a, a, -h);  // a^2 = h + l exactly
    float e = tm_exp_nonpos(TM_MUL(-0.5f, h));
    float E = TM_FMA(e, TM_MUL(-0.5f, l), e);  // * exp(-l/2) ~ (1 - l/2)
    float r = TM_DIV(1.0f, TM_ADD(a, K));
    float t = TM_MUL(TM_ADD(a, -K), r);
    float p = -2.982836304e-05f;
    p = TM_FMA(p, t, -2.068497561e-04f);
    p = TM_FMA(p, t, -2.954241645e-04f);
    p = TM_FMA(p, t, 7.393874694e-04f);
    p = TM_FMA(p, t, 2.528889570e-03f);
    p = TM_FMA(p, t, -1.621615840e-03f);
    p = TM_FMA(p, t, -1.639027148e-02f);
    p = TM_FMA(p, t, 9.238829836e-03f);
    p = TM_FMA(p, t, 1.319876313e-01f);
    p = TM_FMA(p, t, -4.336921275e-01f);
    p = TM_FMA(p, t, 7.066566348e-01f);
    return TM_MUL(TM_MUL(E, p), r);
}

// y = gelu(x) for x in [-13, +inf) finite.  x >= 0 uses x - x*Q(x) with a
// single rounding; a > 13 gives Q < 2^-126 and y == x exactly, as the
// reference's double result rounds there.
TM_HD float tm_gelu_fast(float x) {
    float a = fabsf(x);
    if (a > 13.0f) return x >= 0.0f ? x : 0.0f;  // negative side never taken
    float q = tm_gelu_q(a);
    return x < 0.0f ? TM_MUL(x, q) : TM_FMA(-x, q, x);
}
