// gelu_math.h -- the In-Place GELU forward value, y = x * Phi(x), on sm_100a.
//
// The reference evaluates x * 0.5 * erfc(-x / sqrt2) in double and rounds to
// float once (proj/include/tempo/math.hpp:17-28, tensor.hpp:114-116).  A
// double erfc costs ~60 DFMA per element -- far beyond the HBM roofline
// budget of the forward (8.125 B/elem: ~44 fp32 issue slots per element at
// 6.5 TB/s) -- so the fast path is fp32 and branch free:
//
//   Q(a) = Phi(-a) = exp(-a^2/2) * P(t) / (a + K),   t = (a - K) / (a + K)
//
// where P ~ (a + K) Q(a) e^{a^2/2} is smooth (1.25 .. 0.40 on [0, 13]) and
// is a degree-10 polynomial in t fitted offline (fp32 coefficients, least
// squares in relative error, K = 2.5; tests/tools/fit_gelu_q.py).  a^2 is
// split exactly (h + l) with an FMA so the exponential does not amplify the
// rounding of a^2; exp uses a Cody-Waite reduction and a degree-7 Taylor
// kernel; one rcp.approx + Newton step serves both the variable map and the
// 1/(a+K) factor.  x >= 0 uses y = x - x*Q(x) (one rounding).
//
// Accuracy against the reference's double formula, over EVERY fp32 input
// (tests/tools/gelu_sweep.cu, run by tests/test_gpu_sweep.py): see DESIGN.md.
// Inputs the fast path does not cover -- the window |x - x*| < 1/64 around
// the GELU minimum (where h(y) ~ sqrt(y - y_min) makes the backward ill
// conditioned, SURVEY section 7 hard part 2), x < -13, +-inf, NaN -- are
// routed to the fp64 paths of gelu_fwd_slow.h.
#pragma once

#define TM_GELU_FAST_XMIN (-13.0f)

__device__ __forceinline__ float tm_rcp(float d) {  // ~0.5 ulp for d in [2.5, 16]
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
    return fmaf(r, fmaf(-d, r, 1.0f), r);
}

// Q(a) = Phi(-a), a in [0, 13].
__device__ __forceinline__ float tm_gelu_q(float a) {
    const float K = 2.5f;
    const float ln2_hi = 0.693145751953125f;      // 0x3f317200: n*ln2_hi exact
    const float ln2_lo = 1.428606765330187e-06f;  // 0x35bfbe8e
    const float h = a * a;
    const float l = fmaf(a, a, -h);  // a^2 = h + l exactly
    const float v = -0.5f * h;
    // n = rint(v * log2e) via the 1.5*2^23 shifter (no F2I/FRND)
    const float sh = fmaf(v, 1.44269504088896341f, 12582912.0f);
    const float n = sh - 12582912.0f;
    const int ni = __float_as_int(sh) - 0x4B400000;
    float r = fmaf(n, -ln2_hi, v);
    r = fmaf(n, -ln2_lo, r);
    float p = 1.98412698e-04f;          // 1/5040
    p = fmaf(p, r, 1.38888889e-03f);    // 1/720
    p = fmaf(p, r, 8.33333377e-03f);    // 1/120
    p = fmaf(p, r, 4.16666679e-02f);    // 1/24
    p = fmaf(p, r, 1.66666672e-01f);    // 1/6
    p = fmaf(p, r, 0.5f);
    p = fmaf(p, r, 1.0f);
    p = fmaf(p, r, 1.0f);
    const float e = p * __int_as_float((ni + 127) << 23);  // n >= -122 here
    const float E = fmaf(e, -0.5f * l, e);                 // * exp(-l/2)
    const float rc = tm_rcp(a + K);
    const float t = (a - K) * rc;
    float q = -2.982836304e-05f;
    q = fmaf(q, t, -2.068497561e-04f);
    q = fmaf(q, t, -2.954241645e-04f);
    q = fmaf(q, t, 7.393874694e-04f);
    q = fmaf(q, t, 2.528889570e-03f);
    q = fmaf(q, t, -1.621615840e-03f);
    q = fmaf(q, t, -1.639027148e-02f);
    q = fmaf(q, t, 9.238829836e-03f);
    q = fmaf(q, t, 1.319876313e-01f);
    q = fmaf(q, t, -4.336921275e-01f);
    q = fmaf(q, t, 7.066566348e-01f);
    return (E * q) * rc;
}

// Fast path: valid for finite x >= -13 (x > 13 gives Q < 2^-126 and y = x,
// as the reference's double result rounds there).
__device__ __forceinline__ float tm_gelu_fast(float x) {
    const float q = tm_gelu_q(fminf(fabsf(x), 13.0f));
    return x < 0.0f ? x * q : fmaf(-x, q, x);
}
