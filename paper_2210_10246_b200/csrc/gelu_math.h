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
// is a degree-9 polynomial in t fitted offline (fp32 coefficients, least
// squares in relative error 3.9e-8, K = 2.5; tests/tools/fit_gelu_q.py).
// a^2 is split exactly (h + l) with an FMA and the exponent -a^2/2*log2(e)
// is carried in two floats, so the exponential does not amplify the
// rounding of a^2; 2^frac runs on the SFU; one rcp.approx + Newton step
// serves both the variable map and the 1/(a+K) factor.  x >= 0 uses
// y = x - x*Q(x) (one rounding).
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
//   exp(-a^2/2): w = -a^2/2 * log2(e) carried as w_hi + w_lo (two FMAs on the
//   exact split h + l of a^2), n = rint(w_hi), 2^(w_hi - n) on the SFU
//   (ex2.approx, |arg| <= 1/2), the low part folded back as (1 + w_lo ln2),
//   and 2^n applied to the exponent bits.
__device__ __forceinline__ float tm_ex2_approx(float f) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
    return r;
}

__device__ __forceinline__ float tm_gelu_q(float a) {
    const float K = 2.5f;
    const float C_HI = -0.72134752044448170f;        // -log2(e)/2, fp32
    const float C_LO = -9.62981494545545e-09f;       // -log2(e)/2 - C_HI
    const float LN2 = 0.69314718055994531f;
    const float h = a * a;
    const float l = fmaf(a, a, -h);                  // a^2 = h + l exactly
    const float w_hi = h * C_HI;
    float w_lo = fmaf(h, C_HI, -w_hi);               // exact rounding error of w_hi
    w_lo = fmaf(h, C_LO, w_lo);
    w_lo = fmaf(l, C_HI, w_lo);                      // the l part of -a^2/2 log2(e)
    const float sh = w_hi + 12582912.0f;             // 1.5*2^23 shifter: rint(w_hi)
    const float n = sh - 12582912.0f;
    const int ni = __float_as_int(sh) - 0x4B400000;
    const float e2 = tm_ex2_approx(w_hi - n);        // w_hi - n exact, |.| <= 1/2
    const float e = fmaf(e2, w_lo * LN2, e2);        // * 2^w_lo ~ 1 + w_lo ln2
    const float E = __int_as_float(__float_as_int(e) + (ni << 23));  // * 2^n, n >= -122
    const float rc = tm_rcp(a + K);
    const float t = (a - K) * rc;
    float q = -1.643887081e-04f;
    q = fmaf(q, t, -3.207997943e-04f);
    q = fmaf(q, t, 6.907590432e-04f);
    q = fmaf(q, t, 2.534991596e-03f);
    q = fmaf(q, t, -1.602514880e-03f);
    q = fmaf(q, t, -1.639061980e-02f);
    q = fmaf(q, t, 9.235967882e-03f);
    q = fmaf(q, t, 1.319876313e-01f);
    q = fmaf(q, t, -4.336920083e-01f);
    q = fmaf(q, t, 7.066566348e-01f);
    return (E * q) * rc;
}

// Fast path: valid for finite x >= -13 (x > 13 gives Q < 2^-126 and y = x,
// as the reference's double result rounds there).
__device__ __forceinline__ float tm_min_nan(float a, float b);
__device__ __forceinline__ float tm_gelu_fast(float x) {
    const float q = tm_gelu_q(fminf(fabsf(x), 13.0f));
    return fmaf(-tm_min_nan(fabsf(x), 3.402823466e38f), q, fmaxf(x, 0.0f));
}

// ---- two elements per instruction: Blackwell's packed fp32x2 pipe ----------
// The same arithmetic as tm_gelu_q / tm_gelu_fast, element for element (each
// FFMA2 lane rounds exactly like the scalar FFMA), issued as FFMA2/FMUL2/
// FADD2 so the forward's FMA-pipe instruction count halves.
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }

__device__ __forceinline__ float2 tm_gelu_q2(float2 a) {
    const float2 K = f2(2.5f), NK = f2(-2.5f);
    const float2 C_HI = f2(-0.72134752044448170f);
    const float2 C_LO = f2(-9.62981494545545e-09f);
    const float2 LN2 = f2(0.69314718055994531f);
    const float2 h = __fmul2_rn(a, a);
    const float2 l = __ffma2_rn(a, a, neg2(h));
    const float2 w_hi = __fmul2_rn(h, C_HI);
    float2 w_lo = __ffma2_rn(h, C_HI, neg2(w_hi));
    w_lo = __ffma2_rn(h, C_LO, w_lo);
    w_lo = __ffma2_rn(l, C_HI, w_lo);
    const float2 sh = __fadd2_rn(w_hi, f2(12582912.0f));
    const float2 n = __fadd2_rn(sh, f2(-12582912.0f));
    const float2 fr = __fadd2_rn(w_hi, neg2(n));
    const float2 e2 = make_float2(tm_ex2_approx(fr.x), tm_ex2_approx(fr.y));
    const float2 e = __ffma2_rn(e2, __fmul2_rn(w_lo, LN2), e2);
    const float2 E = make_float2(
        __int_as_float(__float_as_int(e.x) + ((__float_as_int(sh.x) - 0x4B400000) << 23)),
        __int_as_float(__float_as_int(e.y) + ((__float_as_int(sh.y) - 0x4B400000) << 23)));
    const float2 d = __fadd2_rn(a, K);
    float2 r0;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0.x) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0.y) : "f"(d.y));
    const float2 rc = __ffma2_rn(r0, __ffma2_rn(neg2(d), r0, f2(1.0f)), r0);
    const float2 t = __fmul2_rn(__fadd2_rn(a, NK), rc);
    float2 q = f2(-1.643887081e-04f);
    q = __ffma2_rn(q, t, f2(-3.207997943e-04f));
    q = __ffma2_rn(q, t, f2(6.907590432e-04f));
    q = __ffma2_rn(q, t, f2(2.534991596e-03f));
    q = __ffma2_rn(q, t, f2(-1.602514880e-03f));
    q = __ffma2_rn(q, t, f2(-1.639061980e-02f));
    q = __ffma2_rn(q, t, f2(9.235967882e-03f));
    q = __ffma2_rn(q, t, f2(1.319876313e-01f));
    q = __ffma2_rn(q, t, f2(-4.336920083e-01f));
    q = __ffma2_rn(q, t, f2(7.066566348e-01f));
    return __fmul2_rn(__fmul2_rn(E, q), rc);
}

// y = fma(-|x|, Q(|x|), max(x, 0)): x < 0 gives x*Q, x >= 0 gives x - x*Q,
// each with a single rounding, and no per-element select.
// |x| is clamped to FLT_MAX NaN-propagatingly so +inf gives +inf and NaN
// gives NaN without a separate path.
__device__ __forceinline__ float tm_min_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 tm_gelu_fast2(float2 x) {
    const float2 a = make_float2(fminf(fabsf(x.x), 13.0f), fminf(fabsf(x.y), 13.0f));
    const float2 q = tm_gelu_q2(a);
    return __ffma2_rn(make_float2(-tm_min_nan(fabsf(x.x), 3.402823466e38f),
                                  -tm_min_nan(fabsf(x.y), 3.402823466e38f)),
                      q, make_float2(fmaxf(x.x, 0.0f), fmaxf(x.y, 0.0f)));
}
