// gelu_fwd_slow.h -- fp64 paths of the In-Place GELU forward.
//
// (1) The window |x - x*| < 1/64 around the GELU minimum, where the
//     derivative-from-output h(y) ~ sqrt(y - y_min) is ill conditioned
//     (hard part 2): the stored y must round exactly like
//     the reference's double x*Phi(x) so the forward->backward chain matches.
//     There g(x) = x*Phi(x) is a degree-9 Taylor series about x* in fp64
//     (coefficients from tests/tools/gelu_taylor_coeffs.py, mpmath at 50
//     digits; truncation + coefficient rounding < 3e-17 relative), i.e.
//     ~10 DFMA instead of a full erfc.
// (2) x < -13, +-inf and NaN: the reference formula itself in fp64.
#pragma once

#include "gelu_math.h"

// Expansion point: the double nearest the GELU minimum (g'(x*) = 0).
#define TM_GELU_XSTAR_D (-0.7517915246935645)
#define TM_GELU_XSTAR_F (-0.751791525f)
#define TM_GELU_TAYLOR_WINDOW (0.015625f)

__device__ __forceinline__ double tm_gelu_taylor(float x) {
    double h = (double)x - TM_GELU_XSTAR_D;  // exact (Sterbenz)
    double p = -0.00024883756311927746;      // a_9
    p = fma(p, h, 0.000567403547390677);     // a_8
    p = fma(p, h, 0.0027745256911698665);    // a_7
    p = fma(p, h, -0.002461920358040723);    // a_6
    p = fma(p, h, -0.02280164665944434);     // a_5
    p = fma(p, h, -0.00454991909966777);     // a_4
    p = fma(p, h, 0.12942832766351733);      // a_3
    p = fma(p, h, 0.21574699615702345);      // a_2
    p = fma(p, h, -6.453751729367753e-18);   // a_1
    p = fma(p, h, -0.16997120747990366);     // a_0
    return p;
}

// The reference formula (math.hpp:17-28) in fp64.
__device__ __forceinline__ double tm_gelu_exact(float x) {
    double xd = (double)x;
    return xd * (0.5 * erfc(-xd * 0.70710678118654752440));
}

// Does x need an fp64 path?  The window |x - xs_lo| < 1/64 around the GELU
// minimum (xs_lo = the largest float <= the table's x*; for the default
// table exactly TM_GELU_XSTAR_F) tested as the sign of fma(d, d, -2^-12)
// with d = xs_lo - x (exact near the window edge by Sterbenz, and a fused
// sign is the exact sign), plus x < -13 and -inf.  NaN and +inf are handled
// by the fast path itself.  The vector kernel evaluates the same predicate
// with FADD2/FFMA2 sign bits, so both paths fix exactly the same inputs.
#define TM_GELU_WINDOW_SQ_NEG (-0.000244140625f)
__device__ __forceinline__ bool tm_gelu_needs_fix(float x, float xs_lo) {
    const float d = xs_lo - x;
    return fmaf(d, d, TM_GELU_WINDOW_SQ_NEG) < 0.0f || x < TM_GELU_FAST_XMIN;
}

__device__ __noinline__ float tm_gelu_exact_call(float x) { return (float)tm_gelu_exact(x); }

// The fp64 value of a flagged element: the Taylor series inside the window,
// the reference formula elsewhere.
__device__ __forceinline__ float tm_gelu_fix(float x) {
    if (fabsf(x - TM_GELU_XSTAR_F) < TM_GELU_TAYLOR_WINDOW) return (float)tm_gelu_taylor(x);
    return tm_gelu_exact_call(x);
}

// Full forward for one element.
__device__ __forceinline__ float tm_gelu_fwd(float x, float xs_lo) {
    float y = tm_gelu_fast(x);
    if (tm_gelu_needs_fix(x, xs_lo)) y = tm_gelu_fix(x);
    return y;
}
