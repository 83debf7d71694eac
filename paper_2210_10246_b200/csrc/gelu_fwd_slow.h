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

// Does x need an fp64 path?  Two unsigned range tests on the bit pattern:
//  * the window around x* (bits of -0.7361665 .. -0.7674165, widened by 16
//    ulps so it covers the float test |x - x*| < 1/64 used below),
//  * x < -13, -inf and negative NaNs (every pattern above -13's).
// +inf and positive NaNs are handled by the fast path itself.
__device__ __forceinline__ bool tm_gelu_needs_slow(float x) {
    const uint32_t u = __float_as_uint(x);
    return (u - (0xBF3C7569u - 16u)) <= (0xBF447569u - 0xBF3C7569u + 32u) || u > 0xC1500000u;
}

__device__ __noinline__ float tm_gelu_slow(float x) {
    if (fabsf(x - TM_GELU_XSTAR_F) < TM_GELU_TAYLOR_WINDOW) return (float)tm_gelu_taylor(x);
    return (float)tm_gelu_exact(x);
}

// Full forward for one element.
__device__ __forceinline__ float tm_gelu_fwd(float x) {
    float y = tm_gelu_fast(x);
    if (tm_gelu_needs_slow(x)) y = tm_gelu_slow(x);
    return y;
}
