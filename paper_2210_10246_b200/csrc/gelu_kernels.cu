// gelu_kernels.cu -- In-Place GELU forward/backward for sm_100a.
//
// Forward  (tempo_ops::gelu, ops_tempo.cpp:89-96 -> inplace_elementwise
//           :32-58 with gelu_spec :73-78): y = x*Phi(x), m = x > x*.
//           HBM: read x (4 B), write y (4 B) + 1 mask bit  = 8.125 B/elem.
// Backward (closure ops_tempo.cpp:59-68 -> GeluPolyTable::eval,
//           gelu_table.cpp:172-188): dx = dy * h(y, m), Clenshaw on the
//           table's piecewise Chebyshev series.
//           HBM: read dy, y (8 B) + 1 bit, write dx (4 B) = 12.125 B/elem.
//
// Layout: the forward's warp owns 256-element chunks (eight floats per lane,
// one 256-bit LDG/STG, the lane's mask byte stored directly); the backward's
// warp owns 128-element chunks (one float4 per lane).  A ragged tail or
// unaligned pointers take the scalar path (32 elements per warp step, one
// ballot = one mask word).
#include <cmath>
#include <limits>
#include <type_traits>

#include "common.cuh"
#include "gelu_math.h"
#include "gelu_fwd_slow.h"
#include "tempo_internal.h"

namespace tb {
namespace {

#ifdef TM_GELU_FWD_MINB
#define TM_GELU_FWD_BOUNDS __launch_bounds__(256, TM_GELU_FWD_MINB)
#else
#define TM_GELU_FWD_BOUNDS __launch_bounds__(256)
#endif
#ifndef TM_GELU_WAVES
#define TM_GELU_WAVES 1
#endif
#ifndef TM_GELU_FWD_U8
#define TM_GELU_FWD_U8 4
#endif
#ifndef TM_GELU_FWD_PP
#define TM_GELU_FWD_PP 1
#endif
constexpr int kBlock = 256;
constexpr int kUnroll = 4;  // chunks in flight per warp (generic backward)

// ---------------------------------------------------------------- forward
__device__ __forceinline__ void gelu_fwd_scalar_words(const float* __restrict__ x,
                                                      float* __restrict__ y,
                                                      uint32_t* __restrict__ mask, int64_t n,
                                                      float xstar_gt, float xs_lo,
                                                      int64_t w_begin,
                                                      int64_t w_step, int lane) {
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = w_begin; w < nwords; w += w_step) {
        int64_t i = (w << 5) + lane;
        bool in = i < n;
        float xv = in ? x[i] : 0.0f;
        bool m = in && (xv >= xstar_gt);
        uint32_t bits = __ballot_sync(kFull, m);
        if (in) y[i] = tm_gelu_fwd(xv, xs_lo);
        if (lane == 0) mask[w] = bits;
    }
}

// ---- forward, 256-bit variant ---------------------------------------------
// Chunk = 256 elements per warp step: lane L owns elements 8L..8L+7 (one
// 32-byte LDG/STG.256) and therefore byte L of the chunk's 32-byte mask, so
// the mask needs no cross-lane packing.  Per element, besides the fast-path
// math (tm_gelu_fast2), one FADD2 gives d = xs_lo - x, whose sign bit IS the
// mask bit (x > x*  <=>  x > xs_lo, the largest float <= x*; NaN gives a
// positive canonical NaN, i.e. bit 0, as the reference's `x > x*`), and one
// FFMA2 gives d*d - 2^-12, whose sign bit flags the fp64 window |x - x*| <
// 1/64; both are collected with one funnel shift each.  The x < -13 tail
// (and -inf) is caught by a running min and re-examined only in that rare
// case.  Elements needing fp64 are fixed after the vector store by the
// owning lane (same thread, same address: program order).
template <int U>
__device__ __forceinline__ void gelu_fwd8_compute(const F8 (&v)[U], float* __restrict__ y,
                                                  uint8_t* __restrict__ mask8, int64_t c0,
                                                  float xs_lo, int lane, float* stage) {
    const float2 XS = f2(xs_lo), NW = f2(-0.000244140625f);  // -(1/64)^2
    uint32_t win = 0;  // bit 8u+k: element k of chunk u is in the fp64 window
    float xmin = 0.0f;
#pragma unroll
    for (int u = U - 1; u >= 0; --u) {
        F8 o;
        uint32_t mb = 0;
#pragma unroll
        for (int k = 6; k >= 0; k -= 2) {
            const float2 xx = make_float2(v[u].v[k], v[u].v[k + 1]);
            const float2 r = tm_gelu_fast2(xx);
            o.v[k] = r.x;
            o.v[k + 1] = r.y;
            const float2 d = __fadd2_rn(XS, neg2(xx));
            const float2 w = __ffma2_rn(d, d, NW);
            mb = push_sign(push_sign(mb, d.y), d.x);
            win = push_sign(push_sign(win, w.y), w.x);
            xmin = fminf(xmin, fminf(xx.x, xx.y));
        }
        const int64_t c = c0 + u;
        st_stream8(y + (c << 8) + 8 * lane, o);
        st_stream(mask8 + (c << 5) + lane, mb);
    }
    if (xmin < TM_GELU_FAST_XMIN) {  // rare: x < -13 or -inf somewhere in this lane
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                win |= (uint32_t)(v[u].v[k] < TM_GELU_FAST_XMIN) << (8 * u + k);
    }
    if (win != 0u) {
        float4* xs = reinterpret_cast<float4*>(stage) + 2 * lane;  // [U][32 lanes][8]
#pragma unroll
        for (int u = 0; u < U; ++u) {
            xs[u * 64] = make_float4(v[u].v[0], v[u].v[1], v[u].v[2], v[u].v[3]);
            xs[u * 64 + 1] = make_float4(v[u].v[4], v[u].v[5], v[u].v[6], v[u].v[7]);
        }
        const float* xsf = stage + 8 * lane;
        float* yb = y + (c0 << 8) + 8 * lane;
        do {
            const int b = __ffs(win) - 1;
            win &= win - 1;
            const int off = (b >> 3) * 256 + (b & 7);
            st_stream(yb + off, tm_gelu_fix(xsf[off]));
        } while (win != 0u);
    }
}

template <int U>
__global__ void TM_GELU_FWD_BOUNDS gelu_fwd8_kernel(const float* __restrict__ x,
                                                    float* __restrict__ y,
                                                    uint32_t* __restrict__ mask, int64_t n,
                                                    float xstar_gt, float xs_lo) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch_persistent();  // one persistent wave (TM_GELU_WAVES)
    __shared__ __align__(16) float stage_all[kBlock / 32][U * 256];
    const int lane = threadIdx.x & 31;
    float* stage = stage_all[threadIdx.x >> 5];
    uint8_t* mask8 = reinterpret_cast<uint8_t*>(mask);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 8;
    const int64_t ngroups = nchunks / U;
#if TM_GELU_FWD_PP
    // ping-pong register buffers: group gi computes from `a` while gi+nwarps
    // loads into `b`, then the roles swap (no register copies)
    F8 a[U], b[U];
    if (warp < ngroups) {
#pragma unroll
        for (int u = 0; u < U; ++u) a[u] = ld_stream8(x + ((warp * U + u) << 8) + 8 * lane);
    }
    for (int64_t gi = warp; gi < ngroups; gi += 2 * nwarps) {
        const int64_t g1 = gi + nwarps, g2 = gi + 2 * nwarps;
        if (g1 < ngroups) {
#pragma unroll
            for (int u = 0; u < U; ++u) b[u] = ld_stream8(x + ((g1 * U + u) << 8) + 8 * lane);
        }
        gelu_fwd8_compute<U>(a, y, mask8, gi * U, xs_lo, lane, stage);
        if (g1 >= ngroups) break;
        if (g2 < ngroups) {
#pragma unroll
            for (int u = 0; u < U; ++u) a[u] = ld_stream8(x + ((g2 * U + u) << 8) + 8 * lane);
        }
        gelu_fwd8_compute<U>(b, y, mask8, g1 * U, xs_lo, lane, stage);
    }
#else
    F8 nxt[U];
    if (warp < ngroups) {
#pragma unroll
        for (int u = 0; u < U; ++u) nxt[u] = ld_stream8(x + ((warp * U + u) << 8) + 8 * lane);
    }
    for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
        F8 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = nxt[u];
        const int64_t gn = gi + nwarps;
        if (gn < ngroups) {
#pragma unroll
            for (int u = 0; u < U; ++u) nxt[u] = ld_stream8(x + ((gn * U + u) << 8) + 8 * lane);
        }
        gelu_fwd8_compute<U>(v, y, mask8, gi * U, xs_lo, lane, stage);
    }
#endif
    for (int64_t c = ngroups * U + warp; c < nchunks; c += nwarps) {
        F8 v[1] = {ld_stream8(x + (c << 8) + 8 * lane)};
        gelu_fwd8_compute<1>(v, y, mask8, c, xs_lo, lane, stage);
    }
    // ragged tail: mask words [8*nchunks, ceil(n/32)) on the last warp
    if (warp == nwarps - 1) {
        gelu_fwd_scalar_words(x, y, mask, n, xstar_gt, xs_lo, nchunks << 3, 1, lane);
    }
}

__global__ void __launch_bounds__(kBlock) gelu_fwd_scalar_kernel(const float* __restrict__ x,
                                                                 float* __restrict__ y,
                                                                 uint32_t* __restrict__ mask,
                                                                 int64_t n, float xstar_gt,
                                                                 float xs_lo) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    gelu_fwd_scalar_words(x, y, mask, n, xstar_gt, xs_lo, warp, nwarps, lane);
}

// ---- forward, reference-exact mode ----------------------------------------
// y = float(x * 0.5 * erfc(-x / sqrt2)) evaluated in fp64 for EVERY element --
// the reference's own formula (math.hpp:17-28, one rounding to float) instead
// of the fp32 fast path (<= 6 ulp): the survey's <= 2 ulp contract is met
// with room (the only differences from the reference are the rare inputs
// where CUDA's and glibc's double erfc straddle a float rounding boundary).
// Same lanes and mask bytes as gelu_fwd8_kernel (the mask bit is the sign
// bit of xs_lo - x); the fp64 erfc makes it FP64-pipe bound.
// vec = 0 (pointers not 32-byte aligned): every element takes the word loop.
__global__ void __launch_bounds__(kBlock) gelu_fwd_exact_kernel(const float* __restrict__ x,
                                                                float* __restrict__ y,
                                                                uint32_t* __restrict__ mask,
                                                                int64_t n, float xstar_gt,
                                                                float xs_lo, int vec) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    uint8_t* mask8 = reinterpret_cast<uint8_t*>(mask);
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = vec ? n >> 8 : 0;
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const F8 v = ld_stream8(x + (c << 8) + 8 * lane);
        F8 o;
        uint32_t mb = 0;
#pragma unroll
        for (int k = 7; k >= 0; --k) {
            o.v[k] = (float)tm_gelu_exact(v.v[k]);
            mb = push_sign(mb, xs_lo - v.v[k]);  // x > x*  <=>  x > xs_lo (NaN -> 0)
        }
        st_stream8(y + (c << 8) + 8 * lane, o);
        st_stream(mask8 + (c << 5) + lane, mb);
    }
    // the rest by mask words [8*nchunks, ceil(n/32)), one word per warp step
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = (nchunks << 3) + warp; w < nwords; w += nwarps) {
        const int64_t i = (w << 5) + lane;
        const bool in = i < n;
        const float xv = in ? x[i] : 0.0f;
        const uint32_t bits = __ballot_sync(kFull, in && xv >= xstar_gt);
        if (in) y[i] = (float)tm_gelu_exact(xv);
        if (lane == 0) mask[w] = bits;
    }
}

// --------------------------------------------------------------- backward
// Shared-memory copy of the table: per-segment parameters and the padded
// coefficient matrix with an odd stride, so lanes on different segments
// read different banks.
struct SmemTable {
    float lo_up[kMaxSeg];
    float s[kMaxSeg];
    float b[kMaxSeg];
    int sqrt_shift[kMaxSeg];
};

__device__ __forceinline__ void load_table(const GeluDevTable& t, SmemTable& st, float* coef) {
    const int nseg = t.nseg[0] + t.nseg[1];
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) {
        st.lo_up[i] = t.lo_up[i];
        st.s[i] = t.s[i];
        st.b[i] = t.b[i];
        st.sqrt_shift[i] = t.sqrt_shift[i];
    }
    for (int i = threadIdx.x; i < nseg * t.ncoef; i += blockDim.x) {
        int sgi = i / t.ncoef, k = i - sgi * t.ncoef;
        coef[sgi * t.stride + k] = t.coef[sgi][k];
    }
    __syncthreads();
}

// h(y, m) = GeluPolyTable::eval (gelu_table.cpp:172-188) in fp32.
__device__ __forceinline__ float gelu_h(float y, uint32_t m, const GeluDevTable& t,
                                        const SmemTable& st, const float* coef, int maxseg) {
    if (isnan(y)) return y;                 // NaN propagates like the reference
    if (m == 0u && y >= 0.0f) return 0.0f;  // :182 far left tail
    const bool clamped = y < t.ymin_up;     // :183, :186 clamp to y_min
    const int base = m ? t.nseg[0] : 0;
    const int ns = t.nseg[m];
    int seg = base;  // last segment with lo <= y (find_segment :157-170)
    for (int k = 1; k < maxseg; ++k) {
        if (k < ns && y >= st.lo_up[base + k]) seg = base + k;
    }
    // u: sqrt(max(y - y_min, 0)) on sqrt-shift segments, y on direct-y ones
    // (eval_segment :66-74).
    float d = (y - t.ymin_hi) - t.ymin_lo;
    float u = st.sqrt_shift[seg] ? sqrtf(fmaxf(d, 0.0f)) : y;
    float tt = fmaf(u, st.s[seg], st.b[seg]);
    tt = fminf(fmaxf(tt, -1.0f), 1.0f);  // :79
    if (clamped) tt = -1.0f;             // u == u_lo exactly after the clamp
    if (st.s[seg] == 0.0f) tt = 0.0f;    // constant segment: c0 (:64)
    // Clenshaw (:43-51): b_k = 2t b_{k+1} - b_{k+2} + c_k; t b_1 - b_2 + c_0.
    const float* c = coef + seg * t.stride;
    const float t2 = tt + tt;
    float b1 = 0.0f, b2 = 0.0f;
    for (int k = t.ncoef - 1; k >= 1; --k) {
        float bk = fmaf(t2, b1, c[k] - b2);
        b2 = b1;
        b1 = bk;
    }
    return fmaf(tt, b1, c[0] - b2);
}

__device__ __forceinline__ void gelu_bwd_scalar_words(const float* __restrict__ dy,
                                                      const float* __restrict__ y,
                                                      const uint32_t* __restrict__ mask,
                                                      float* __restrict__ dx, int64_t n,
                                                      const GeluDevTable& t,
                                                      const SmemTable& st, const float* coef,
                                                      int maxseg, int64_t w_begin,
                                                      int64_t w_step, int lane) {
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = w_begin; w < nwords; w += w_step) {
        int64_t i = (w << 5) + lane;
        uint32_t word = mask[w];
        if (i < n) {
            float h = gelu_h(y[i], (word >> lane) & 1u, t, st, coef, maxseg);
            dx[i] = dy[i] * h;
        }
    }
}

__global__ void __launch_bounds__(kBlock) gelu_bwd_vec_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const uint32_t* __restrict__ mask,
    float* __restrict__ dx, int64_t n, const __grid_constant__ GeluDevTable t) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    __shared__ SmemTable st;
    extern __shared__ float coef[];
    load_table(t, st, coef);
    const int maxseg = max(t.nseg[0], t.nseg[1]);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 7;
    const float4* dy4 = reinterpret_cast<const float4*>(dy);
    const float4* y4 = reinterpret_cast<const float4*>(y);
    float4* dx4 = reinterpret_cast<float4*>(dx);
    for (int64_t c0 = warp * kUnroll; c0 < nchunks; c0 += nwarps * kUnroll) {
        float4 g[kUnroll], v[kUnroll];
        uint32_t nib[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (c0 + u < nchunks) {
                const int64_t off = ((c0 + u) << 5) + lane;
                v[u] = ld_stream(y4 + off);
                g[u] = ld_stream(dy4 + off);
                nib[u] = chunk_nibble(mask + ((c0 + u) << 2), lane);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (c0 + u < nchunks) {
                float4 o;
                o.x = g[u].x * gelu_h(v[u].x, nib[u] & 1u, t, st, coef, maxseg);
                o.y = g[u].y * gelu_h(v[u].y, (nib[u] >> 1) & 1u, t, st, coef, maxseg);
                o.z = g[u].z * gelu_h(v[u].z, (nib[u] >> 2) & 1u, t, st, coef, maxseg);
                o.w = g[u].w * gelu_h(v[u].w, (nib[u] >> 3) & 1u, t, st, coef, maxseg);
                st_stream(dx4 + ((c0 + u) << 5) + lane, o);
            }
        }
    }
    if (warp == nwarps - 1) {
        gelu_bwd_scalar_words(dy, y, mask, dx, n, t, st, coef, maxseg, nchunks << 2, 1, lane);
    }
}

__global__ void __launch_bounds__(kBlock) gelu_bwd_scalar_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const uint32_t* __restrict__ mask,
    float* __restrict__ dx, int64_t n, const __grid_constant__ GeluDevTable t) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    __shared__ SmemTable st;
    extern __shared__ float coef[];
    load_table(t, st, coef);
    const int maxseg = max(t.nseg[0], t.nseg[1]);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    gelu_bwd_scalar_words(dy, y, mask, dx, n, t, st, coef, maxseg, warp, nwarps, lane);
}

// ------------------------------------------------ backward, specialized path
// Tables with <= 4 segments per branch and <= 16 coefficients (the default
// fit: 3 + 3 segments, degree <= 10) use compile-time NC4 = ceil(ncoef/4):
//  * segment search against thresholds held in registers (no smem),
//  * the segment's coefficients read as NC4 128-bit smem loads from a
//    record whose stride keeps up to 8 segments on distinct bank groups,
//  * (s, b) of t = u*s + b as one 64-bit smem load,
//  * a fully unrolled Clenshaw over the zero-padded coefficients,
//  * sqrt.approx for the sqrt-shift variable (rel. error ~2^-23, far inside
//    the 1e-5 tolerance after the smooth Chebyshev map),
// and no data-dependent branches.
constexpr int kFastSegPerBranch = 4;

template <int NC4>
struct FastTable {
    static constexpr int kStride4 = (NC4 & 1) ? NC4 : NC4 + 1;  // float4 units
    float4 rec[kMaxSeg * kStride4];
    float2 sb[kMaxSeg];
};

__device__ __forceinline__ float sqrt_approx(float v) {
    // .ftz: d = y - y_min below 2^-126 flushes to 0 (u ~ 1e-19 either way,
    // far below the evaluation tolerance) and saves the denormal rescaling
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
// NaN-propagating min/max (PTX min/max.NaN): a NaN output y flows through
// to dx exactly as in the reference's double evaluation.
__device__ __forceinline__ float max_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float min_nan(float a, float b) {
    float r;
    asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}

// h(y, m) without data-dependent branches.  y < y_min -> y_min (:183,:186)
// is a clamp on y (the first segment of each branch starts at y_min, and
// sqrt(max(y - y_min, 0)) = 0 for sqrt-shift segments); m = 0, y >= 0 -> 0
// (:182) is the device table's extra constant-0 segment [0, inf) on branch
// 0; y = +inf is clamped to FLT_MAX so constant segments see 0 * v = 0.
// HV (Horner in v = u - u0): the segment record holds the power-basis
// coefficients of v in its first 4*NC4-1 slots and u0 in the last, so one
// segment costs NC4 128-bit smem loads and no (s, b) load or t clamp (the
// segment search keeps v inside the segment up to fp32 rounding, which the
// host's error bound covers).  Else Clenshaw in t as the reference.
template <int NC4, bool HV>
__device__ __forceinline__ float gelu_h_fast(float y, uint32_t m, const FastTable<NC4>& ft,
                                             const float (&thr0)[3], const float (&thr1)[3],
                                             int base1, uint32_t sqrt_mask, float ymin_hi,
                                             float ymin_lo) {
    y = min_nan(y, 3.402823466e38f);
    int seg = m ? base1 : 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) seg += (y >= (m ? thr1[k] : thr0[k])) ? 1 : 0;
    const float d = (y - ymin_hi) - ymin_lo;
    // branch-free variable choice (the SFU sqrt is cheaper than a divergent branch)
    const float sq = sqrt_approx(max_nan(d, 0.0f));
    float u;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.ne.u32 p, %3, 0;\n\t"
        "selp.f32 %0, %1, %2, p;\n}"
        : "=f"(u)
        : "f"(sq), "f"(HV ? max_nan(y, ymin_hi) : y), "r"((sqrt_mask >> seg) & 1u));
    const float4* rec = ft.rec + seg * FastTable<NC4>::kStride4;
    float c[4 * NC4];
#pragma unroll
    for (int j = 0; j < NC4; ++j) {
        const float4 q = rec[j];
        c[4 * j] = q.x;
        c[4 * j + 1] = q.y;
        c[4 * j + 2] = q.z;
        c[4 * j + 3] = q.w;
    }
    if (HV) {
        const float v = u - c[4 * NC4 - 1];
        float h = c[4 * NC4 - 2];
#pragma unroll
        for (int k = 4 * NC4 - 3; k >= 0; --k) h = fmaf(h, v, c[k]);
        return h;
    }
    const float2 sb = ft.sb[seg];
    const float tt = max_nan(min_nan(fmaf(u, sb.x, sb.y), 1.0f), -1.0f);
    const float t2 = tt + tt;  // Clenshaw (gelu_table.cpp:43-51)
    float b1 = 0.0f, b2 = 0.0f;
#pragma unroll
    for (int k = 4 * NC4 - 1; k >= 1; --k) {
        const float bk = fmaf(t2, b1, c[k] - b2);
        b2 = b1;
        b1 = bk;
    }
    return fmaf(tt, b1, c[0] - b2);
}

#ifndef TM_GELU_BWD_V8
#define TM_GELU_BWD_V8 1
#endif
#ifndef TM_GELU_BWD_U8
#define TM_GELU_BWD_U8 2
#endif
template <int NC4, bool HORNER, bool V8, int U8 = TM_GELU_BWD_U8>
__global__ void __launch_bounds__(kBlock) gelu_bwd_fast_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const uint32_t* __restrict__ mask,
    float* __restrict__ dx, int64_t n, const __grid_constant__ GeluDevTable t, int vec) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch_persistent();  // one persistent wave (TM_GELU_WAVES)
    __shared__ FastTable<NC4> ft;
    const int nseg = t.nseg[0] + t.nseg[1];
    for (int i = threadIdx.x; i < nseg * FastTable<NC4>::kStride4; i += kBlock) {
        const int sgi = i / FastTable<NC4>::kStride4, j = i - sgi * FastTable<NC4>::kStride4;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < NC4) {
            const int k = 4 * j;
            const float* src = HORNER ? t.monov[sgi] : t.coef[sgi];
            float e[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                e[r] = k + r < t.ncoef ? src[k + r] : 0.f;
                if (HORNER && k + r == 4 * NC4 - 1) e[r] = t.u0[sgi];  // last slot: u0
            }
            q = make_float4(e[0], e[1], e[2], e[3]);
        }
        ft.rec[i] = q;
    }
    if (!HORNER)
        for (int i = threadIdx.x; i < nseg; i += kBlock) ft.sb[i] = make_float2(t.s[i], t.b[i]);
    float thr0[3], thr1[3];
    uint32_t sqrt_mask = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        thr0[k] = k + 1 < t.nseg[0] ? t.lo_up[k + 1] : __int_as_float(0x7fffffff);  // NaN: never >=
        thr1[k] = k + 1 < t.nseg[1] ? t.lo_up[t.nseg[0] + k + 1] : __int_as_float(0x7fffffff);
    }
    for (int i = 0; i < nseg; ++i) sqrt_mask |= (t.sqrt_shift[i] ? 1u : 0u) << i;

    const int base1 = t.nseg[0];
    const float ymin_hi = t.ymin_hi, ymin_lo = t.ymin_lo;
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
#define TB_H(val, m) gelu_h_fast<NC4, HORNER>(val, m, ft, thr0, thr1, base1, sqrt_mask, \
                                              ymin_hi, ymin_lo)
    if constexpr (V8) {
        // 256-element chunks: lane L owns elements 8L..8L+7 (one 32-byte
        // vector of y, of dy and of dx) and reads its own mask byte.
        constexpr int U = U8;
        const uint8_t* mask8 = reinterpret_cast<const uint8_t*>(mask);
        // vec == 0 (pointers not 32-byte aligned): everything through the
        // scalar loop below -- the same evaluator, so the same bits
        const int64_t nchunks = vec ? (n >> 8) : 0;
        const int64_t ngroups = nchunks / U;
        struct Group {
            F8 g[U], v[U];
            uint32_t mb[U];
        };
        auto load = [&](Group& G, int64_t c0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t off = ((c0 + u) << 8) + 8 * lane;
                G.v[u] = ld_stream8(y + off);
                G.g[u] = ld_stream8(dy + off);
                G.mb[u] = ld_byte(mask8 + ((c0 + u) << 5) + lane);
            }
        };
        auto compute = [&](const Group& G, int64_t c0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                F8 o;
#pragma unroll
                for (int k = 0; k < 8; ++k) o.v[k] = G.g[u].v[k] * TB_H(G.v[u].v[k], (G.mb[u] >> k) & 1u);
                st_stream8(dx + ((c0 + u) << 8) + 8 * lane, o);
            }
        };
        Group a, b;  // ping-pong register buffers
        if (warp < ngroups) load(a, warp * U);
        for (int64_t gi = warp; gi < ngroups; gi += 2 * nwarps) {
            const int64_t g1 = gi + nwarps, g2 = gi + 2 * nwarps;
            if (g1 < ngroups) load(b, g1 * U);
            compute(a, gi * U);
            if (g1 >= ngroups) break;
            if (g2 < ngroups) load(a, g2 * U);
            compute(b, g1 * U);
        }
        // leftover chunks and the ragged tail (< 256 elements): scalar
        for (int64_t i = ((ngroups * U) << 8) + warp * 32 + lane; i < n; i += nwarps * 32) {
            const uint32_t m = (mask[i >> 5] >> (i & 31)) & 1u;
            dx[i] = dy[i] * TB_H(y[i], m);
        }
        return;
    }
#undef TB_H
    const int64_t nchunks = n >> 7;
    const float4* dy4 = reinterpret_cast<const float4*>(dy);
    const float4* y4 = reinterpret_cast<const float4*>(y);
    float4* dx4 = reinterpret_cast<float4*>(dx);
    constexpr int U = 2;
    struct Group {
        float4 g[U], v[U];
        uint32_t nib[U];
    };
    auto load = [&](Group& G, int64_t c0, int uu) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < uu) {
                const int64_t off = ((c0 + u) << 5) + lane;
                G.v[u] = ld_stream(y4 + off);
                G.g[u] = ld_stream(dy4 + off);
                G.nib[u] = chunk_nibble(mask + ((c0 + u) << 2), lane);
            }
        }
    };
    auto compute = [&](const Group& G, int64_t c0, int uu) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < uu) {
#define TB_H(val, bit) gelu_h_fast<NC4, HORNER>(val, (G.nib[u] >> bit) & 1u, ft, thr0, thr1, \
                                                base1, sqrt_mask, ymin_hi, ymin_lo)
                float4 o;
                o.x = G.g[u].x * TB_H(G.v[u].x, 0);
                o.y = G.g[u].y * TB_H(G.v[u].y, 1);
                o.z = G.g[u].z * TB_H(G.v[u].z, 2);
                o.w = G.g[u].w * TB_H(G.v[u].w, 3);
#undef TB_H
                st_stream(dx4 + ((c0 + u) << 5) + lane, o);
            }
        }
    };
    // whole groups of U chunks with the next group's loads in flight during
    // this group's math (register double buffering)
    const int64_t ngroups = nchunks / U;
    Group nxt;
    if (warp < ngroups) load(nxt, warp * U, U);
    for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
        const Group cur = nxt;
        if (gi + nwarps < ngroups) load(nxt, (gi + nwarps) * U, U);
        compute(cur, gi * U, U);
    }
    for (int64_t c = ngroups * U + warp; c < nchunks; c += nwarps) {
        Group one;
        load(one, c, 1);
        compute(one, c, 1);
    }
    // ragged tail (< 128 elements): scalar, same math
    if (warp == nwarps - 1) {
        for (int64_t i = (nchunks << 7) + lane; i < n; i += 32) {
            const uint32_t m = (mask[i >> 5] >> (i & 31)) & 1u;
            dx[i] = dy[i] * gelu_h_fast<NC4, HORNER>(y[i], m, ft, thr0, thr1, base1, sqrt_mask,
                                                     ymin_hi, ymin_lo);
        }
    }
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
// below this many elements the 256-bit kernels take one chunk per register
// group (A/B at configs[0], 3.1 M elements: fwd+bwd 22.5 -> 20.5 us; at the
// 134 M-element bench shape U = 4 / 2 stay faster: 193 vs 221 us fwd)
#ifndef TM_GELU_SMALL_N
#define TM_GELU_SMALL_N (1 << 24)
#endif
constexpr int64_t kSmallN = TM_GELU_SMALL_N;

}  // namespace

cudaError_t launch_gelu_fwd(const float* x, float* y, uint32_t* mask, int64_t n, float xstar_gt,
                            cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const float xs_lo = std::nextafter(xstar_gt, -std::numeric_limits<float>::infinity());
    if (aligned32(x) && aligned32(y) && aligned16(mask)) {
        // small tensors (configs[0]: 3.1 M elements) balance better with one
        // chunk per group (the last group of a warp is the tail)
        const bool small = n < kSmallN;
        const int U = small ? 1 : TM_GELU_FWD_U8;
        const int64_t warps_needed = ((n >> 8) + U - 1) / U + 1;
        auto k = small ? gelu_fwd8_kernel<1> : gelu_fwd8_kernel<TM_GELU_FWD_U8>;
        int grid = grid_for((const void*)k, kBlock, 0, (warps_needed * 32 + kBlock - 1) / kBlock, 0,
                            TM_GELU_WAVES);
        launch(k, grid, kBlock, 0, st)(x, y, mask, n, xstar_gt, xs_lo);
    } else {
        int grid = grid_for((const void*)gelu_fwd_scalar_kernel, kBlock, 0,
                            (((n + 31) >> 5) * 32 + kBlock - 1) / kBlock);
        launch(gelu_fwd_scalar_kernel, grid, kBlock, 0, st)(x, y, mask, n, xstar_gt, xs_lo);
    }
    return cudaGetLastError();
}

cudaError_t launch_gelu_fwd_exact(const float* x, float* y, uint32_t* mask, int64_t n,
                                  float xstar_gt, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const float xs_lo = std::nextafter(xstar_gt, -std::numeric_limits<float>::infinity());
    const int vec = aligned32(x) && aligned32(y) && aligned16(mask);
    const int64_t warps_needed = vec ? (n >> 8) + 1 : (n + 31) >> 5;
    int grid = grid_for((const void*)gelu_fwd_exact_kernel, kBlock, 0,
                        (warps_needed * 32 + kBlock - 1) / kBlock, 0, 4);
    launch(gelu_fwd_exact_kernel, grid, kBlock, 0, st)(x, y, mask, n, xstar_gt, xs_lo, vec);
    return cudaGetLastError();
}

cudaError_t launch_gelu_bwd(const float* dy, const float* y, const uint32_t* mask,
                            const GeluDevTable& t, float* dx, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(dy) && aligned16(y) && aligned16(dx) && aligned16(mask);
    // tables within the fast evaluator's limits always use it (any alignment:
    // the 256-bit, float4 and scalar loops share gelu_h_fast -> same bits)
    const bool fast = t.nseg[0] <= kFastSegPerBranch && t.nseg[1] <= kFastSegPerBranch &&
                      t.ncoef <= 16;
    const bool hv = t.horner && t.ncoef <= 15;  // Horner in v: u0 takes one more slot
    if (fast) {
        // Horner in v needs one slot for u0 after the coefficients
        const int nc4 = (t.ncoef + (hv ? 4 : 3)) / 4;
        const bool v8a = TM_GELU_BWD_V8 && aligned32(dy) && aligned32(y) && aligned32(dx);
        const bool v8 = v8a || !vec;  // unaligned: the V8 kernel's scalar loop
        const int vflag = v8a ? 1 : 0;
        const int64_t blocks = ((n >> 7) / 2 + 1) * 32 / kBlock + 1;
        const bool small = n < kSmallN;  // one chunk per group (see the forward)
#define TB_CASE(NC)                                                                       \
    case NC: {                                                                            \
        auto k = v8 ? (small ? (hv ? gelu_bwd_fast_kernel<NC, true, true, 1>               \
                                   : gelu_bwd_fast_kernel<NC, false, true, 1>)            \
                             : (hv ? gelu_bwd_fast_kernel<NC, true, true>                  \
                                   : gelu_bwd_fast_kernel<NC, false, true>))              \
                    : (hv ? gelu_bwd_fast_kernel<NC, true, false>                        \
                                : gelu_bwd_fast_kernel<NC, false, false>);               \
        int grid = grid_for((const void*)k, kBlock, 0, blocks, 0, TM_GELU_WAVES);         \
        launch(k, grid, kBlock, 0, st)(dy, y, mask, dx, n, t, vflag);                         \
        break;                                                                            \
    }
        switch (nc4) {
            TB_CASE(1)
            TB_CASE(2)
            TB_CASE(3)
            TB_CASE(4)
            default: return cudaErrorInvalidValue;
        }
#undef TB_CASE
        return cudaGetLastError();
    }
    const size_t smem = (size_t)(t.nseg[0] + t.nseg[1]) * t.stride * sizeof(float);
    const void* k = vec ? (const void*)gelu_bwd_vec_kernel : (const void*)gelu_bwd_scalar_kernel;
    const int64_t warps_needed = vec ? ((n >> 7) + kUnroll - 1) / kUnroll + 1 : (n + 31) >> 5;
    int grid = grid_for(k, kBlock, smem, (warps_needed * 32 + kBlock - 1) / kBlock);
    if (vec) {
        launch(gelu_bwd_vec_kernel, grid, kBlock, smem, st)(dy, y, mask, dx, n, t);
    } else {
        launch(gelu_bwd_scalar_kernel, grid, kBlock, smem, st)(dy, y, mask, dx, n, t);
    }
    return cudaGetLastError();
}

}  // namespace tb
