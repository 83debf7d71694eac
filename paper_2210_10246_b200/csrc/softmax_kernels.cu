// softmax_kernels.cu -- output-only softmax + sub-layer dropout recomputation
// for sm_100a (attention probabilities, rows of S columns).
//
// Forward (tempo_ops::softmax ops_tempo.cpp:158-166 -> softmax_forward
//   ops_reference.cpp:104-125; tempo_ops::dropout_recompute :168-194 ->
//   dropout_apply :147-153 -> mask_scale kernels.cpp:285-295), fused:
//   read z (4 B), write P (4 B), D (4 B) and the mask bit  = 12.125 B/elem.
//   The stash is P + bits; D goes to the consumer and is never stashed.
// Backward (dropout_backward ops_tempo.cpp:188-190 -> softmax_backward_
//   from_output ops_reference.cpp:127-145, plus the "dropout-rescale"
//   recompute of D for the consumer, ops_tempo.cpp:17-26), fused:
//   read dD, P (8 B) + bit, write dZ (4 B)   = 12.125 B/elem (+4 B with D).
//
// Numerics follow the reference's F32 path where it is cheap to do so
// exactly: dP and D are the fp64 products rounded once (bit-exact with
// mask_scale on the same inputs) and the row dot sum(dP*P) accumulates in
// fp64; the forward's exp runs in fp32 with the rounding error of (z - max)
// folded back in (TwoSum), the row denominator is an fp32 tree sum and
// P = e * (1/denom) -- within 1e-5 relative of the reference's fp64 P.
//
// Layout: one warp per row, VPL float4 per lane (cols = 128*VPL <= 1024),
// the whole row in registers (one HBM read per element, no smem staging
// needed at S <= 1024); longer rows (cols % 128 == 0, <= 16384) stream
// through a TMA ring into a CTA of W warps that shares each row
// (softmax_*_long_kernel).  Other shapes use the generic warp-per-row kernels.
#include <initializer_list>

#include "common.cuh"
#include "mt19937.h"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kBlock = 256;
#ifndef TM_SOFTMAX_WAVES
#define TM_SOFTMAX_WAVES 64  // measured: 16-64 waves beat one persistent wave by 7-8 %; 64 > 32 by 1 % (fwd, with PDL)
#endif

enum FwdMode { kPlain = 0, kSupplied = 1, kPhilox = 2 };
#ifndef TM_SOFTMAX_LONG_MIN
#define TM_SOFTMAX_LONG_MIN 1024  // rows longer than this take the TMA row-group kernels
#endif
#ifndef TM_SOFTMAX_LONG_MIN_BWD
#define TM_SOFTMAX_LONG_MIN_BWD 512  // backward: S = 1024 too (vec VPL=8 needs 154+ regs: 0.70 -> 0.84)
#endif

#ifndef TM_SOFTMAX_TWOSUM
#define TM_SOFTMAX_TWOSUM 1
#endif
#ifndef TM_SOFTMAX_EXP
#define TM_SOFTMAX_EXP 1  // 1: SFU ex2 + FMA-split exponent (+ TwoSum: 0.94 -> 0.96, P err 5e-7); 0: expf + TwoSum
#endif
// max that propagates NaN (the reference's row max: a NaN anywhere makes the
// whole row NaN, ops_reference.cpp:113-121).
__device__ __forceinline__ float fmax_nan(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float warp_max_nan(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax_nan(v, __shfl_xor_sync(kFull, v, o));
    return v;
}
// Masked scores (-inf, finfo(f32).min, anything with z - max below the
// fp32 exp range) must give exactly 0, as the reference's double exp does
// (ops_reference.cpp:111-118).  There ex2 gives e = 0 while the exponent
// split / TwoSum terms of an infinite or overflowed (z - max) are NaN or
// inf, so the result is formed by ONE saturating FMA, r = sat(e + e*corr):
// .sat maps NaN to +0 and r <= 1 holds anyway (z <= max), so a masked
// element costs no extra instruction.  The NaN rows of the reference (NaN
// anywhere, a +inf score, or an all -inf row: exp(inf - inf)) are exactly
// the rows whose NaN-propagating max is not finite; they get 1/sum = NaN
// once per row.
__device__ __forceinline__ float fma_sat(float a, float b, float c) {
    float r;
    asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float row_inv(float sum, float mx) {
    return isfinite(mx) ? 1.0f / sum : __int_as_float(0x7fffffff);
}
__device__ __forceinline__ float ex2_approx_ftz(float f) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
    return r;
}
// exp(z - mx) with the rounding error of the subtraction restored.
__device__ __forceinline__ float exp_shift(float z, float mx) {
#if TM_SOFTMAX_EXP == 1
    // 2^(d log2 e): w = d*L2E rounded, its error folded back (~2 ulp total)
    const float L2E = 1.44269502162933349609f, L2E_LO = 1.925963033500011e-08f;
    const float d = z - mx;
    const float w = d * L2E;
    const float wl = fmaf(d, L2E_LO, fmaf(d, L2E, -w));
    const float e = ex2_approx_ftz(w);
#if TM_SOFTMAX_TWOSUM
    const float bb = d - z;
    const float err = (z - (d - bb)) + (-mx - bb);  // TwoSum: (z - mx) = d + err exactly
    return fma_sat(e, fmaf(wl, 0.69314718055994531f, err), e);
#else
    return fma_sat(e, wl * 0.69314718055994531f, e);
#endif
#else
    float d = z - mx;
    float bb = d - z;
    float err = (z - (d - bb)) + (-mx - bb);  // TwoSum: (z - mx) = d + err exactly
    float e = expf(d);
    return fma_sat(e, err, e);
#endif
}

// exp_shift for two elements on the packed fp32x2 pipe (FADD2/FMUL2/FFMA2):
// every lane rounds exactly like the scalar exp_shift, so the bits are the
// same; the instruction count per element roughly halves.
#ifndef TM_SOFTMAX_PACKED
#define TM_SOFTMAX_PACKED 1
#endif
__device__ __forceinline__ float2 exp_shift2(float2 z, float mx) {
#if TM_SOFTMAX_EXP == 1
    const float2 L2E = make_float2(1.44269502162933349609f, 1.44269502162933349609f);
    const float2 L2E_LO = make_float2(1.925963033500011e-08f, 1.925963033500011e-08f);
    const float2 NMX = make_float2(-mx, -mx);
    const float2 d = __fadd2_rn(z, NMX);
    const float2 w = __fmul2_rn(d, L2E);
    const float2 wl = __ffma2_rn(d, L2E_LO, __ffma2_rn(d, L2E, make_float2(-w.x, -w.y)));
    const float2 e = make_float2(ex2_approx_ftz(w.x), ex2_approx_ftz(w.y));
    const float2 LN2 = make_float2(0.69314718055994531f, 0.69314718055994531f);
#if TM_SOFTMAX_TWOSUM
    const float2 bb = __fadd2_rn(d, make_float2(-z.x, -z.y));
    const float2 t1 = __fadd2_rn(d, make_float2(-bb.x, -bb.y));
    const float2 err = __fadd2_rn(__fadd2_rn(z, make_float2(-t1.x, -t1.y)),
                                  __fadd2_rn(NMX, make_float2(-bb.x, -bb.y)));
    const float2 c = __ffma2_rn(wl, LN2, err);
#else
    const float2 c = __fmul2_rn(wl, LN2);
#endif
    // the final FMA per lane with .sat (no packed .sat form): see fma_sat
    return make_float2(fma_sat(e.x, c.x, e.x), fma_sat(e.y, c.y, e.y));
#else
    return make_float2(exp_shift(z.x, mx), exp_shift(z.y, mx));
#endif
}

__device__ __forceinline__ float dscale(float v, double s) { return (float)((double)v * s); }

template <int VPL, int MODE>
__global__ void __launch_bounds__(kBlock) softmax_fwd_vec_kernel(
    const float* __restrict__ z, float* __restrict__ P, float* __restrict__ D,
    uint32_t* __restrict__ mask, double scale, uint64_t thresh, uint64_t seed, uint64_t offset,
    int64_t rows) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int C = VPL * 128;
    constexpr int R = VPL <= 4 ? 2 : 1;  // rows per warp iteration (loads in flight)
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t r0 = warp * R; r0 < rows; r0 += nwarps * R) {
        float4 v[R][VPL];
        uint32_t nib[R][VPL];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t r = min(r0 + i, rows - 1);  // duplicate the last row if odd
            const float4* zr = reinterpret_cast<const float4*>(z + r * C);
#pragma unroll
            for (int k = 0; k < VPL; ++k) v[i][k] = ld_stream(zr + k * 32 + lane);
            if (MODE == kSupplied) {
#pragma unroll
                for (int k = 0; k < VPL; ++k)
                    nib[i][k] = chunk_nibble(mask + ((r * C) >> 5) + k * 4, lane);
            }
        }
        float inv[R];
#pragma unroll
        for (int i = 0; i < R; ++i) {
            float mx = v[i][0].x;
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                mx = fmax_nan(mx, fmax_nan(fmax_nan(v[i][k].x, v[i][k].y),
                                           fmax_nan(v[i][k].z, v[i][k].w)));
            mx = warp_max_nan(mx);
            float acc = 0.0f;
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
#if TM_SOFTMAX_PACKED
                const float2 lo = exp_shift2(make_float2(v[i][k].x, v[i][k].y), mx);
                const float2 hi = exp_shift2(make_float2(v[i][k].z, v[i][k].w), mx);
                v[i][k] = make_float4(lo.x, lo.y, hi.x, hi.y);
#else
                v[i][k].x = exp_shift(v[i][k].x, mx);
                v[i][k].y = exp_shift(v[i][k].y, mx);
                v[i][k].z = exp_shift(v[i][k].z, mx);
                v[i][k].w = exp_shift(v[i][k].w, mx);
#endif
                acc += (v[i][k].x + v[i][k].y) + (v[i][k].z + v[i][k].w);
            }
            inv[i] = row_inv(warp_sumf(acc), mx);
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int64_t r = r0 + i;
            if (r >= rows) break;  // warp-uniform
            float4* Pr = reinterpret_cast<float4*>(P + r * C);
            float4* Dr = reinterpret_cast<float4*>(D + r * C);
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                float4 p;
                p.x = v[i][k].x * inv[i];
                p.y = v[i][k].y * inv[i];
                p.z = v[i][k].z * inv[i];
                p.w = v[i][k].w * inv[i];
                st_stream(Pr + k * 32 + lane, p);
                if (MODE == kPlain) continue;
                uint32_t bits;
                if (MODE == kPhilox) {
                    U4 rnd = philox_quad(seed,
                                         (offset + (uint64_t)(r * C + k * 128 + lane * 4)) >> 2);
                    bits = nibble4((uint64_t)rnd.x >= thresh, (uint64_t)rnd.y >= thresh,
                                   (uint64_t)rnd.z >= thresh, (uint64_t)rnd.w >= thresh);
                    store_chunk_mask(mask + ((r * C) >> 5) + k * 4, bits, lane);
                } else {
                    bits = nib[i][k];
                }
                if (D) {
                    float4 d;
                    d.x = (bits & 1u) ? dscale(p.x, scale) : 0.0f;
                    d.y = (bits & 2u) ? dscale(p.y, scale) : 0.0f;
                    d.z = (bits & 4u) ? dscale(p.z, scale) : 0.0f;
                    d.w = (bits & 8u) ? dscale(p.w, scale) : 0.0f;
                    st_stream(Dr + k * 32 + lane, d);
                }
            }
        }
    }
}

// Backward.  DROP: dP = mask ? dD*scale : 0 (else dP = dD, plain softmax);
// WRITE_D: recomputed D = mask ? P*scale : 0.
template <int VPL, bool DROP, bool WRITE_D>
__global__ void __launch_bounds__(kBlock) softmax_bwd_vec_kernel(
    const float* __restrict__ dD, const float* __restrict__ P, const uint32_t* __restrict__ mask,
    double scale, float* __restrict__ dZ, float* __restrict__ D, int64_t rows) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int C = VPL * 128;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const float4* gr = reinterpret_cast<const float4*>(dD + r * C);
        const float4* pr = reinterpret_cast<const float4*>(P + r * C);
        float4 g[VPL], p[VPL];
        uint32_t nib[VPL];
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            g[k] = ld_stream(gr + k * 32 + lane);
            p[k] = ld_stream(pr + k * 32 + lane);
            if (DROP) nib[k] = chunk_nibble(mask + ((r * C) >> 5) + k * 4, lane);
        }
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            if (DROP) {  // dropout_backward: F32-stored dP (ops_reference.cpp:155-161)
                g[k].x = (nib[k] & 1u) ? dscale(g[k].x, scale) : 0.0f;
                g[k].y = (nib[k] & 2u) ? dscale(g[k].y, scale) : 0.0f;
                g[k].z = (nib[k] & 4u) ? dscale(g[k].z, scale) : 0.0f;
                g[k].w = (nib[k] & 8u) ? dscale(g[k].w, scale) : 0.0f;
            }
            acc = fma((double)g[k].x, (double)p[k].x, acc);
            acc = fma((double)g[k].y, (double)p[k].y, acc);
            acc = fma((double)g[k].z, (double)p[k].z, acc);
            acc = fma((double)g[k].w, (double)p[k].w, acc);
        }
        const double s = warp_sum(acc);
        float4* zr = reinterpret_cast<float4*>(dZ + r * C);
        float4* Dr = reinterpret_cast<float4*>(D + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            float4 o;
            o.x = (float)((double)p[k].x * ((double)g[k].x - s));
            o.y = (float)((double)p[k].y * ((double)g[k].y - s));
            o.z = (float)((double)p[k].z * ((double)g[k].z - s));
            o.w = (float)((double)p[k].w * ((double)g[k].w - s));
            st_stream(zr + k * 32 + lane, o);
            if (WRITE_D) {
                float4 d;
                d.x = (nib[k] & 1u) ? dscale(p[k].x, scale) : 0.0f;
                d.y = (nib[k] & 2u) ? dscale(p[k].y, scale) : 0.0f;
                d.z = (nib[k] & 4u) ? dscale(p[k].z, scale) : 0.0f;
                d.w = (nib[k] & 8u) ? dscale(p[k].w, scale) : 0.0f;
                st_stream(Dr + k * 32 + lane, d);
            }
        }
    }
}

// ------------------------------------------------------------- long rows
// S > 1024 (the paper's sweep reaches S = 3072): one CTA =
// one row group of W warps, persistent over rows r = blockIdx.x + i*gridDim.x.
// The rows stream into a shallow shared-memory ring by TMA bulk
// copies (cp.async.bulk, one mbarrier per stage; thread 0 issues): the bytes
// in flight per SM are bounded by shared memory, not by the registers that
// hold a row -- a register-only row group keeps ~64 KB per SM in flight and
// reaches 0.58-0.75 of the copy peak at S = 2048-8192.  The row's 128-column
// chunks are dealt round-robin to the warps (warp w: chunks w, w+W, ...; at
// most VPL each), read from the stage into registers, and the row max / sum /
// dot are warp shuffles plus ONE exchange of the W warp partials through
// shared memory (__syncthreads; partials combined in warp order in every
// thread, slots alternating by row parity).  The first exchange of a row also
// proves every warp has read the stage, so thread 0 refills it right there.
// Still one HBM read and one write per element; numerics as the vec kernels
// (the plain and dropout P are bitwise equal).
// ring depth per direction (fewer when a row is too long for the smem
// budget): measured, occupancy (CTAs per SM) is worth more than depth
#ifndef TM_SMXL_FWD_STAGES
#define TM_SMXL_FWD_STAGES 2
#endif
#ifndef TM_SMXL_BWD_STAGES
#define TM_SMXL_BWD_STAGES 1  // A/B: 1 stage 0.92/0.86/0.91/0.86 at S = 2048/3072/4096/8192 vs 0.87/0.87/0.87/0.67 with 2
#endif
constexpr size_t kLongRingBytes = 192 * 1024;

__device__ __forceinline__ void ring_init(uint64_t* full, int ns) {
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
}

template <int W, int VPL, int MODE>
__global__ void __launch_bounds__(W * 32) softmax_fwd_long_kernel(
    const float* __restrict__ z, float* __restrict__ P, float* __restrict__ D,
    uint32_t* __restrict__ mask, double scale, uint64_t thresh, uint64_t seed, uint64_t offset,
    int64_t rows, int nch, int ns) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    const float4* ring = reinterpret_cast<const float4*>(dsm + 128);
    __shared__ float red[2][2][W];  // [row parity][max, sum][warp]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t C = (int64_t)nch * 128;
    const uint32_t row_bytes = (uint32_t)C * 4u;
    ring_init(full, ns);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            const int64_t r = blockIdx.x + (int64_t)s * gridDim.x;
            if (r < rows) {
                mbar_expect_tx(&full[s], row_bytes);
                bulk_g2s((void*)(ring + (size_t)s * (C / 4)), z + r * C, row_bytes, &full[s]);
            }
        }
    }
    int it = 0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
        const int st = it % ns;
        uint32_t nib[VPL];
        if (MODE == kSupplied) {  // mask words straight from global (1/32 of the bytes)
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                if (w + k * W < nch) nib[k] = chunk_nibble(mask + ((r * C) >> 5) + (w + k * W) * 4, lane);
        }
        mbar_wait(&full[st], (uint32_t)((it / ns) & 1));
        const float4* sp = ring + (size_t)st * (C / 4);
        float4 v[VPL];
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const int c = w + k * W;
            if (c < nch) {
                v[k] = sp[c * 32 + lane];
                mx = fmax_nan(mx, fmax_nan(fmax_nan(v[k].x, v[k].y), fmax_nan(v[k].z, v[k].w)));
            }
        }
        const int par = it & 1;
        mx = warp_max_nan(mx);
        if (lane == 0) red[par][0][w] = mx;
        __syncthreads();  // every warp has read stage st: refill it
        if (threadIdx.x == 0) {
            const int64_t rn = r + (int64_t)ns * gridDim.x;
            if (rn < rows) {
                fence_proxy_async_smem();
                mbar_expect_tx(&full[st], row_bytes);
                bulk_g2s((void*)(ring + (size_t)st * (C / 4)), z + rn * C, row_bytes, &full[st]);
            }
        }
        mx = red[par][0][0];
#pragma unroll
        for (int i = 1; i < W; ++i) mx = fmax_nan(mx, red[par][0][i]);
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            if (w + k * W >= nch) continue;
#if TM_SOFTMAX_PACKED
            const float2 lo = exp_shift2(make_float2(v[k].x, v[k].y), mx);
            const float2 hi = exp_shift2(make_float2(v[k].z, v[k].w), mx);
            v[k] = make_float4(lo.x, lo.y, hi.x, hi.y);
#else
            v[k] = make_float4(exp_shift(v[k].x, mx), exp_shift(v[k].y, mx),
                               exp_shift(v[k].z, mx), exp_shift(v[k].w, mx));
#endif
            acc += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        }
        acc = warp_sumf(acc);
        if (lane == 0) red[par][1][w] = acc;
        __syncthreads();
        float sum = red[par][1][0];
#pragma unroll
        for (int i = 1; i < W; ++i) sum += red[par][1][i];
        const float inv = row_inv(sum, mx);
        float4* Pr = reinterpret_cast<float4*>(P + r * C);
        float4* Dr = reinterpret_cast<float4*>(D + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const int c = w + k * W;
            if (c >= nch) continue;
            const float4 p = make_float4(v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
            st_stream(Pr + c * 32 + lane, p);
            if (MODE == kPlain) continue;
            uint32_t bits;
            if (MODE == kPhilox) {
                U4 rnd = philox_quad(seed, (offset + (uint64_t)(r * C + c * 128 + lane * 4)) >> 2);
                bits = nibble4((uint64_t)rnd.x >= thresh, (uint64_t)rnd.y >= thresh,
                               (uint64_t)rnd.z >= thresh, (uint64_t)rnd.w >= thresh);
                store_chunk_mask(mask + ((r * C) >> 5) + c * 4, bits, lane);
            } else {
                bits = nib[k];
            }
            if (D) {
                float4 d;
                d.x = (bits & 1u) ? dscale(p.x, scale) : 0.0f;
                d.y = (bits & 2u) ? dscale(p.y, scale) : 0.0f;
                d.z = (bits & 4u) ? dscale(p.z, scale) : 0.0f;
                d.w = (bits & 8u) ? dscale(p.w, scale) : 0.0f;
                st_stream(Dr + c * 32 + lane, d);
            }
        }
    }
}

template <int W, int VPL, bool DROP, bool WRITE_D>
__global__ void __launch_bounds__(W * 32) softmax_bwd_long_kernel(
    const float* __restrict__ dD, const float* __restrict__ P, const uint32_t* __restrict__ mask,
    double scale, float* __restrict__ dZ, float* __restrict__ D, int64_t rows, int nch, int ns) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    const float4* ring = reinterpret_cast<const float4*>(dsm + 128);  // [stage][dD, P][C/4]
    __shared__ double red[2][W];  // [row parity][warp]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t C = (int64_t)nch * 128;
    const uint32_t row_bytes = (uint32_t)C * 4u;
    auto issue = [&](int64_t r, int s) {
        mbar_expect_tx(&full[s], 2 * row_bytes);
        bulk_g2s((void*)(ring + (size_t)(2 * s) * (C / 4)), dD + r * C, row_bytes, &full[s]);
        bulk_g2s((void*)(ring + (size_t)(2 * s + 1) * (C / 4)), P + r * C, row_bytes, &full[s]);
    };
    ring_init(full, ns);
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) {
            const int64_t r = blockIdx.x + (int64_t)s * gridDim.x;
            if (r < rows) issue(r, s);
        }
    }
    int it = 0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
        const int st = it % ns;
        uint32_t nib[VPL];
        if (DROP) {
#pragma unroll
            for (int k = 0; k < VPL; ++k)
                if (w + k * W < nch) nib[k] = chunk_nibble(mask + ((r * C) >> 5) + (w + k * W) * 4, lane);
        }
        mbar_wait(&full[st], (uint32_t)((it / ns) & 1));
        const float4* gs = ring + (size_t)(2 * st) * (C / 4);
        const float4* ps = ring + (size_t)(2 * st + 1) * (C / 4);
        float4 gv[VPL], p[VPL];
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const int c = w + k * W;
            if (c >= nch) continue;
            gv[k] = gs[c * 32 + lane];
            p[k] = ps[c * 32 + lane];
            if (DROP) {  // dropout_backward: F32-stored dP (ops_reference.cpp:155-161)
                gv[k].x = (nib[k] & 1u) ? dscale(gv[k].x, scale) : 0.0f;
                gv[k].y = (nib[k] & 2u) ? dscale(gv[k].y, scale) : 0.0f;
                gv[k].z = (nib[k] & 4u) ? dscale(gv[k].z, scale) : 0.0f;
                gv[k].w = (nib[k] & 8u) ? dscale(gv[k].w, scale) : 0.0f;
            }
            acc = fma((double)gv[k].x, (double)p[k].x, acc);
            acc = fma((double)gv[k].y, (double)p[k].y, acc);
            acc = fma((double)gv[k].z, (double)p[k].z, acc);
            acc = fma((double)gv[k].w, (double)p[k].w, acc);
        }
        const int par = it & 1;
        acc = warp_sum(acc);
        if (lane == 0) red[par][w] = acc;
        __syncthreads();  // every warp has read stage st: refill it
        if (threadIdx.x == 0) {
            const int64_t rn = r + (int64_t)ns * gridDim.x;
            if (rn < rows) {
                fence_proxy_async_smem();
                issue(rn, st);
            }
        }
        double s = red[par][0];
#pragma unroll
        for (int i = 1; i < W; ++i) s += red[par][i];
        float4* zr = reinterpret_cast<float4*>(dZ + r * C);
        float4* Dr = reinterpret_cast<float4*>(D + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const int c = w + k * W;
            if (c >= nch) continue;
            float4 o;
            o.x = (float)((double)p[k].x * ((double)gv[k].x - s));
            o.y = (float)((double)p[k].y * ((double)gv[k].y - s));
            o.z = (float)((double)p[k].z * ((double)gv[k].z - s));
            o.w = (float)((double)p[k].w * ((double)gv[k].w - s));
            st_stream(zr + c * 32 + lane, o);
            if (WRITE_D) {
                float4 d;
                d.x = (nib[k] & 1u) ? dscale(p[k].x, scale) : 0.0f;
                d.y = (nib[k] & 2u) ? dscale(p[k].y, scale) : 0.0f;
                d.z = (nib[k] & 4u) ? dscale(p[k].z, scale) : 0.0f;
                d.w = (nib[k] & 8u) ? dscale(p[k].w, scale) : 0.0f;
                st_stream(Dr + c * 32 + lane, d);
            }
        }
    }
}

// ------------------------------------- the reference's mask stream, fused
// softmax -> dropout_recompute forward whose mask is the reference's own
// BoolMask::bernoulli_keep stream (std::mt19937_64, tensor.cpp:186-203)
// GENERATED INSIDE the kernel instead of by a separate pass (§3a computes
// the same bits in mt_keep_kernel).  One CTA per 2^19-output chunk of the
// stream, warp-specialised:
//   * 4 generator warps run the chunk's recurrence from its jumped start
//     state (128 outputs per step, 312-word ring in smem, a named barrier
//     of the 128 generator threads per step), temper, compare with the
//     integer threshold and ballot one mask word per warp and step into a
//     kMtSlots-deep smem ring of slots of 4 rows (4C outputs, C/32 steps);
//   * 4 consumer warps, one row of the slot each, run softmax_fwd_vec_kernel's
//     per-row math (the row's loads issued before the slot wait), read their
//     mask nibbles from the ring, store P, D and the row's mask words (the
//     stash) to HBM;
//   * full[s] (4 generator arrivals) / empty[s] (4 consumer arrivals)
//     mbarriers hand the slots over.
// The chunk's generation is sequential (2^19 / 128 steps), so the kernel is
// only as fast as the chunks that run CONCURRENTLY: 256-thread CTAs within
// 64 registers give 4 CTAs per SM, i.e. all 512 chunks of a 2^28-element
// mask resident at once (2 per SM -- the first version's 384-thread CTAs at
// 80 registers -- ran two waves: 1.07 ms vs 0.58 + 0.47 for the passes).
// Needs C in {128, 256, 512, 1024}, e_begin % 2^19 == 0 and rows*C % 4C
// == 0 (the launcher falls back to the separate passes otherwise).  Bits, P
// and D are exactly those of mt_keep_kernel + the supplied-mask forward.
constexpr int kMtGenWarps = 4, kMtConsWarps = 4;
constexpr int kMtThreads = 32 * (kMtGenWarps + kMtConsWarps);
constexpr int kMtSlots = 8;
#ifndef TM_MTGEN_MINB
#define TM_MTGEN_MINB 4
#endif

template <int VPL>
__global__ void __launch_bounds__(kMtThreads, TM_MTGEN_MINB) softmax_fwd_mtgen_kernel(
    const float* __restrict__ z, float* __restrict__ P, float* __restrict__ D,
    uint32_t* __restrict__ mask, const uint64_t* __restrict__ states, double scale,
    uint64_t xmin, int64_t rows) {
    grid_dep_wait();  // PDL: predecessor (the chunk-state jump) complete and visible
    grid_dep_launch();
    constexpr int C = VPL * 128;
    constexpr int kSlotSteps = kMtConsWarps * C / 128;  // steps per slot (one row per consumer)
    constexpr int kSlotWords = kSlotSteps * 4;
    constexpr int kRowsPerChunk = (int)(kMtChunk / C);
    __shared__ uint64_t ring[512];
    __shared__ uint32_t mring[kMtSlots * kSlotWords];
    __shared__ __align__(8) uint64_t full[kMtSlots], empty[kMtSlots];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t r_begin = (int64_t)blockIdx.x * kRowsPerChunk;
    const int64_t r_end = min(rows, r_begin + kRowsPerChunk);
    const int nslots = (int)((r_end - r_begin) / kMtConsWarps);
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMtSlots; ++s) {
            mbar_init(&full[s], kMtGenWarps);
            mbar_init(&empty[s], kMtConsWarps);
        }
        mbar_fence_init();
    }
    if (warp < kMtGenWarps) {
        const uint64_t* st = states + (size_t)blockIdx.x * kMtN;
        for (int i = threadIdx.x; i < (int)kMtN; i += 32 * kMtGenWarps) ring[i] = st[i];
    }
    __syncthreads();
    if (warp < kMtGenWarps) {
        // ---- generator: as mt_keep_kernel, one ballot word per warp and step
        const int tid = threadIdx.x;
        int a312[4], a311[4], a156[4], aw[4];
#pragma unroll
        for (int ph = 0; ph < 4; ++ph) {
            const int j = ph * 128 + kMtN + tid;  // sequence index mod 512
            a312[ph] = (j - 312) & 511;
            a311[ph] = (j - 311) & 511;
            a156[ph] = (j - 156) & 511;
            aw[ph] = j & 511;
        }
        for (int sl = 0; sl < nslots; ++sl) {
            const int s = sl % kMtSlots;
            if (sl >= kMtSlots) {  // the consumers are done with this slot's previous use
                if (lane == 0) mbar_wait(&empty[s], (uint32_t)(((sl / kMtSlots) - 1) & 1));
                __syncwarp();
            }
            uint32_t* words = mring + s * kSlotWords;
#pragma unroll 1
            for (int t4 = 0; t4 < kSlotSteps; t4 += 4) {  // kSlotSteps % 4 == 0
#pragma unroll
                for (int ph = 0; ph < 4; ++ph) {
                    const uint64_t w = mt_next_word(ring[a312[ph]], ring[a311[ph]], ring[a156[ph]]);
                    ring[aw[ph]] = w;
                    group_bar(1, 32 * kMtGenWarps);  // w visible to the next step
                    const uint32_t word = __ballot_sync(kFull, mt_keep(w, xmin));
                    if (lane == 0) words[(t4 + ph) * 4 + warp] = word;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        }
        return;
    }
    // ---- consumers: warp cw takes row cw of every slot
    const int cw = warp - kMtGenWarps;
    for (int sl = 0; sl < nslots; ++sl) {
        const int s = sl % kMtSlots;
        const int64_t r = r_begin + (int64_t)sl * kMtConsWarps + cw;
        float4 v[VPL];
        const float4* zr = reinterpret_cast<const float4*>(z + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) v[k] = ld_stream(zr + k * 32 + lane);
        if (lane == 0) mbar_wait(&full[s], (uint32_t)((sl / kMtSlots) & 1));
        __syncwarp();
        const uint32_t* words = mring + s * kSlotWords + cw * (C / 32);  // this row's words
        float mx = v[0].x;
#pragma unroll
        for (int k = 0; k < VPL; ++k)
            mx = fmax_nan(mx, fmax_nan(fmax_nan(v[k].x, v[k].y), fmax_nan(v[k].z, v[k].w)));
        mx = warp_max_nan(mx);
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
#if TM_SOFTMAX_PACKED
            const float2 lo = exp_shift2(make_float2(v[k].x, v[k].y), mx);
            const float2 hi = exp_shift2(make_float2(v[k].z, v[k].w), mx);
            v[k] = make_float4(lo.x, lo.y, hi.x, hi.y);
#else
            v[k] = make_float4(exp_shift(v[k].x, mx), exp_shift(v[k].y, mx),
                               exp_shift(v[k].z, mx), exp_shift(v[k].w, mx));
#endif
            acc += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        }
        const float inv = row_inv(warp_sumf(acc), mx);
        float4* Pr = reinterpret_cast<float4*>(P + r * C);
        float4* Dr = reinterpret_cast<float4*>(D + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float4 p = make_float4(v[k].x * inv, v[k].y * inv, v[k].z * inv, v[k].w * inv);
            st_stream(Pr + k * 32 + lane, p);
            if (D) {  // the chunk_nibble layout: word k*4 + lane/8, nibble lane%8
                const uint32_t bits = (words[k * 4 + (lane >> 3)] >> (4 * (lane & 7))) & 0xfu;
                float4 d;
                d.x = (bits & 1u) ? dscale(p.x, scale) : 0.0f;
                d.y = (bits & 2u) ? dscale(p.y, scale) : 0.0f;
                d.z = (bits & 4u) ? dscale(p.z, scale) : 0.0f;
                d.w = (bits & 8u) ? dscale(p.w, scale) : 0.0f;
                st_stream(Dr + k * 32 + lane, d);
            }
        }
        if (lane < C / 32) st_stream(mask + ((r * C) >> 5) + lane, words[lane]);  // the stash
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }
}

// ---------------------------------------------------------------- generic
__device__ __forceinline__ bool mask_bit(const uint32_t* mask, int64_t i) {
    return (__ldg(mask + (i >> 5)) >> (i & 31)) & 1u;
}

__global__ void __launch_bounds__(kBlock) softmax_fwd_generic_kernel(
    const float* __restrict__ z, float* __restrict__ P, float* __restrict__ D,
    uint32_t* __restrict__ mask, int mode, double scale, uint64_t thresh, uint64_t seed,
    uint64_t offset, int64_t rows, int64_t C) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
        const float* zr = z + r * C;
        float mx = -INFINITY;
        for (int64_t j = lane; j < C; j += 32) mx = fmax_nan(mx, zr[j]);
        mx = warp_max_nan(mx);
        double acc = 0.0;
        for (int64_t j = lane; j < C; j += 32) acc += (double)exp_shift(zr[j], mx);
        const double inv = isfinite(mx) ? 1.0 / warp_sum(acc) : __longlong_as_double(0x7ff8000000000000ll);
        for (int64_t j = lane; j < C; j += 32) {
            const int64_t i = r * C + j;
            float p = (float)((double)exp_shift(zr[j], mx) * inv);
            P[i] = p;
            if (mode == kPlain) continue;
            const bool keep = mode == kPhilox
                                  ? (uint64_t)philox_at(seed, offset + (uint64_t)i) >= thresh
                                  : mask_bit(mask, i);
            if (D) D[i] = keep ? dscale(p, scale) : 0.0f;
        }
        if (mode == kPhilox) {
            // The row's mask words, whole words per lane (no atomics): a word
            // shared with the neighbouring row is written by both warps with
            // the same value -- its bits depend only on (seed, index).
            const int64_t n = rows * C;
            for (int64_t wd = (r * C) >> 5, w1 = (r * C + C - 1) >> 5; wd <= w1; wd += 32) {
                if (wd + lane > w1) break;
                const int64_t i0 = (wd + lane) * 32;
                uint32_t word = 0;
                uint64_t qi = ~0ull;
                U4 q{};
                for (int b = 0; b < 32 && i0 + b < n; ++b) {
                    const uint64_t gi = offset + (uint64_t)(i0 + b);
                    if ((gi >> 2) != qi) {
                        qi = gi >> 2;
                        q = philox_quad(seed, qi);
                    }
                    const uint32_t x = (gi & 3) == 0 ? q.x : (gi & 3) == 1 ? q.y : (gi & 3) == 2 ? q.z : q.w;
                    word |= (uint32_t)((uint64_t)x >= thresh) << b;
                }
                mask[wd + lane] = word;
            }
        }
    }
}

__global__ void __launch_bounds__(kBlock) softmax_bwd_generic_kernel(
    const float* __restrict__ dD, const float* __restrict__ P, const uint32_t* __restrict__ mask,
    int drop, double scale, float* __restrict__ dZ, float* __restrict__ D, int64_t rows,
    int64_t C) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    for (int64_t r = warp; r < rows; r += nwarps) {
        double acc = 0.0;
        for (int64_t j = lane; j < C; j += 32) {
            const int64_t i = r * C + j;
            float g = dD[i];
            if (drop) g = mask_bit(mask, i) ? dscale(g, scale) : 0.0f;
            acc = fma((double)g, (double)P[i], acc);
        }
        const double s = warp_sum(acc);
        for (int64_t j = lane; j < C; j += 32) {
            const int64_t i = r * C + j;
            float g = dD[i];
            const bool keep = drop ? mask_bit(mask, i) : true;
            if (drop) g = keep ? dscale(g, scale) : 0.0f;
            dZ[i] = (float)((double)P[i] * ((double)g - s));
            if (D) D[i] = keep ? dscale(P[i], scale) : 0.0f;
        }
    }
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <int MODE>
cudaError_t fwd_vec(int vpl, const float* z, float* P, float* D, uint32_t* mask, double scale,
                    uint64_t thresh, uint64_t seed, uint64_t offset, int64_t rows,
                    cudaStream_t st) {
#define TB_FWD_CASE(V)                                                                       \
    case V: {                                                                                \
        auto k = softmax_fwd_vec_kernel<V, MODE>;                                            \
        int grid = grid_for((const void*)k, kBlock, 0, (rows * 32 + kBlock - 1) / kBlock, 0, TM_SOFTMAX_WAVES);  \
        launch(k, grid, kBlock, 0, st)(z, P, D, mask, scale, thresh, seed, offset, rows);        \
        break;                                                                               \
    }
    switch (vpl) {
        TB_FWD_CASE(1)
        TB_FWD_CASE(2)
        TB_FWD_CASE(3)
        TB_FWD_CASE(4)
        TB_FWD_CASE(5)
        TB_FWD_CASE(6)
        TB_FWD_CASE(7)
        TB_FWD_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef TB_FWD_CASE
    return cudaGetLastError();
}

template <bool DROP, bool WRITE_D>
cudaError_t bwd_vec(int vpl, const float* dD, const float* P, const uint32_t* mask, double scale,
                    float* dZ, float* D, int64_t rows, cudaStream_t st) {
#define TB_BWD_CASE(V)                                                                       \
    case V: {                                                                                \
        auto k = softmax_bwd_vec_kernel<V, DROP, WRITE_D>;                                   \
        int grid = grid_for((const void*)k, kBlock, 0, (rows * 32 + kBlock - 1) / kBlock, 0, TM_SOFTMAX_WAVES);  \
        launch(k, grid, kBlock, 0, st)(dD, P, mask, scale, dZ, D, rows);                         \
        break;                                                                               \
    }
    switch (vpl) {
        TB_BWD_CASE(1)
        TB_BWD_CASE(2)
        TB_BWD_CASE(3)
        TB_BWD_CASE(4)
        TB_BWD_CASE(5)
        TB_BWD_CASE(6)
        TB_BWD_CASE(7)
        TB_BWD_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef TB_BWD_CASE
    return cudaGetLastError();
}

bool vec_ok(int64_t cols, uint64_t offset, std::initializer_list<const void*> ptrs,
            int64_t max_cols = TM_SOFTMAX_LONG_MIN) {
    if (cols % 128 != 0 || cols > 1024 || cols > max_cols || cols == 0 || (offset & 3u))
        return false;
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return false;
    return true;
}

// long rows: cols % 128 == 0, TM_SOFTMAX_LONG_MIN < cols <= 16384, with
// VPL = 4 chunks per warp (W = nch/4 rounded up to a power of two, <= 16) or
// VPL = 8 at W = 16
constexpr int kLongMaxCols = 16 * 8 * 128;
bool long_ok(int64_t cols, uint64_t offset, std::initializer_list<const void*> ptrs,
             int64_t min_cols = TM_SOFTMAX_LONG_MIN) {
    if (cols % 128 != 0 || cols <= min_cols || cols > kLongMaxCols || (offset & 3u))
        return false;
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return false;
    return true;
}
// (W, VPL) code W*10 + VPL with W*VPL >= nch: VPL (4 or 8) chunks per warp,
// W the smallest power of two that covers the row (<= 16).  Measured at
// 2^27 elements (tools/long_rows_bench.py): the forward wants more work per
// warp between the row's barriers (VPL 8: S = 2048/3072/8192 at 0.90/0.87/
// 0.86 of the copy peak vs 0.83/0.77/0.80 with VPL 4), the backward -- twice
// the registers and smem per row -- more CTAs per SM (VPL 4).
#ifndef TM_SMXL_FWD_VPL
#define TM_SMXL_FWD_VPL 8
#endif
#ifndef TM_SMXL_BWD_VPL
#define TM_SMXL_BWD_VPL 4
#endif
// W from {2, 3, 4, 6, 8, 12, 16}: the common S (1536, 2048, 3072, 4096, 6144,
// 8192, 12288) fill every chunk slot of every warp.  A/B (2^27 elements):
// backward S = 1536/3072/6144 at 0.89/0.88/0.89 vs 0.88/0.86/0.80 with
// W in {2,4,8,16}; forward S = 6144/12288 0.87/0.80 vs 0.80/0.76, but S =
// 3072 0.83 with W = 3 vs 0.86 with W = 4 (6 of 8 slots): the forward skips
// W = 3 (its CTAs are smem-limited per SM, so more warps per CTA win).
inline int long_cfg(int nch, int vpl, bool allow3) {
    static const int kW[] = {2, 3, 4, 6, 8, 12, 16};
    for (int w : kW) {
        if (w == 3 && !allow3) continue;
        if (w * vpl >= nch) return w * 10 + vpl;
    }
    return 168;  // 16 warps x 8 chunks: S <= 16384
}
inline int long_stages(int64_t cols, int tensors) {
    const size_t stage = (size_t)tensors * cols * sizeof(float);
    const int ns = (int)(kLongRingBytes / stage);
    const int want = tensors == 1 ? TM_SMXL_FWD_STAGES : TM_SMXL_BWD_STAGES;
    return ns < 1 ? 1 : ns > want ? want : ns;
}
inline size_t long_smem(int64_t cols, int tensors) {
    return 128 + (size_t)long_stages(cols, tensors) * tensors * cols * sizeof(float);
}

template <int MODE>
cudaError_t fwd_long(int nch, const float* z, float* P, float* D, uint32_t* mask, double scale,
                     uint64_t thresh, uint64_t seed, uint64_t offset, int64_t rows,
                     cudaStream_t st) {
    const size_t smem = long_smem((int64_t)nch * 128, 1);
#define TB_FWDL_CASE(W, V)                                                                    \
    case W * 10 + V: {                                                                        \
        auto k = softmax_fwd_long_kernel<W, V, MODE>;                                         \
        int grid = grid_for((const void*)k, W * 32, smem, rows);                              \
        launch(k, grid, W * 32, smem, st)(z, P, D, mask, scale, thresh, seed, offset, rows, nch, \
                                          long_stages((int64_t)nch * 128, 1));                \
        break;                                                                                \
    }
    switch (long_cfg(nch, TM_SMXL_FWD_VPL, false)) {
#if TM_SMXL_FWD_VPL == 8
        TB_FWDL_CASE(2, 8)
        TB_FWDL_CASE(4, 8)
        TB_FWDL_CASE(6, 8)
        TB_FWDL_CASE(8, 8)
        TB_FWDL_CASE(12, 8)
#else
        TB_FWDL_CASE(2, 4)
        TB_FWDL_CASE(3, 4)
        TB_FWDL_CASE(4, 4)
        TB_FWDL_CASE(6, 4)
        TB_FWDL_CASE(8, 4)
        TB_FWDL_CASE(12, 4)
        TB_FWDL_CASE(16, 4)
#endif
        TB_FWDL_CASE(16, 8)
        default: return cudaErrorInvalidValue;
    }
#undef TB_FWDL_CASE
    return cudaGetLastError();
}

template <bool DROP, bool WRITE_D>
cudaError_t bwd_long(int nch, const float* dD, const float* P, const uint32_t* mask, double scale,
                     float* dZ, float* D, int64_t rows, cudaStream_t st) {
    const size_t smem = long_smem((int64_t)nch * 128, 2);
#define TB_BWDL_CASE(W, V)                                                                    \
    case W * 10 + V: {                                                                        \
        auto k = softmax_bwd_long_kernel<W, V, DROP, WRITE_D>;                                \
        int grid = grid_for((const void*)k, W * 32, smem, rows);                              \
        launch(k, grid, W * 32, smem, st)(dD, P, mask, scale, dZ, D, rows, nch,               \
                                          long_stages((int64_t)nch * 128, 2));                \
        break;                                                                                \
    }
    switch (long_cfg(nch, TM_SMXL_BWD_VPL, true)) {
#if TM_SMXL_BWD_VPL == 8
        TB_BWDL_CASE(2, 8)
        TB_BWDL_CASE(3, 8)
        TB_BWDL_CASE(4, 8)
        TB_BWDL_CASE(6, 8)
        TB_BWDL_CASE(8, 8)
        TB_BWDL_CASE(12, 8)
#else
        TB_BWDL_CASE(2, 4)
        TB_BWDL_CASE(3, 4)
        TB_BWDL_CASE(4, 4)
        TB_BWDL_CASE(6, 4)
        TB_BWDL_CASE(8, 4)
        TB_BWDL_CASE(12, 4)
        TB_BWDL_CASE(16, 4)
#endif
        TB_BWDL_CASE(16, 8)
        default: return cudaErrorInvalidValue;
    }
#undef TB_BWDL_CASE
    return cudaGetLastError();
}

int generic_grid(const void* k, int64_t rows) {
    return grid_for(k, kBlock, 0, (rows * 32 + kBlock - 1) / kBlock);
}

}  // namespace

cudaError_t launch_softmax_fwd(const float* z, float* P, int64_t rows, int64_t cols,
                               cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (vec_ok(cols, 0, {z, P}))
        return fwd_vec<kPlain>((int)(cols / 128), z, P, nullptr, nullptr, 1.0, 0, 0, 0, rows, st);
    if (long_ok(cols, 0, {z, P}))
        return fwd_long<kPlain>((int)(cols / 128), z, P, nullptr, nullptr, 1.0, 0, 0, 0, rows, st);
    launch(softmax_fwd_generic_kernel, generic_grid((const void*)softmax_fwd_generic_kernel, rows),
                                 kBlock, 0, st)(z, P, nullptr, nullptr, kPlain, 1.0, 0, 0, 0,
                                                  rows, cols);
    return cudaGetLastError();
}

cudaError_t launch_softmax_bwd(const float* dP, const float* P, float* dZ, int64_t rows,
                               int64_t cols, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (vec_ok(cols, 0, {dP, P, dZ}, TM_SOFTMAX_LONG_MIN_BWD))
        return bwd_vec<false, false>((int)(cols / 128), dP, P, nullptr, 1.0, dZ, nullptr, rows,
                                     st);
    if (long_ok(cols, 0, {dP, P, dZ}, TM_SOFTMAX_LONG_MIN_BWD))
        return bwd_long<false, false>((int)(cols / 128), dP, P, nullptr, 1.0, dZ, nullptr, rows,
                                      st);
    launch(softmax_bwd_generic_kernel, generic_grid((const void*)softmax_bwd_generic_kernel, rows),
                                 kBlock, 0, st)(dP, P, nullptr, 0, 1.0, dZ, nullptr, rows,
                                                  cols);
    return cudaGetLastError();
}

cudaError_t launch_softmax_dropout_fwd(const float* z, double scale, uint64_t thresh, int philox,
                                       uint32_t* mask, uint64_t seed, uint64_t offset, float* P,
                                       float* D, int64_t rows, int64_t cols, cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (vec_ok(cols, offset, {z, P, D, mask})) {
        const int vpl = (int)(cols / 128);
        return philox ? fwd_vec<kPhilox>(vpl, z, P, D, mask, scale, thresh, seed, offset, rows, st)
                      : fwd_vec<kSupplied>(vpl, z, P, D, mask, scale, thresh, seed, offset, rows,
                                           st);
    }
    if (long_ok(cols, offset, {z, P, D, mask})) {
        const int nch = (int)(cols / 128);
        return philox ? fwd_long<kPhilox>(nch, z, P, D, mask, scale, thresh, seed, offset, rows, st)
                      : fwd_long<kSupplied>(nch, z, P, D, mask, scale, thresh, seed, offset, rows,
                                            st);
    }
    launch(softmax_fwd_generic_kernel, generic_grid((const void*)softmax_fwd_generic_kernel, rows),
                                 kBlock, 0, st)(z, P, D, mask, philox ? kPhilox : kSupplied,
                                                  scale, thresh, seed, offset, rows, cols);
    return cudaGetLastError();
}

cudaError_t launch_softmax_dropout_fwd_mt(const float* z, double p, uint64_t seed,
                                          uint64_t e_begin, uint32_t* mask, float* P, float* D,
                                          int64_t rows, int64_t cols, void* ws, size_t ws_bytes,
                                          cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    const int64_t n = rows * cols;
    const double scale = 1.0 / (1.0 - p);
    const bool fused = (cols == 128 || cols == 256 || cols == 512 || cols == 1024) &&
                       e_begin % (uint64_t)kMtChunk == 0 && rows % kMtConsWarps == 0 &&
                       vec_ok(cols, 0, {z, P, D, mask});
    if (!fused) {  // the separate passes: generation, then the supplied-mask forward
        cudaError_t e = launch_mt_keep_bits(seed, p, e_begin, n, mask, ws, ws_bytes, st);
        if (e != cudaSuccess) return e;
        return launch_softmax_dropout_fwd(z, scale, 0, 0, mask, 0, 0, P, D, rows, cols, st);
    }
    const uint64_t* states = nullptr;
    cudaError_t e = launch_mt_chunk_states(seed, e_begin, n, ws, ws_bytes, &states, st);
    if (e != cudaSuccess) return e;
    const unsigned nchunks = (unsigned)((n + kMtChunk - 1) / kMtChunk);
    const uint64_t xmin = mt_keep_threshold(p);
#define TB_MTG_CASE(V)                                                                         \
    case V:                                                                                    \
        launch(softmax_fwd_mtgen_kernel<V>, nchunks, kMtThreads, 0, st)(z, P, D, mask, states,  \
                                                                     scale, xmin, rows);       \
        break;
    switch (cols / 128) {
        TB_MTG_CASE(1)
        TB_MTG_CASE(2)
        TB_MTG_CASE(4)
        TB_MTG_CASE(8)
        default: return cudaErrorInvalidValue;
    }
#undef TB_MTG_CASE
    return cudaGetLastError();
}

cudaError_t launch_attn_probs_bwd(const float* dD, const float* P, const uint32_t* mask,
                                  double scale, float* dZ, float* D, int64_t rows, int64_t cols,
                                  cudaStream_t st) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if (vec_ok(cols, 0, {dD, P, dZ, D, mask}, TM_SOFTMAX_LONG_MIN_BWD)) {
        const int vpl = (int)(cols / 128);
        return D ? bwd_vec<true, true>(vpl, dD, P, mask, scale, dZ, D, rows, st)
                 : bwd_vec<true, false>(vpl, dD, P, mask, scale, dZ, nullptr, rows, st);
    }
    if (long_ok(cols, 0, {dD, P, dZ, D, mask}, TM_SOFTMAX_LONG_MIN_BWD)) {
        const int nch = (int)(cols / 128);
        return D ? bwd_long<true, true>(nch, dD, P, mask, scale, dZ, D, rows, st)
                 : bwd_long<true, false>(nch, dD, P, mask, scale, dZ, nullptr, rows, st);
    }
    launch(softmax_bwd_generic_kernel, generic_grid((const void*)softmax_bwd_generic_kernel, rows),
                                 kBlock, 0, st)(dD, P, mask, 1, scale, dZ, D, rows, cols);
    return cudaGetLastError();
}

}  // namespace tb
