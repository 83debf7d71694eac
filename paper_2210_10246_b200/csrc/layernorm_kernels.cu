// layernorm_kernels.cu -- In-Place LayerNorm forward/backward for sm_100a.
//
// Forward  (tempo_ops::layernorm, ops_tempo.cpp:98-119 -> layernorm_forward
//           ops_reference.cpp:47-65 -> row_moments kernels.cpp:153-179):
//   mean = sum x / M and var = sum (x - mean)^2 / M, two-pass as the
//   reference, as fp32 tree sums plus one refinement step of the mean
//   (refine_moments: the reference sums in fp64 and stores float(mean); the
//   refined fp32 mean rounds the same way at any |mean|/std); rstd =
//   1/sqrt(var + eps) in fp64 per row
//   (ops_tempo.cpp:111-112, F32-stored); y = fma(gamma*rstd, x - mean, beta)
//   in fp32.  (The generic fallback kernel keeps the fp64 formulation.)
//   Stash: y and rstd[row] only.
//   HBM: read x (4 B) + write y (4 B) per element, + 4 B/row + 8 B/column.
// Backward (closure ops_tempo.cpp:121-155): xhat = (y - beta)/gamma,
//   s1 = sum g*gamma, s2 = sum g*gamma*xhat (fp32 row reductions),
//   dx = (g*gamma - s1/M - xhat*s2/M) * rstd; dgamma/dbeta: fp64 per-CTA
//   column partials (stage 1, in registers) reduced across CTAs in a fixed
//   order by a second kernel (stage 2) -- bitwise reproducible.
//   HBM: read dy, y (8 B) + write dx (4 B) per element, + rows/cols terms.
//
// Layout: a CTA spans the columns of a row (thread t owns the float4 at
// column 4t), gamma/beta for its columns stay in registers, and the CTA
// walks row tiles with a grid stride; the tiles arrive through a TMA
// (cp.async.bulk) ring in shared memory, kStages deep.  Row reductions are
// warp shuffles plus one smem exchange (fixed order, identical in every
// thread).  Long rows: the forward (cols % 128 == 0, > 1024) streams whole
// rows through a TMA ring into a CTA of W warps (ln_fwd_long_kernel); the
// backward (cols % 4 == 0, 2048 < cols <= 16384) splits the columns over a
// thread-block cluster whose CTAs exchange the row sums through distributed
// shared memory (ln_bwd_cluster_kernel).  Other shapes and unaligned
// pointers use the generic kernels (one element per thread per pass).
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "common.cuh"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kRows = 4;           // rows in flight per CTA iteration (forward)
#ifndef TM_LN_WAVES
#define TM_LN_WAVES 8  // forward warp kernel: 8 waves measured 6 % faster than 1
#endif
#ifndef TM_LN_BWD_CPT2
#define TM_LN_BWD_CPT2 0
#endif
#ifndef TM_LN_BWD_ROWS
#define TM_LN_BWD_ROWS 4
#endif
#ifndef TM_LN_BWD_STAGES
#define TM_LN_BWD_STAGES 2  // re-tuned with PDL: 2 stages 77.0 -> 75.2 us, bit-identical
#endif
constexpr int kRowsB = TM_LN_BWD_ROWS;  // rows per CTA iteration (backward)
constexpr int kStagesB = TM_LN_BWD_STAGES;
constexpr int kMaxThreads = 512;  // cols <= 2048 on the vector path
// 2048 < cols <= 4096: the vector backward with 1024-thread CTAs (one row
// per thread-column group, ROWS-row tiles; 64 registers) instead of the
// cluster kernel
#ifndef TM_LN_BWD_WIDE
#define TM_LN_BWD_WIDE 1
#endif
#ifndef TM_LN_BWD_WIDE_ROWS
#define TM_LN_BWD_WIDE_ROWS 1
#endif
constexpr int kWideThreads = 1024;
constexpr int kRowsW = TM_LN_BWD_WIDE_ROWS;
constexpr int kVecMaxCols = 4 * (TM_LN_BWD_WIDE ? kWideThreads : kMaxThreads);
constexpr double kGammaMin = 1e-12;  // ops_tempo.hpp:46

// Block-wide sum of kN values per thread.  `red` holds 2 buffers of
// [kN][32] values; `phase` alternates so one __syncthreads per reduction
// suffices.  Every thread gets the same result (fixed summation order).
__device__ __forceinline__ float warp_sum_t(float v) { return warp_sumf(v); }
__device__ __forceinline__ double warp_sum_t(double v) { return warp_sum(v); }

template <int kN, typename T>
__device__ __forceinline__ void block_sum(T (&v)[kN], T* red, int& phase) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    T* buf = red + phase * (kN * 32);
#pragma unroll
    for (int i = 0; i < kN; ++i) {
        T s = warp_sum_t(v[i]);
        if (lane == 0) buf[i * 32 + wid] = s;
    }
    __syncthreads();
    // cross-warp step, lane-parallel: lane l reads warp l's partial (l < nw)
    // and a butterfly over the warp finishes the sum -- the same fixed order
    // in every warp, so every thread gets the identical value.
#pragma unroll
    for (int i = 0; i < kN; ++i) {
        T s = lane < nw ? buf[i * 32 + lane] : T(0);
        v[i] = warp_sum_t(s);
    }
    phase ^= 1;
}

// Row moments from a first mean estimate m0 (an fp32 tree sum / M) and the
// sums over the row of d = x - m0 (t) and d^2 (q): one step of iterative
// refinement.  The reference sums in fp64 and stores float(mean)
// (kernels.cpp:165-176); an fp32 tree sum alone drifts by several ulps of the
// mean when |mean| >> std (rel_err 1e-4 on y at |mean|/std = 1000).  Here
// d = x - m0 is exact wherever x is within 2x of m0 (Sterbenz), so t/M is
// the small correction mean - m0 accurate to ~M ulps of std, and
// float(m0 + t/M) rounds to the reference's float(mean) except within
// ~1e-7 std of a rounding tie.  var = q/M - (t/M)^2 (the sum of squares about
// m0 minus the shift term), the reference's two-pass variance to fp32
// accuracy.
__device__ __forceinline__ void refine_moments(float m0, float t, float q, float inv_m,
                                               float& mean, float& var) {
    const double delta = (double)t * (double)inv_m;
    mean = (float)((double)m0 + delta);
    // clamp rounding-negative variances to 0 but keep a NaN (a NaN in the
    // row makes the reference's var and rstd NaN; fmaxf would turn it into 0
    // and rstd into 1/sqrt(eps))
    const float v = fmaf(-(float)delta, (float)delta, q * inv_m);
    var = v < 0.0f ? 0.0f : v;
}

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// y = gamma * ((x - mean) * rs) + beta, no contraction (ops_reference.cpp:61-62).
__device__ __forceinline__ float ln_y(float x, double mean_f, double rs, double g, double b) {
    return (float)dadd(dmul(g, dmul(dadd((double)x, -mean_f), rs)), b);
}

// ------------------------------------------------------------------ forward
// TMA-staged pipeline: thread 0 streams row tiles (kRows contiguous rows)
// into a kStages-deep shared-memory ring with cp.async.bulk, completing on
// one mbarrier per stage; all threads consume a tile from smem (thread t:
// the float4 at column 4t), so HBM reads stay in flight across the block
// reductions.  A stage is refilled as soon as the tile's first block
// reduction proves every thread has read it.
constexpr int kStages = 3;

__device__ __forceinline__ void ln_issue(const float* src, int64_t tile, int tile_rows,
                                         int64_t rows, int cols, float* dst, uint64_t* bar) {
    const int64_t r0 = tile * tile_rows;
    const int nr = (int)min((int64_t)tile_rows, rows - r0);
    const uint32_t bytes = (uint32_t)nr * (uint32_t)cols * 4u;
    mbar_expect_tx(bar, bytes);
    bulk_g2s(dst, src + r0 * cols, bytes, bar);
}

template <int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 3 : 1) ln_fwd_vec_kernel(
    const float* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    double eps, float* __restrict__ y, float* __restrict__ rstd, int64_t rows, int cols,
    int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    float* ring = reinterpret_cast<float*>(dsm + 128);
    __shared__ float red[2 * 2 * kRows * 32];
    int phase = 0;
    const int tile_floats = kRows * cols;
    const int64_t ntiles = (rows + kRows - 1) / kRows;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < ntiles) ln_issue(x, t, kRows, rows, cols, ring + s * tile_floats, &full[s]);
        }
    }
    const int c4 = threadIdx.x;  // float4 column group
    const bool act = c4 * 4 < cols;
    float4 g = make_float4(1.f, 1.f, 1.f, 1.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
    if (act) {
        g = reinterpret_cast<const float4*>(gamma)[c4];
        b = reinterpret_cast<const float4*>(beta)[c4];
        if (status && blockIdx.x == 0) {
            if (fabs((double)g.x) < kGammaMin || fabs((double)g.y) < kGammaMin ||
                fabs((double)g.z) < kGammaMin || fabs((double)g.w) < kGammaMin) {
                *status = TEMPO_ERR_PARAM;
            }
        }
    }
    const float inv_m = 1.0f / (float)cols;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % kStages;
        mbar_wait(&full[st], (uint32_t)((it / kStages) & 1));
        const int64_t r0 = tile * kRows;
        const float* sp = ring + st * tile_floats;
        float4 v[kRows];
        float s[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (act && r0 + i < rows) v[i] = reinterpret_cast<const float4*>(sp + i * cols)[c4];
            s[i] = (v[i].x + v[i].y) + (v[i].z + v[i].w);
        }
        block_sum<kRows>(s, red, phase);
        if (threadIdx.x == 0) {  // every thread has read stage st: refill it
            const int64_t nt = tile + (int64_t)kStages * gridDim.x;
            if (nt < ntiles) {
                fence_proxy_async_smem();
                ln_issue(x, nt, kRows, rows, cols, ring + st * tile_floats, &full[st]);
            }
        }
        float mean[kRows], q[2 * kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            mean[i] = s[i] * inv_m;  // first estimate, refined below
            const float d0 = v[i].x - mean[i], d1 = v[i].y - mean[i];
            const float d2 = v[i].z - mean[i], d3 = v[i].w - mean[i];
            q[i] = act ? fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3) : 0.0f;
            q[kRows + i] = act ? (d0 + d1) + (d2 + d3) : 0.0f;
        }
        block_sum<2 * kRows>(q, red, phase);
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int64_t r = r0 + i;
            if (r >= rows) break;
            float var_f;
            refine_moments(mean[i], q[kRows + i], q[i], inv_m, mean[i], var_f);
            const double rsd = 1.0 / sqrt((double)var_f + eps);  // ops_tempo.cpp:111-112
            const float rs = (float)rsd;
            if (act) {
                float4 o;
                o.x = fmaf(g.x * rs, v[i].x - mean[i], b.x);
                o.y = fmaf(g.y * rs, v[i].y - mean[i], b.y);
                o.z = fmaf(g.z * rs, v[i].z - mean[i], b.z);
                o.w = fmaf(g.w * rs, v[i].w - mean[i], b.w);
                st_stream(reinterpret_cast<float4*>(y + r * cols) + c4, o);
            }
            if (threadIdx.x == 0) rstd[r] = rs;
        }
    }
}

// Warp-per-row forward for cols = 128*VPL (768, 1024, ...): each warp
// streams ITS OWN rows through a private kWStages-deep TMA ring (lane 0
// issues cp.async.bulk of the next row as soon as the warp has read a stage),
// so there is no block-wide synchronization at all; the row statistics are
// warp shuffles; gamma/beta are read from shared memory.
#ifndef TM_LN_FWD_STAGES
#define TM_LN_FWD_STAGES 3
#endif
constexpr int kWStages = TM_LN_FWD_STAGES;
constexpr int kWWarps = 8;

template <int VPL>
__global__ void __launch_bounds__(kWWarps * 32, 2) ln_fwd_warp_kernel(
    const float* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    double eps, float* __restrict__ y, float* __restrict__ rstd, int64_t rows,
    int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int C = VPL * 128;
    extern __shared__ __align__(128) unsigned char dsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(dsm) + wid * kWStages;
    float4* gb = reinterpret_cast<float4*>(dsm + 1024);  // gamma [C/4] then beta [C/4]
    float* ring = reinterpret_cast<float*>(dsm + 1024 + 2 * C * 4) + wid * kWStages * C;
    for (int i = threadIdx.x; i < C / 4; i += blockDim.x) {
        const float4 g = reinterpret_cast<const float4*>(gamma)[i];
        gb[i] = g;
        gb[C / 4 + i] = reinterpret_cast<const float4*>(beta)[i];
        if (status && blockIdx.x == 0 &&
            (fabsf(g.x) < 1e-12f || fabsf(g.y) < 1e-12f || fabsf(g.z) < 1e-12f ||
             fabsf(g.w) < 1e-12f)) {
            // exact |gamma| < 1e-12 test in double for values near the bound
            if (fabs((double)g.x) < kGammaMin || fabs((double)g.y) < kGammaMin ||
                fabs((double)g.z) < kGammaMin || fabs((double)g.w) < kGammaMin)
                *status = TEMPO_ERR_PARAM;
        }
    }
    const int64_t gw = (int64_t)blockIdx.x * kWWarps + wid;   // global warp
    const int64_t nw = (int64_t)gridDim.x * kWWarps;
    if (lane == 0) {
        for (int s = 0; s < kWStages; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    __syncthreads();  // gamma/beta staged, barriers initialised
    if (lane == 0) {
        for (int s = 0; s < kWStages; ++s) {
            const int64_t r = gw + (int64_t)s * nw;
            if (r < rows) {
                mbar_expect_tx(&bars[s], C * 4);
                bulk_g2s(ring + s * C, x + r * C, C * 4, &bars[s]);
            }
        }
    }
    const float inv_m = 1.0f / (float)C;
    int it = 0;
    for (int64_t r = gw; r < rows; r += nw, ++it) {
        const int st = it % kWStages;
        mbar_wait(&bars[st], (uint32_t)((it / kWStages) & 1));
        float4 v[VPL];
        const float4* sp = reinterpret_cast<const float4*>(ring + st * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) v[k] = sp[k * 32 + lane];
        __syncwarp();
        if (lane == 0) {  // the warp has read stage st: refill it with its next row
            const int64_t rn = r + (int64_t)kWStages * nw;
            if (rn < rows) {
                fence_proxy_async_smem();
                mbar_expect_tx(&bars[st], C * 4);
                bulk_g2s(ring + st * C, x + rn * C, C * 4, &bars[st]);
            }
        }
        float s = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        const float m0 = warp_sumf(s) * inv_m;  // first estimate of the mean
        float q = 0.0f, t = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float d0 = v[k].x - m0, d1 = v[k].y - m0;
            const float d2 = v[k].z - m0, d3 = v[k].w - m0;
            q += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
            t += (d0 + d1) + (d2 + d3);
        }
        float mean, var_f;
        refine_moments(m0, warp_sumf(t), warp_sumf(q), inv_m, mean, var_f);
        const float rs = (float)(1.0 / sqrt((double)var_f + eps));  // ops_tempo.cpp:111-112
        float4* yr = reinterpret_cast<float4*>(y + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float4 g = gb[k * 32 + lane], b = gb[C / 4 + k * 32 + lane];
            float4 o;
            o.x = fmaf(g.x * rs, v[k].x - mean, b.x);
            o.y = fmaf(g.y * rs, v[k].y - mean, b.y);
            o.z = fmaf(g.z * rs, v[k].z - mean, b.z);
            o.w = fmaf(g.w * rs, v[k].w - mean, b.w);
            st_stream(yr + k * 32 + lane, o);
        }
        if (lane == 0) rstd[r] = rs;
    }
}

// ---- hidden dropout -> residual add -> LayerNorm, fused (forward) --------
// The reference layer chains ref_ops::dropout(proj) -> g.add(residual, .) ->
// tempo_ops::layernorm (encoder.cpp:180-191, 198-210).  Here one pass reads
// the projection and the residual rows and writes only y, rstd and the mask
// bits: r = residual + (keep ? float(double(proj) * scale) : 0) is formed in
// registers (bit-exact with the reference's F32 dropout then add: the
// dropout product rounds once from fp64 as mask_scale does, kernels.cpp:
// 285-295, and an fp32 add equals float(double(a) + double(b))), then the
// in-place LayerNorm of r exactly as ln_fwd_warp_kernel.  Neither the
// dropout output nor r is stored (the Tempo layer stashes neither).
// MODE 1: supplied mask; MODE 2: Philox mask generated by global element
// index (the same bits as tempo_dropout_fwd's) and written.
// HBM: read proj + residual (8 B) + write y (4 B) + 1 bit per element.
#ifndef TM_DAL_STAGES
#define TM_DAL_STAGES 1  // per-warp ring depth (A/B: 1 74.2, 2 75.8, 3 80.4 us at 32768x1024)
#endif
constexpr int kDStages = TM_DAL_STAGES;

template <int VPL, int MODE>
#ifndef TM_DAL_MINB
#define TM_DAL_MINB 2
#endif
__global__ void __launch_bounds__(kWWarps * 32, TM_DAL_MINB) dal_fwd_warp_kernel(
    const float* __restrict__ proj, const float* __restrict__ res, uint32_t* __restrict__ mask,
    double scale, uint64_t thresh, uint64_t seed, uint64_t offset,
    const float* __restrict__ gamma, const float* __restrict__ beta, double eps,
    float* __restrict__ y, float* __restrict__ rstd, int64_t rows, int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int C = VPL * 128;
    extern __shared__ __align__(128) unsigned char dsm[];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint64_t* bars = reinterpret_cast<uint64_t*>(dsm) + wid * kDStages;
    float4* gb = reinterpret_cast<float4*>(dsm + 1024);  // gamma [C/4] then beta [C/4]
    // per warp: a kDStages-deep TMA ring of projection rows; the residual
    // row is loaded straight into registers at the top of the row, so its
    // latency overlaps the mask generation and the ring wait (smem stays
    // small enough for two CTAs per SM)
    float* ring = reinterpret_cast<float*>(dsm + 1024 + 2 * C * 4) + wid * kDStages * C;
    for (int i = threadIdx.x; i < C / 4; i += blockDim.x) {
        const float4 g = reinterpret_cast<const float4*>(gamma)[i];
        gb[i] = g;
        gb[C / 4 + i] = reinterpret_cast<const float4*>(beta)[i];
        if (status && blockIdx.x == 0 &&
            (fabs((double)g.x) < kGammaMin || fabs((double)g.y) < kGammaMin ||
             fabs((double)g.z) < kGammaMin || fabs((double)g.w) < kGammaMin))
            *status = TEMPO_ERR_PARAM;
    }
    const int64_t gw = (int64_t)blockIdx.x * kWWarps + wid;
    const int64_t nw = (int64_t)gridDim.x * kWWarps;
    auto issue = [&](int64_t r, int s) {
        mbar_expect_tx(&bars[s], C * 4);
        bulk_g2s(ring + s * C, proj + r * C, C * 4, &bars[s]);
    };
    if (lane == 0) {
        for (int s = 0; s < kDStages; ++s) mbar_init(&bars[s], 1);
        mbar_fence_init();
    }
    __syncthreads();  // gamma/beta staged, barriers initialised
    if (lane == 0) {
        for (int s = 0; s < kDStages; ++s) {
            const int64_t r = gw + (int64_t)s * nw;
            if (r < rows) issue(r, s);
        }
    }
    const float inv_m = 1.0f / (float)C;
    int it = 0;
    for (int64_t r = gw; r < rows; r += nw, ++it) {
        const int st = it % kDStages;
        float4 v[VPL];
        const float4* rr = reinterpret_cast<const float4*>(res + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) v[k] = ld_stream(rr + k * 32 + lane);
        uint32_t nib[VPL];
        uint32_t* mrow = mask + ((r * C) >> 5);  // C % 128 == 0: the row owns whole words
        if (MODE == 1) {
#pragma unroll
            for (int k = 0; k < VPL; ++k) nib[k] = chunk_nibble(mrow + k * 4, lane);
        } else {
#pragma unroll
            for (int k = 0; k < VPL; ++k) {
                const U4 q = philox_quad(seed, (offset + (uint64_t)(r * C + k * 128 + lane * 4)) >> 2);
                nib[k] = nibble4((uint64_t)q.x >= thresh, (uint64_t)q.y >= thresh,
                                 (uint64_t)q.z >= thresh, (uint64_t)q.w >= thresh);
                store_chunk_mask(mrow + k * 4, nib[k], lane);
            }
        }
        mbar_wait(&bars[st], (uint32_t)((it / kDStages) & 1));
        const float4* sp = reinterpret_cast<const float4*>(ring + st * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float4 p = sp[k * 32 + lane];
            v[k].x += (nib[k] & 1u) ? (float)((double)p.x * scale) : 0.0f;
            v[k].y += (nib[k] & 2u) ? (float)((double)p.y * scale) : 0.0f;
            v[k].z += (nib[k] & 4u) ? (float)((double)p.z * scale) : 0.0f;
            v[k].w += (nib[k] & 8u) ? (float)((double)p.w * scale) : 0.0f;
        }
        __syncwarp();
        if (lane == 0) {  // the warp has read stage st: refill it with its next row
            const int64_t rn = r + (int64_t)kDStages * nw;
            if (rn < rows) {
                fence_proxy_async_smem();
                issue(rn, st);
            }
        }
        float s = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        const float m0 = warp_sumf(s) * inv_m;
        float q = 0.0f, t = 0.0f;
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float d0 = v[k].x - m0, d1 = v[k].y - m0;
            const float d2 = v[k].z - m0, d3 = v[k].w - m0;
            q += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
            t += (d0 + d1) + (d2 + d3);
        }
        float mean, var_f;
        refine_moments(m0, warp_sumf(t), warp_sumf(q), inv_m, mean, var_f);
        const float rs = (float)(1.0 / sqrt((double)var_f + eps));  // ops_tempo.cpp:111-112
        float4* yr = reinterpret_cast<float4*>(y + r * C);
#pragma unroll
        for (int k = 0; k < VPL; ++k) {
            const float4 g = gb[k * 32 + lane], b = gb[C / 4 + k * 32 + lane];
            float4 o;
            o.x = fmaf(g.x * rs, v[k].x - mean, b.x);
            o.y = fmaf(g.y * rs, v[k].y - mean, b.y);
            o.z = fmaf(g.z * rs, v[k].z - mean, b.z);
            o.w = fmaf(g.w * rs, v[k].w - mean, b.w);
            st_stream(yr + k * 32 + lane, o);
        }
        if (lane == 0) rstd[r] = rs;
    }
}

size_t dal_fwd_smem(int vpl) {
    return 1024 + 2 * (size_t)vpl * 128 * 4 + (size_t)kWWarps * kDStages * vpl * 128 * 4;
}

// Generic fused forward (cols % 32 == 0, any length): one CTA per row, the
// row's r = residual + dropout(proj) materialised in shared memory (fp32,
// cols floats), then the moments and y as ln_fwd_generic_kernel (fp64
// sums).  32 consecutive elements of a row are one mask word (ballot).
__global__ void __launch_bounds__(256) dal_fwd_generic_kernel(
    const float* __restrict__ proj, const float* __restrict__ res, uint32_t* __restrict__ mask,
    int mode, double scale, uint64_t thresh, uint64_t seed, uint64_t offset,
    const float* __restrict__ gamma, const float* __restrict__ beta, double eps,
    float* __restrict__ y, float* __restrict__ rstd, int64_t rows, int cols,
    int32_t* __restrict__ status, int r_in_y) {
    grid_dep_wait();
    grid_dep_launch();
    extern __shared__ float xr_sm[];  // [cols]; 0 bytes: r staged in the output row itself
    __shared__ double red[2 * 32];
    int phase = 0;
    const int lane = threadIdx.x & 31;
    if (status && blockIdx.x == 0) {
        for (int j = threadIdx.x; j < cols; j += blockDim.x)
            if (fabs((double)gamma[j]) < kGammaMin) *status = TEMPO_ERR_PARAM;
    }
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        // every element is written and read back by the same thread (same j
        // loop), so the global staging needs no barrier
        float* xr = r_in_y ? y + r * cols : xr_sm;
        double s[1] = {0.0};
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {  // cols % 32 == 0: full warps
            const int64_t i = r * cols + j;
            bool keep;
            if (mode == 2) {
                keep = (uint64_t)philox_at(seed, offset + (uint64_t)i) >= thresh;
                const uint32_t bits = __ballot_sync(kFull, keep);
                if (lane == 0) mask[i >> 5] = bits;
            } else {
                keep = (mask[i >> 5] >> (i & 31)) & 1u;
            }
            const float v = res[i] + (keep ? (float)((double)proj[i] * scale) : 0.0f);
            xr[j] = v;
            s[0] += (double)v;
        }
        block_sum<1>(s, red, phase);
        const double mean = s[0] / (double)cols;
        double q[1] = {0.0};
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            const double d = (double)xr[j] - mean;
            q[0] = dadd(q[0], dmul(d, d));
        }
        block_sum<1>(q, red, phase);
        const double mean_f = (double)(float)mean;
        const float var_f = (float)(q[0] / (double)cols);
        const double rs = 1.0 / sqrt((double)var_f + eps);
        for (int j = threadIdx.x; j < cols; j += blockDim.x)
            y[r * cols + j] = ln_y(xr[j], mean_f, rs, (double)gamma[j], (double)beta[j]);
        if (threadIdx.x == 0) rstd[r] = (float)rs;
        __syncthreads();  // xr is rewritten by the next row
    }
}

// ---- long rows (cols % 128 == 0, 1024 < cols <= 16384), forward ---------
// One CTA = one row group of W warps, persistent over rows r = blockIdx.x +
// i*gridDim.x; the rows (x, or proj and residual for the fused dropout -> add
// -> LayerNorm: MODE 1 supplied mask, MODE 2 Philox, the same bits as
// dal_fwd_warp_kernel's) stream into a shallow TMA ring in shared memory (one
// mbarrier per stage, thread 0 issues), so the bytes in flight per SM are
// bounded by smem, not by the registers holding a row.  The row's 128-column
// chunks are dealt round-robin to the warps (warp w: chunks w, w+W, ..., at
// most VPL) and read from the stage into registers; the row sums are warp
// shuffles plus an exchange of the W warp partials through shared memory
// (__syncthreads; combined in warp order in every thread, slots alternating by
// row parity).  The first exchange proves every warp has read the stage, so
// thread 0 refills it there.  One HBM read and one write per element;
// statistics as ln_fwd_warp_kernel (fp32 sums refined once, rstd in fp64);
// gamma/beta are L1-resident __ldg float4s.
constexpr int kLongVPL = 8;
#ifndef TM_LNL_STAGES
#define TM_LNL_STAGES 1  // A/B at 2^25 elements: 1 stage 0.82/0.81/0.80 of the copy peak at H = 2048/4096/8192 vs 0.76/0.73/0.71 (2), 0.69/0.65/0.65 (3)
#endif
constexpr size_t kLnlRingBytes = 160 * 1024;

template <int W, int MODE>
__global__ void __launch_bounds__(W * 32) ln_fwd_long_kernel(
    const float* __restrict__ x, const float* __restrict__ res, uint32_t* __restrict__ mask,
    double scale, uint64_t thresh, uint64_t seed, uint64_t offset,
    const float* __restrict__ gamma, const float* __restrict__ beta, double eps,
    float* __restrict__ y, float* __restrict__ rstd, int64_t rows, int nch, int ns,
    int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int T = MODE == 0 ? 1 : 2;  // tensors per stage: x | proj, residual
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    const float4* ring = reinterpret_cast<const float4*>(dsm + 128);
    __shared__ float red[2][3][W];  // [row parity][s, t, q][warp]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t C = (int64_t)nch * 128;
    const uint32_t row_bytes = (uint32_t)C * 4u;
    auto issue = [&](int64_t r, int st) {
        mbar_expect_tx(&full[st], T * row_bytes);
        bulk_g2s((void*)(ring + (size_t)(T * st) * (C / 4)), x + r * C, row_bytes, &full[st]);
        if (T == 2)
            bulk_g2s((void*)(ring + (size_t)(T * st + 1) * (C / 4)), res + r * C, row_bytes, &full[st]);
    };
    if (threadIdx.x == 0) {
        for (int st = 0; st < ns; ++st) mbar_init(&full[st], 1);
        mbar_fence_init();
    }
    if (status && blockIdx.x == 0) {
        for (int64_t i = threadIdx.x; i < C; i += W * 32)
            if (fabs((double)gamma[i]) < kGammaMin) *status = TEMPO_ERR_PARAM;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int st = 0; st < ns; ++st) {
            const int64_t r = blockIdx.x + (int64_t)st * gridDim.x;
            if (r < rows) issue(r, st);
        }
    }
    const float inv_m = 1.0f / (float)C;
    int it = 0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x, ++it) {
        const int st = it % ns, par = it & 1;
        uint32_t nb[kLongVPL];
        uint32_t* mrow = mask + ((r * C) >> 5);
        if (MODE != 0) {
#pragma unroll
            for (int k = 0; k < kLongVPL; ++k) {
                const int c = w + k * W;
                if (c >= nch) continue;
                if (MODE == 1) {
                    nb[k] = chunk_nibble(mrow + c * 4, lane);
                } else {
                    const U4 q = philox_quad(seed, (offset + (uint64_t)(r * C + c * 128 + lane * 4)) >> 2);
                    nb[k] = nibble4((uint64_t)q.x >= thresh, (uint64_t)q.y >= thresh,
                                    (uint64_t)q.z >= thresh, (uint64_t)q.w >= thresh);
                    store_chunk_mask(mrow + c * 4, nb[k], lane);
                }
            }
        }
        mbar_wait(&full[st], (uint32_t)((it / ns) & 1));
        const float4* sx = ring + (size_t)(T * st) * (C / 4);
        float4 v[kLongVPL];
        float s = 0.0f;
#pragma unroll
        for (int k = 0; k < kLongVPL; ++k) {
            const int c = w + k * W;
            if (c >= nch) continue;
            v[k] = sx[c * 32 + lane];
            if (MODE != 0) {  // v = residual + dropout(proj)
                const float4 rv = sx[C / 4 + c * 32 + lane];
                v[k].x = rv.x + ((nb[k] & 1u) ? (float)((double)v[k].x * scale) : 0.0f);
                v[k].y = rv.y + ((nb[k] & 2u) ? (float)((double)v[k].y * scale) : 0.0f);
                v[k].z = rv.z + ((nb[k] & 4u) ? (float)((double)v[k].z * scale) : 0.0f);
                v[k].w = rv.w + ((nb[k] & 8u) ? (float)((double)v[k].w * scale) : 0.0f);
            }
            s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
        }
        s = warp_sumf(s);
        if (lane == 0) red[par][0][w] = s;
        __syncthreads();  // every warp has read stage st: refill it
        if (threadIdx.x == 0) {
            const int64_t rn = r + (int64_t)ns * gridDim.x;
            if (rn < rows) {
                fence_proxy_async_smem();
                issue(rn, st);
            }
        }
        s = red[par][0][0];
#pragma unroll
        for (int i = 1; i < W; ++i) s += red[par][0][i];
        const float m0 = s * inv_m;  // first estimate of the mean
        float q = 0.0f, t = 0.0f;
#pragma unroll
        for (int k = 0; k < kLongVPL; ++k) {
            if (w + k * W >= nch) continue;
            const float d0 = v[k].x - m0, d1 = v[k].y - m0;
            const float d2 = v[k].z - m0, d3 = v[k].w - m0;
            q += fmaf(d0, d0, d1 * d1) + fmaf(d2, d2, d3 * d3);
            t += (d0 + d1) + (d2 + d3);
        }
        t = warp_sumf(t);
        q = warp_sumf(q);
        if (lane == 0) {
            red[par][1][w] = t;
            red[par][2][w] = q;
        }
        __syncthreads();
        t = red[par][1][0];
        q = red[par][2][0];
#pragma unroll
        for (int i = 1; i < W; ++i) {
            t += red[par][1][i];
            q += red[par][2][i];
        }
        float mean, var_f;
        refine_moments(m0, t, q, inv_m, mean, var_f);
        const float rs = (float)(1.0 / sqrt((double)var_f + eps));  // ops_tempo.cpp:111-112
        float4* yr = reinterpret_cast<float4*>(y + r * C);
#pragma unroll
        for (int k = 0; k < kLongVPL; ++k) {
            const int c = w + k * W;
            if (c >= nch) continue;
            const float4 gm = __ldg(reinterpret_cast<const float4*>(gamma) + c * 32 + lane);
            const float4 b = __ldg(reinterpret_cast<const float4*>(beta) + c * 32 + lane);
            float4 o;
            o.x = fmaf(gm.x * rs, v[k].x - mean, b.x);
            o.y = fmaf(gm.y * rs, v[k].y - mean, b.y);
            o.z = fmaf(gm.z * rs, v[k].z - mean, b.z);
            o.w = fmaf(gm.w * rs, v[k].w - mean, b.w);
            st_stream(yr + c * 32 + lane, o);
        }
        if (threadIdx.x == 0) rstd[r] = rs;
    }
}

inline int lnl_stages(int64_t cols, int tensors) {
    const int ns = (int)(kLnlRingBytes / ((size_t)tensors * cols * 4));
    return ns < 1 ? 1 : ns > TM_LNL_STAGES ? TM_LNL_STAGES : ns;
}
inline size_t lnl_smem(int64_t cols, int tensors) {
    return 128 + (size_t)lnl_stages(cols, tensors) * tensors * cols * 4;
}
// forward: W * 8 chunks cover the row
inline int lnl_fwd_warps(int64_t nch) {
    return nch <= 8 ? 1 : nch <= 16 ? 2 : nch <= 32 ? 4 : nch <= 64 ? 8 : 16;
}
#ifndef TM_LN_LONG_MIN
#define TM_LN_LONG_MIN 1024  // LN forward: rows longer than this take ln_fwd_long_kernel
#endif
#ifndef TM_DAL_LONG_MIN
#define TM_DAL_LONG_MIN 1024  // fused dropout -> add -> LN forward: likewise
#endif
// Small LN forwards (configs[1]: 16384 x 768 = 12.6 M elements) take the TMA
// row-group kernel at any row length (one-warp CTAs for H <= 1024): A/B
// configs[1] fwd+bwd 57.3 -> 52.9 us; at 32768 x 1024 the warp kernel stays
// ahead (0.88 vs 0.86 of the copy peak), hence the size switch.
#ifndef TM_LN_LONG_SMALL_N
#define TM_LN_LONG_SMALL_N (int64_t(1) << 24)
#endif

size_t warp_fwd_smem(int vpl) {
    return 1024 + 2 * (size_t)vpl * 128 * 4 + (size_t)kWWarps * kWStages * vpl * 128 * 4;
}

// Generic: any cols, any alignment; thread t handles columns t, t+bs, ...
// Three passes over the row (L1/L2 resident for moderate cols).
__global__ void __launch_bounds__(256) ln_fwd_generic_kernel(
    const float* __restrict__ x, const float* __restrict__ gamma, const float* __restrict__ beta,
    double eps, float* __restrict__ y, float* __restrict__ rstd, int64_t rows, int cols,
    int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    __shared__ double red[2 * 32];
    int phase = 0;
    if (status && blockIdx.x == 0) {
        for (int j = threadIdx.x; j < cols; j += blockDim.x)
            if (fabs((double)gamma[j]) < kGammaMin) *status = TEMPO_ERR_PARAM;
    }
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float* xr = x + r * cols;
        double s[1] = {0.0};
        for (int j = threadIdx.x; j < cols; j += blockDim.x) s[0] += (double)xr[j];
        block_sum<1>(s, red, phase);
        const double mean = s[0] / (double)cols;
        double q[1] = {0.0};
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            double d = (double)xr[j] - mean;
            q[0] = dadd(q[0], dmul(d, d));
        }
        block_sum<1>(q, red, phase);
        const double mean_f = (double)(float)mean;
        const float var_f = (float)(q[0] / (double)cols);
        const double rs = 1.0 / sqrt((double)var_f + eps);
        for (int j = threadIdx.x; j < cols; j += blockDim.x)
            y[r * cols + j] = ln_y(xr[j], mean_f, rs, (double)gamma[j], (double)beta[j]);
        if (threadIdx.x == 0) rstd[r] = (float)rs;
    }
}

// ----------------------------------------------------------------- backward
// Stage 1, vector path: dx per row, per-CTA fp64 column partials of
// dgamma = sum g*xhat and dbeta = sum g, written to ws[cta][2][cols].
// Same TMA ring as the forward; a stage holds kRowsB rows of dy and of y.
// DROP (the fused dropout -> residual add -> LayerNorm backward): dx is the
// residual's gradient d(r) and, from the stashed mask bits, the
// projection's gradient d(proj) = keep ? float(double(dx) * scale) : 0
// (dropout_backward, ops_reference.cpp:155-161) is written beside it -- one
// pass instead of LN backward + a dropout backward re-reading dx.
template <int NT, int CPT, bool DROP = false, int ROWS = kRowsB>
__global__ void __launch_bounds__(NT) ln_bwd_vec_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const float* __restrict__ rstd,
    const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ dx,
    double* __restrict__ ws, int64_t rows, int cols, const uint32_t* __restrict__ mask,
    double scale, float* __restrict__ dproj) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    // persistent grid: let stage 2 (a PDL dependent) get resident in the
    // leftover slots; it waits for us to finish
    grid_dep_launch_persistent();
    // Thread t owns the CPT float4 column groups t, t + blockDim, ... of every
    // row (conflict-free 128-bit smem reads, coalesced stores); more columns
    // per thread amortise the per-row block reduction.
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);
    float* ring = reinterpret_cast<float*>(dsm + 128);
    __shared__ float red[2 * 2 * ROWS * 32];
    int phase = 0;
    const int tile_floats = ROWS * cols;  // per tensor; a stage holds dy then y
    const int64_t ntiles = (rows + ROWS - 1) / ROWS;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesB; ++s) mbar_init(&full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int64_t t, int s) {
        const int64_t r0 = t * ROWS;
        const int nr = (int)min((int64_t)ROWS, rows - r0);
        const uint32_t bytes = (uint32_t)nr * (uint32_t)cols * 4u;
        mbar_expect_tx(&full[s], 2 * bytes);
        bulk_g2s(ring + (2 * s) * tile_floats, dy + r0 * cols, bytes, &full[s]);
        bulk_g2s(ring + (2 * s + 1) * tile_floats, y + r0 * cols, bytes, &full[s]);
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesB; ++s) {
            const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
            if (t < ntiles) issue(t, s);
        }
    }
    const int ncg = cols / 4;  // float4 column groups
    int cg[CPT];
    bool act[CPT];
    float gm[CPT][4], bt[CPT][4], igf[CPT][4];
    double pg[CPT][4], pb[CPT][4];  // fp64 column partials
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        cg[c] = threadIdx.x + c * blockDim.x;
        act[c] = cg[c] < ncg;
        float4 g = make_float4(1.f, 1.f, 1.f, 1.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act[c]) {
            g = reinterpret_cast<const float4*>(gamma)[cg[c]];
            b = reinterpret_cast<const float4*>(beta)[cg[c]];
        }
        const float ga[4] = {g.x, g.y, g.z, g.w}, ba[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            gm[c][k] = ga[k];
            bt[c][k] = ba[k];
            igf[c][k] = (float)(1.0 / (double)ga[k]);
            pg[c][k] = 0.0;
            pb[c][k] = 0.0;
        }
    }
    const float inv_m = 1.0f / (float)cols;
    // rstd (and, DROP, the mask words) of a tile are loaded one tile ahead:
    // they are needed only after the row reduction, and a global load issued
    // there would stall the whole output loop on its latency
    float rs_nx[ROWS];
    uint32_t mw_nx[ROWS][CPT];
    auto prefetch = [&](int64_t t) {
        const int64_t q0 = t * ROWS;
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            const bool in = t < ntiles && q0 + i < rows;
            rs_nx[i] = in ? __ldg(rstd + q0 + i) : 0.f;
            if (DROP) {
#pragma unroll
                for (int c = 0; c < CPT; ++c)
                    mw_nx[i][c] = (in && act[c]) ? __ldg(mask + (((q0 + i) * cols + 4 * cg[c]) >> 5)) : 0u;
            }
        }
    };
    prefetch(blockIdx.x);
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        float rsv[ROWS];
        uint32_t mwv[ROWS][CPT];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            rsv[i] = rs_nx[i];
#pragma unroll
            for (int c = 0; c < CPT; ++c) mwv[i][c] = DROP ? mw_nx[i][c] : 0u;
        }
        prefetch(tile + gridDim.x);
        const int st = it % kStagesB;
        mbar_wait(&full[st], (uint32_t)((it / kStagesB) & 1));
        const int64_t r0 = tile * ROWS;
        const float* gs = ring + (2 * st) * tile_floats;
        const float* ys = ring + (2 * st + 1) * tile_floats;
        float4 gv[ROWS][CPT], yv[ROWS][CPT];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                gv[i][c] = make_float4(0.f, 0.f, 0.f, 0.f);
                yv[i][c] = gv[i][c];
                if (r0 + i < rows && act[c]) {
                    gv[i][c] = reinterpret_cast<const float4*>(gs + i * cols)[cg[c]];
                    yv[i][c] = reinterpret_cast<const float4*>(ys + i * cols)[cg[c]];
                }
            }
        }
        float s[2 * ROWS];
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            float s1 = 0.0f, s2 = 0.0f;
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                const float ga[4] = {gv[i][c].x, gv[i][c].y, gv[i][c].z, gv[i][c].w};
                const float ya[4] = {yv[i][c].x, yv[i][c].y, yv[i][c].z, yv[i][c].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float gg = ga[k] * gm[c][k];
                    const float xh = (ya[k] - bt[c][k]) * igf[c][k];
                    s1 += gg;
                    s2 = fmaf(gg, xh, s2);
                }
            }
            s[2 * i] = s1;
            s[2 * i + 1] = s2;
        }
        block_sum<2 * ROWS>(s, red, phase);
        if (threadIdx.x == 0) {  // stage consumed by every thread: refill
            const int64_t nt = tile + (int64_t)kStagesB * gridDim.x;
            if (nt < ntiles) {
                fence_proxy_async_smem();
                issue(nt, st);
            }
        }
#pragma unroll
        for (int i = 0; i < ROWS; ++i) {
            if (r0 + i >= rows) continue;
            const float c1 = s[2 * i] * inv_m, c2 = s[2 * i + 1] * inv_m;
            const float rs = rsv[i];
#pragma unroll
            for (int c = 0; c < CPT; ++c) {
                if (!act[c]) continue;
                const float ga[4] = {gv[i][c].x, gv[i][c].y, gv[i][c].z, gv[i][c].w};
                const float ya[4] = {yv[i][c].x, yv[i][c].y, yv[i][c].z, yv[i][c].w};
                float o[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float xh = (ya[k] - bt[c][k]) * igf[c][k];
                    o[k] = (fmaf(ga[k], gm[c][k], -c1) - xh * c2) * rs;
                    // dgamma/dbeta partials in fp64 (the F64 oracle's accuracy
                    // over tens of thousands of rows).  sum_i g*xhat =
                    // (sum_i g*y - beta*sum_i g)/gamma per column, so a row
                    // costs one DFMA + one DADD; the column's correction is
                    // applied once, after the row loop.
                    const double gd = (double)ga[k];
                    pg[c][k] = fma(gd, (double)ya[k], pg[c][k]);
                    pb[c][k] += gd;
                }
                st_stream(reinterpret_cast<float4*>(dx + (r0 + i) * cols) + cg[c],
                          make_float4(o[0], o[1], o[2], o[3]));
                if (DROP) {  // 4 elements at a multiple of 4: one nibble of one word
                    const int64_t e = (r0 + i) * cols + 4 * cg[c];
                    const uint32_t nb = (mwv[i][c] >> (e & 31)) & 0xfu;
                    float4 dp;
                    dp.x = (nb & 1u) ? (float)((double)o[0] * scale) : 0.0f;
                    dp.y = (nb & 2u) ? (float)((double)o[1] * scale) : 0.0f;
                    dp.z = (nb & 4u) ? (float)((double)o[2] * scale) : 0.0f;
                    dp.w = (nb & 8u) ? (float)((double)o[3] * scale) : 0.0f;
                    st_stream(reinterpret_cast<float4*>(dproj + (r0 + i) * cols) + cg[c], dp);
                }
            }
        }
    }
    double* wg = ws + (size_t)blockIdx.x * 2 * cols;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        if (!act[c]) continue;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            // fp64 1/gamma and beta rebuilt here (not kept live across the
            // row loop: registers for the 1024-thread variant)
            wg[cg[c] * 4 + k] = fma(-(double)bt[c][k], pb[c][k], pg[c][k]) * (1.0 / (double)gm[c][k]);
            wg[cols + cg[c] * 4 + k] = pb[c][k];
        }
    }
}

// Stage 1, generic path: partials accumulated in shared memory (each column
// owned by one thread, so no races), then written to ws[cta][2][cols].
__global__ void __launch_bounds__(256) ln_bwd_generic_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const float* __restrict__ rstd,
    const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ dx,
    double* __restrict__ ws, int64_t rows, int cols, const uint32_t* __restrict__ mask,
    double scale, float* __restrict__ dproj, int part_in_ws) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    extern __shared__ double part_sm[];  // [2][cols], or the CTA's own ws row for very long rows
    __shared__ double red[2 * 2 * 32];
    int phase = 0;
    double* part = part_in_ws ? ws + (size_t)blockIdx.x * 2 * cols : part_sm;
    for (int j = threadIdx.x; j < 2 * cols; j += blockDim.x) part[j] = 0.0;
    const double inv_m = 1.0 / (double)cols;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float* gr = dy + r * cols;
        const float* yr = y + r * cols;
        double s[2] = {0.0, 0.0};
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            double gg = (double)gr[j] * (double)gamma[j];
            double xh = ((double)yr[j] - (double)beta[j]) / (double)gamma[j];
            s[0] += gg;
            s[1] += gg * xh;
        }
        block_sum<2>(s, red, phase);
        const double c1 = s[0] * inv_m, c2 = s[1] * inv_m, rs = (double)rstd[r];
        for (int j = threadIdx.x; j < cols; j += blockDim.x) {
            double g = (double)gr[j];
            double xh = ((double)yr[j] - (double)beta[j]) / (double)gamma[j];
            const float o = (float)((g * (double)gamma[j] - c1 - xh * c2) * rs);
            dx[r * cols + j] = o;
            if (dproj) {  // fused dropout backward (see ln_bwd_vec_kernel, DROP)
                const int64_t e = r * cols + j;
                dproj[e] = ((mask[e >> 5] >> (e & 31)) & 1u) ? (float)((double)o * scale) : 0.0f;
            }
            part[j] += g * xh;
            part[cols + j] += g;
        }
    }
    if (part_in_ws) return;  // each column's partial is one thread's: already in place
    __syncthreads();
    double* wg = ws + (size_t)blockIdx.x * 2 * cols;
    for (int j = threadIdx.x; j < 2 * cols; j += blockDim.x) wg[j] = part[j];
}

// Stage 1, long rows on a thread-block CLUSTER (2048 < cols <= 16384): the K
// CTAs of a cluster split the columns (CTA rank q owns the slice [q*sw,
// q*sw + sw), sw <= 4*NT, thread t the float4 at column q*sw + 4t) and walk the
// SAME row tiles, so each CTA is ln_bwd_vec_kernel on its slice -- TMA ring of
// kRowsB-row tiles (one bulk copy per row slice), gamma/beta and the fp64
// dgamma/dbeta column partials in registers -- and the two row sums of a tile
// are the fixed-order sum of the K CTAs' block sums, exchanged through
// distributed shared memory.  The exchange is decoupled, one tile ahead: in
// iteration i a CTA (A) computes its block sums of tile i+1 and PUSHES them
// into slot (i+1)%4 of every cluster CTA's inbox (st.shared::cluster, then a
// release-arrive on that CTA's inbox mbarrier, K arrivals per phase), then
// (B) waits for its own inbox slot i%4 -- filled by the peers one iteration
// earlier -- and produces tile i's dx and partials from the stage still in
// smem.  No cluster-wide barrier per tile: a CTA waits only for the peers'
// sums of a tile it has not computed on yet.  Slots: a peer pushes tile i+4
// into slot i%4 only after its B(i+2), which needs this CTA's push of tile
// i+2, made after this CTA's B(i) -- so 4 slots never overwrite unread sums.
// Stages: tile i (B), i+1 (A), i+2 in flight: 3-deep ring; tile t lives in
// stage t%3, and tile i+2 is loaded once B(i-1) has released its stage (at
// A(i+1)'s block barrier).
// The partial row of cluster c is ws[c] (its K CTAs write disjoint column
// slices), reduced by the usual stage 2.
constexpr int kStagesC = 3;
constexpr int kInbox = 4;

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster_f32(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TB_WAITC_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TB_WAITC_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

template <int NT, bool DROP>
__global__ void __launch_bounds__(NT, 1) ln_bwd_cluster_kernel(
    const float* __restrict__ dy, const float* __restrict__ y, const float* __restrict__ rstd,
    const float* __restrict__ gamma, const float* __restrict__ beta, float* __restrict__ dx,
    double* __restrict__ ws, int64_t rows, int cols, int sw, const uint32_t* __restrict__ mask,
    double scale, float* __restrict__ dproj) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch_persistent();
    extern __shared__ __align__(128) unsigned char dsm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(dsm);           // [kStagesC]
    uint64_t* inbar = full + kStagesC;                            // [kInbox]
    float* ring = reinterpret_cast<float*>(dsm + 128);
    __shared__ float red[2 * 2 * kRowsB * 32];
    __shared__ __align__(16) float inbox[kInbox][8][2 * kRowsB];  // [slot][rank][s1, s2 per row]
    int phase = 0;
    const int K = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
    const int64_t cid = blockIdx.x / K, ncl = gridDim.x / K;
    const int c0 = q * sw;                        // first column of the slice
    const int width = max(0, min(sw, cols - c0));  // columns of the slice (% 4 == 0)
    const int tile_floats = kRowsB * sw;          // per tensor; a stage holds dy then y
    const int64_t ntiles = (rows + kRowsB - 1) / kRowsB;
    const int n = cid < ntiles ? (int)((ntiles - 1 - cid) / ncl + 1) : 0;  // this cluster's tiles
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesC; ++s) mbar_init(&full[s], 1);
        for (int s = 0; s < kInbox; ++s) mbar_init(&inbar[s], (uint32_t)K);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int i, int s) {  // local tile i into stage s
        const int64_t r0 = (cid + (int64_t)i * ncl) * kRowsB;
        const int nr = (int)min((int64_t)kRowsB, rows - r0);
        const uint32_t bytes = (uint32_t)width * 4u;
        mbar_expect_tx(&full[s], 2 * nr * bytes);
        for (int j = 0; j < nr; ++j) {
            bulk_g2s(ring + (2 * s) * tile_floats + j * sw, dy + (r0 + j) * cols + c0, bytes, &full[s]);
            bulk_g2s(ring + (2 * s + 1) * tile_floats + j * sw, y + (r0 + j) * cols + c0, bytes,
                     &full[s]);
        }
    };
    if (threadIdx.x == 0 && width > 0) {
        for (int i = 0; i < kStagesC && i < n; ++i) issue(i, i);
    }
    const int cg4 = threadIdx.x;  // float4 column group within the slice
    const bool act = 4 * cg4 < width;
    const int col = c0 + 4 * cg4;
    float gm[4], bt[4], igf[4];
    double pg[4], pb[4];
    {
        float4 g = make_float4(1.f, 1.f, 1.f, 1.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act) {
            g = *reinterpret_cast<const float4*>(gamma + col);
            b = *reinterpret_cast<const float4*>(beta + col);
        }
        const float ga[4] = {g.x, g.y, g.z, g.w}, ba[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            gm[k] = ga[k];
            bt[k] = ba[k];
            igf[k] = (float)(1.0 / (double)ga[k]);
            pg[k] = 0.0;
            pb[k] = 0.0;
        }
    }
    const float inv_m = 1.0f / (float)cols;
    cluster.sync();  // every CTA's inbox barriers are initialised before the first push
    // A(i): block sums of local tile i from its stage, pushed to every CTA's inbox
    auto phase_a = [&](int i) {
        const int st = i % kStagesC;
        const int64_t r0 = (cid + (int64_t)i * ncl) * kRowsB;
        if (width > 0) mbar_wait(&full[st], (uint32_t)((i / kStagesC) & 1));
        const float* gs = ring + (2 * st) * tile_floats;
        const float* ys = ring + (2 * st + 1) * tile_floats;
        float s[2 * kRowsB];
#pragma unroll
        for (int j = 0; j < kRowsB; ++j) {
            float s1 = 0.0f, s2 = 0.0f;
            if (r0 + j < rows && act) {
                const float4 gv = reinterpret_cast<const float4*>(gs + j * sw)[cg4];
                const float4 yv = reinterpret_cast<const float4*>(ys + j * sw)[cg4];
                const float ga[4] = {gv.x, gv.y, gv.z, gv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float gg = ga[k] * gm[k];
                    const float xh = (ya[k] - bt[k]) * igf[k];
                    s1 += gg;
                    s2 = fmaf(gg, xh, s2);
                }
            }
            s[2 * j] = s1;
            s[2 * j + 1] = s2;
        }
        block_sum<2 * kRowsB>(s, red, phase);  // (its barrier also ends the previous B)
        // lane p of warp 1 pushes to cluster CTA p (in parallel: one remote
        // round trip, not K; the release-arrive waits for its own stores only)
        if ((threadIdx.x >> 5) == 1 && (threadIdx.x & 31) < K) {
            const uint32_t p = threadIdx.x & 31;
            const int slot = i % kInbox;
            const uint32_t ra = mapa_u32(smem_u32(&inbox[slot][q][0]), p);
#pragma unroll
            for (int j = 0; j < 2 * kRowsB; ++j) st_cluster_f32(ra + 4 * j, s[j]);
            mbar_arrive_remote(mapa_u32(smem_u32(&inbar[slot]), p));
        }
        // phase_a(i) runs in iteration i-1, BEFORE B(i-1): the stage that is
        // free here is tile i-2's (read by B(i-2) in the previous iteration;
        // the block barrier above orders every thread's reads of it) -> tile i+1
        if (threadIdx.x == 0 && i >= 2 && i + 1 < n && width > 0) {
            fence_proxy_async_smem();
            issue(i + 1, (i - 2) % kStagesC);
        }
    };
    float rs_nx[kRowsB];
    uint32_t mw_nx[kRowsB];
    auto prefetch = [&](int i) {
        const int64_t r0 = (cid + (int64_t)i * ncl) * kRowsB;
#pragma unroll
        for (int j = 0; j < kRowsB; ++j) {
            const bool in = i < n && r0 + j < rows;
            rs_nx[j] = in ? __ldg(rstd + r0 + j) : 0.f;
            mw_nx[j] = (DROP && in && act) ? __ldg(mask + (((r0 + j) * cols + col) >> 5)) : 0u;
        }
    };
    if (n > 0) {
        phase_a(0);
        prefetch(0);
    }
    for (int i = 0; i < n; ++i) {
        float rsv[kRowsB];
        uint32_t mwv[kRowsB];
#pragma unroll
        for (int j = 0; j < kRowsB; ++j) {
            rsv[j] = rs_nx[j];
            mwv[j] = mw_nx[j];
        }
        if (i + 1 < n) {
            prefetch(i + 1);
            phase_a(i + 1);
        }
        // B(i): the K CTAs' sums of tile i, then dx / d(proj) / partials
        const int slot = i % kInbox;
        // one acquiring waiter per warp (a cluster-scope acquire invalidates
        // L1: once per warp, not per thread); __syncwarp orders its lanes after it
        if ((threadIdx.x & 31) == 0) mbar_wait_cluster(&inbar[slot], (uint32_t)((i / kInbox) & 1));
        __syncwarp();
        float s[2 * kRowsB];
#pragma unroll
        for (int j = 0; j < 2 * kRowsB; ++j) s[j] = inbox[slot][0][j];
        for (int p = 1; p < K; ++p) {  // fixed rank order: identical sums in every CTA
#pragma unroll
            for (int j = 0; j < 2 * kRowsB; ++j) s[j] += inbox[slot][p][j];
        }
        const int st = i % kStagesC;
        const int64_t r0 = (cid + (int64_t)i * ncl) * kRowsB;
        const float* gs = ring + (2 * st) * tile_floats;
        const float* ys = ring + (2 * st + 1) * tile_floats;
#pragma unroll
        for (int j = 0; j < kRowsB; ++j) {
            if (r0 + j >= rows || !act) continue;
            const float c1 = s[2 * j] * inv_m, c2 = s[2 * j + 1] * inv_m;
            const float4 gv = reinterpret_cast<const float4*>(gs + j * sw)[cg4];
            const float4 yv = reinterpret_cast<const float4*>(ys + j * sw)[cg4];
            const float ga[4] = {gv.x, gv.y, gv.z, gv.w}, ya[4] = {yv.x, yv.y, yv.z, yv.w};
            float o[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float xh = (ya[k] - bt[k]) * igf[k];
                o[k] = (fmaf(ga[k], gm[k], -c1) - xh * c2) * rsv[j];
                const double gd = (double)ga[k];
                pg[k] = fma(gd, (double)ya[k], pg[k]);
                pb[k] += gd;
            }
            const int64_t e = (r0 + j) * cols + col;
            st_stream(reinterpret_cast<float4*>(dx + e), make_float4(o[0], o[1], o[2], o[3]));
            if (DROP) {
                const uint32_t nb = (mwv[j] >> (e & 31)) & 0xfu;
                float4 dp;
                dp.x = (nb & 1u) ? (float)((double)o[0] * scale) : 0.0f;
                dp.y = (nb & 2u) ? (float)((double)o[1] * scale) : 0.0f;
                dp.z = (nb & 4u) ? (float)((double)o[2] * scale) : 0.0f;
                dp.w = (nb & 8u) ? (float)((double)o[3] * scale) : 0.0f;
                st_stream(reinterpret_cast<float4*>(dproj + e), dp);
            }
        }
    }
    if (act) {
        double* wg = ws + (size_t)cid * 2 * cols;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            wg[col + k] = fma(-(double)bt[k], pb[k], pg[k]) * (1.0 / (double)gm[k]);
            wg[cols + col + k] = pb[k];
        }
    }
    // every push into this CTA's inbox was consumed above (B(n-1) waited for
    // the last), and this CTA's own pushes completed before its arrives: no
    // DSMEM access can target an exited CTA
}

// CTA size of the cluster backward: 256 threads (1024 columns per CTA, two
// CTAs per SM) while K <= 8 covers the row, 512 beyond (A/B with the
// decoupled exchange: H = 4096 / 8192 at 0.56 / 0.50 vs 0.53 / 0.48)
#ifndef TM_LN_CLUSTER_NT_MAX
#define TM_LN_CLUSTER_NT_MAX 512
#endif
inline int cluster_nt(int64_t cols) {
    return cols <= 8 * 4 * 256 ? 256 : TM_LN_CLUSTER_NT_MAX;
}
// cluster size and slice width for a long row: K = ceil(cols / (4*NT)), the
// slice rounded up to a multiple of 4 columns
inline int cluster_k(int64_t cols) {
    const int nt = cluster_nt(cols);
    return (int)((cols + 4 * nt - 1) / (4 * nt));
}
inline int cluster_sw(int64_t cols) {
    const int k = cluster_k(cols);
    return (int)(((cols + k - 1) / k + 3) / 4 * 4);
}
size_t bwd_cluster_smem(int64_t cols) {
    return 128 + (size_t)kStagesC * 2 * kRowsB * cluster_sw(cols) * sizeof(float);
}
const void* bwd_cluster_fn(int64_t cols, bool drop) {
    if (cluster_nt(cols) == 256)
        return drop ? (const void*)ln_bwd_cluster_kernel<256, true>
                    : (const void*)ln_bwd_cluster_kernel<256, false>;
    return drop ? (const void*)ln_bwd_cluster_kernel<512, true>
                : (const void*)ln_bwd_cluster_kernel<512, false>;
}

// Stage 2: out[j] = sum over CTAs c (fixed order) of ws[c][j], j < 2*cols.
// A 32 x 32 block: column lane tx owns output j0 + tx, slice ty sums the
// partial rows c = ty, ty + 32, ... (coalesced 256-byte rows); all of a
// slice's loads are issued before the first add (up to 16 in registers), and
// the 32 slices are then added in a fixed order by ty == 0 -- bitwise
// reproducible.  Launched as a programmatic dependent of stage 1 (PDL): the
// launch overlaps stage 1's tail and griddepcontrol.wait orders the reads.
__global__ void __launch_bounds__(1024) ln_param_reduce_kernel(const double* __restrict__ ws,
                                                               int nparts, int cols,
                                                               float* __restrict__ dgamma,
                                                               float* __restrict__ dbeta) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    __shared__ double part[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t total = 2 * (int64_t)cols;
    const int64_t j = (int64_t)blockIdx.x * 32 + tx;
    double acc = 0.0;
    if (j < total) {
        constexpr int L = 16;
        int c0 = ty;
        for (; c0 < nparts; c0 += 32 * L) {
            double a[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const int c = c0 + 32 * l;
                a[l] = c < nparts ? ws[(size_t)c * total + j] : 0.0;
            }
#pragma unroll
            for (int l = 0; l < L; ++l) acc += a[l];  // adding +0.0 past the end is exact
        }
    }
    part[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && j < total) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < 32; ++k) v += part[k][tx];
        if (j < cols) dgamma[j] = (float)v; else dbeta[j - cols] = (float)v;
    }
}

// Stage 2, narrow column blocks: 8 outputs (one 64-byte row segment = two
// full sectors) x 64 partial-row slices per 512-thread CTA, so the grid is
// 2*cols/8 CTAs (256 at H = 1024) instead of 2*cols/32 one-per-SM CTAs, and
// each thread has a handful of loads in flight at once.  The 64 slice sums
// are combined by a fixed shuffle tree inside each warp (4 slices) and then
// over the 16 warps in a fixed order -- the same tree every run: bitwise
// reproducible (fp addition is commutative, so both xor partners hold the
// same bits).
#ifndef TM_LN_REDUCE_NARROW
#define TM_LN_REDUCE_NARROW 1
#endif
#ifndef TM_LN_REDUCE_COLS
#define TM_LN_REDUCE_COLS 8
#endif
constexpr int kRedCols = TM_LN_REDUCE_COLS, kRedSlices = 512 / kRedCols;
static_assert(kRedCols >= 1 && kRedCols <= 16 && (kRedCols & (kRedCols - 1)) == 0, "");
__global__ void __launch_bounds__(kRedCols * kRedSlices) ln_param_reduce8_kernel(
    const double* __restrict__ ws, int nparts, int cols, float* __restrict__ dgamma,
    float* __restrict__ dbeta) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    constexpr int kWarps = kRedCols * kRedSlices / 32;
    __shared__ double part[kWarps][kRedCols];
    const int tx = threadIdx.x % kRedCols, ty = threadIdx.x / kRedCols;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t total = 2 * (int64_t)cols;
    const int64_t j = (int64_t)blockIdx.x * kRedCols + tx;
    double acc = 0.0;
    if (j < total) {
        constexpr int L = 8;
        for (int c0 = ty; c0 < nparts; c0 += kRedSlices * L) {
            double a[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const int c = c0 + kRedSlices * l;
                a[l] = c < nparts ? ws[(size_t)c * total + j] : 0.0;
            }
#pragma unroll
            for (int l = 0; l < L; ++l) acc += a[l];  // adding +0.0 past the end is exact
        }
    }
#pragma unroll
    for (int m = kRedCols; m < 32; m <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (lane < kRedCols) part[w][lane] = acc;
    __syncthreads();
    if (w == 0) {  // lane = q * kRedCols + column: warps q, q + Q, q + 2Q, ..., then the tree
        constexpr int Q = 32 / kRedCols;
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < kWarps / Q; ++k) v += part[lane / kRedCols + Q * k][lane % kRedCols];
#pragma unroll
        for (int m = kRedCols; m < 32; m <<= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
        const int64_t jo = (int64_t)blockIdx.x * kRedCols + lane;
        if (lane < kRedCols && jo < total) {
            if (jo < cols) dgamma[jo] = (float)v; else dbeta[jo - cols] = (float)v;
        }
    }
}

// Stage 2 fused with the cross-rank sum (the path's one collective, SURVEY
// 8e) over peer memory, in place of ln_param_reduce_kernel + an all-reduce.
// CTA cb owns outputs j in [32 cb, 32 cb + 32) of the 2*cols (dgamma | dbeta):
//  1. its local fixed-order sum over the nparts stage-1 partial rows (fp64);
//  2. the 32 values are stored into slot [par][rank] of EVERY rank's inbox
//     (P2P stores over NVLink; the own inbox included);
//  3. one thread: system-scope fence, then flag[par][rank][cb] = epoch on
//     every rank (st.release.sys);
//  4. one thread waits for flag[par][s][cb] == epoch for all s on its own
//     rank (ld.acquire.sys, bounded spin: a missing peer sets *status and
//     the kernel finishes instead of hanging);
//  5. the final value is the sum over s = 0 .. world-1 IN RANK ORDER of the
//     inbox slots: every rank computes identical bits, independent of the
//     arrival order (bitwise reproducible, unlike a generic all-reduce).
// No grid-wide barrier: each column block synchronises only with the same
// block on the other ranks.  par = epoch & 1 double-buffers the inbox: a
// rank can only reach epoch e+2 (parity reuse) after every peer has set its
// e+1 flags, i.e. after every peer finished reading its epoch-e slots.
constexpr int kPeerCols = 32;
constexpr uint64_t kPeerDefaultTimeoutNs = 30ull * 1000000000ull;  // 30 s
constexpr int kPeerRowGroups = 8;

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Failure semantics (a straggler or a dead peer): the wait is bounded by
// timeout_ns (caller-chosen; the library default is 30 s, NCCL-like
// patience for checkpoint saves / data stalls, yet finite so the GPU is never
// hung); a block whose peers do not all arrive sets *status =
// TEMPO_ERR_STATE and writes NaN to its dgamma/dbeta outputs instead of a
// partial sum (the inbox may hold another epoch's data).  *status is
// sticky: every later exchange on this rank sees it, skips the exchange
// (no flags published, no waiting) and writes NaN, so a broken group fails
// loudly until it is rebuilt -- never silently wrong.
__device__ __forceinline__ int32_t ld_volatile_i32(const int32_t* p) {
    return *reinterpret_cast<const volatile int32_t*>(p);
}

__global__ void __launch_bounds__(kPeerCols * kPeerRowGroups) ln_param_reduce_peer_kernel(
    const double* __restrict__ ws, int nparts, int cols, int rank, int world,
    double* const* __restrict__ inbox, uint32_t* const* __restrict__ flags, uint32_t epoch,
    uint64_t timeout_ns, float* __restrict__ dgamma, float* __restrict__ dbeta,
    int32_t* __restrict__ status) {
    grid_dep_wait();
    __shared__ double part[kPeerRowGroups][kPeerCols + 1];
    __shared__ int failed;
    const int tx = threadIdx.x % kPeerCols, ty = threadIdx.x / kPeerCols;
    const int64_t total = 2 * (int64_t)cols;
    const int cb = blockIdx.x, ncb = gridDim.x;
    const int64_t j = (int64_t)cb * kPeerCols + tx;
    const int par = (int)(epoch & 1u);
    const int64_t tstride = (int64_t)ncb * kPeerCols;  // inbox slot stride (padded)
    if (threadIdx.x == 0) failed = ld_volatile_i32(status) != 0;  // sticky: an earlier failure
    __syncthreads();
    if (failed) {
        if (ty == 0 && j < total) {
            if (j < cols) dgamma[j] = __int_as_float(0x7fc00000); else dbeta[j - cols] = __int_as_float(0x7fc00000);
        }
        return;
    }
    double acc = 0.0;
    if (j < total)
        for (int c = ty; c < nparts; c += kPeerRowGroups) acc += ws[(size_t)c * total + j];
    part[ty][tx] = acc;
    __syncthreads();
    if (ty == 0) {
        double v = 0.0;
#pragma unroll
        for (int k = 0; k < kPeerRowGroups; ++k) v += part[k][tx];
        // slot [par][rank] of every rank's inbox ([2][world][tstride] doubles)
        for (int p = 0; p < world; ++p) inbox[p][((size_t)par * world + rank) * tstride + j] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int p = 0; p < world; ++p)
            st_release_sys(flags[p] + ((size_t)par * world + rank) * ncb + cb, epoch);
        const uint32_t* mine = flags[rank] + (size_t)par * world * ncb + cb;
        const uint64_t t0 = globaltimer_ns();
        for (int s = 0; s < world && !failed; ++s) {
            while (ld_acquire_sys(mine + (size_t)s * ncb) != epoch) {
                if (globaltimer_ns() - t0 > timeout_ns) {  // a peer never arrived
                    atomicExch(status, TEMPO_ERR_STATE);
                    failed = 1;
                    break;
                }
                __nanosleep(128);
            }
        }
    }
    __syncthreads();
    if (ty == 0 && j < cols * 2) {
        const double* my = inbox[rank] + (size_t)par * world * tstride;
        double v = 0.0;
        for (int s = 0; s < world; ++s) v += __ldcg(my + (size_t)s * tstride + j);
        const float out = failed ? __int_as_float(0x7fc00000) : (float)v;  // NaN: not a partial sum
        if (j < cols) dgamma[j] = out; else dbeta[j - cols] = out;
    }
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bool use_vec(int64_t cols, const void* a, const void* b, const void* c, const void* d,
             const void* e, int64_t max_cols = 4 * kMaxThreads) {
    return cols % 4 == 0 && cols <= max_cols && aligned16(a) && aligned16(b) &&
           aligned16(c) && aligned16(d) && aligned16(e);
}

int vec_threads(int64_t cols) { return (int)(((cols / 4) + 31) / 32 * 32); }
// backward: two float4 column groups per thread when cols % 8 == 0
int bwd_cpt(int64_t cols) { return (TM_LN_BWD_CPT2 && cols % 8 == 0) ? 2 : 1; }
int bwd_threads(int64_t cols) {
    return (int)(((cols / 4 + bwd_cpt(cols) - 1) / bwd_cpt(cols) + 31) / 32 * 32);
}
const void* bwd_vec_fn(int64_t cols, bool drop = false) {
    const int t = bwd_threads(cols);
    if (t > kMaxThreads)  // (only with TM_LN_BWD_WIDE: use_vec / cluster_bwd_ok)
        return drop ? (const void*)ln_bwd_vec_kernel<kWideThreads, 1, true, kRowsW>
                    : (const void*)ln_bwd_vec_kernel<kWideThreads, 1, false, kRowsW>;
#if TM_LN_BWD_CPT2  // (off by default: measured slower; not instantiated)
    if (bwd_cpt(cols) == 2)
        return t <= 256 ? (const void*)ln_bwd_vec_kernel<256, 2>
                        : (const void*)ln_bwd_vec_kernel<kMaxThreads, 2>;
#endif
    if (drop)
        return t <= 256 ? (const void*)ln_bwd_vec_kernel<256, 1, true>
                        : (const void*)ln_bwd_vec_kernel<kMaxThreads, 1, true>;
    return t <= 256 ? (const void*)ln_bwd_vec_kernel<256, 1>
                    : (const void*)ln_bwd_vec_kernel<kMaxThreads, 1>;
}

// Stage-1 grid for the backward: its CTA count is also the number of
// partial rows in the workspace, so it depends only on (rows, cols, device).
size_t fwd_smem(int64_t cols) { return 128 + (size_t)kStages * kRows * cols * sizeof(float); }
size_t bwd_smem(int64_t cols) {
    const int rows = cols > 4 * kMaxThreads ? kRowsW : kRowsB;
    return 128 + (size_t)kStagesB * 2 * rows * cols * sizeof(float);
}

// long-row paths (cols % 128 == 0): forward 2048 < cols <= 16384 (the fused
// dropout -> add -> LayerNorm forward from 1024), backward up to 8192
bool long_fwd_ok(int64_t cols, int64_t min_cols) {
    return cols % 128 == 0 && cols > min_cols && cols <= 16 * kLongVPL * 128;
}
bool cluster_bwd_ok(int64_t cols) {
    return cols % 4 == 0 && cols > kVecMaxCols && cluster_k(cols) <= 8;
}
// CTAs (a multiple of K): as many clusters as can be co-resident -- a
// persistent grid with clusters waiting for a second wave would serialise
// (cluster placement is per GPC, so this is below SMs / K)
int bwd_cluster_grid(int64_t rows, int64_t cols) {
    static std::mutex mu;
    static std::map<std::pair<int, int64_t>, int> cache;  // (device, cols) -> max active clusters
    const int k = cluster_k(cols);
    const int64_t ntiles = (rows + kRowsB - 1) / kRowsB;
    const void* kf = bwd_cluster_fn(cols, false);
    const int nt = cluster_nt(cols);
    const size_t smem = bwd_cluster_smem(cols);
    (void)grid_for(kf, nt, smem, 1);  // dynamic smem opt-in
    int dev = 0;
    cudaGetDevice(&dev);
    int maxcl = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find({dev, cols});
        if (it != cache.end()) {
            maxcl = it->second;
        } else {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3((unsigned)(k * 148));
            cfg.blockDim = dim3((unsigned)nt);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = (unsigned)k;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&maxcl, kf, &cfg) != cudaSuccess || maxcl < 1) {
                cudaGetLastError();
                maxcl = 1;
            }
            cache[{dev, cols}] = maxcl;
        }
    }
    const int64_t ncl = std::min<int64_t>(maxcl, ntiles);
    return (int)(ncl < 1 ? 1 : ncl) * k;
}

// generic backward: partials in smem up to this many bytes, else in the
// CTA's own workspace row (global, L2-resident)
constexpr size_t kGenericPartSmem = 160 * 1024;
size_t generic_bwd_smem(int64_t cols) {
    const size_t b = (size_t)2 * cols * sizeof(double);
    return b <= kGenericPartSmem ? b : 0;
}

int bwd_grid(int64_t rows, int64_t cols, bool vec) {
    const int tr = cols > 4 * kMaxThreads ? kRowsW : kRowsB;  // rows per tile
    int64_t work = vec ? (rows + tr - 1) / tr : rows;
    const void* k = !vec ? (const void*)ln_bwd_generic_kernel : bwd_vec_fn(cols);
    int block = vec ? bwd_threads(cols) : 256;
    size_t smem = vec ? bwd_smem(cols) : generic_bwd_smem(cols);
    return grid_for(k, block, smem, work);
}

template <int MODE>
cudaError_t launch_ln_long_fwd(const float* x, const float* res, uint32_t* mask, double scale,
                               uint64_t thresh, uint64_t seed, uint64_t offset,
                               const float* gamma, const float* beta, double eps, float* y,
                               float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                               cudaStream_t st) {
    const int nch = (int)(cols / 128);
    const int T = MODE == 0 ? 1 : 2;
    const size_t smem = lnl_smem(cols, T);
    const int ns = lnl_stages(cols, T);
#define TB_LNL(W)                                                                            \
    case W: {                                                                                \
        auto k = ln_fwd_long_kernel<W, MODE>;                                                \
        int grid = grid_for((const void*)k, W * 32, smem, rows);                             \
        launch(k, grid, W * 32, smem, st)(x, res, mask, scale, thresh, seed, offset, gamma, beta, \
                                          eps, y, rstd, rows, nch, ns, dev_status);          \
        break;                                                                               \
    }
    switch (lnl_fwd_warps(nch)) {
        TB_LNL(1)
        TB_LNL(2)
        TB_LNL(4)
        TB_LNL(8)
        TB_LNL(16)
        default: return cudaErrorInvalidValue;
    }
#undef TB_LNL
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_ln_fwd(const float* x, const float* gamma, const float* beta, double eps,
                          float* y, float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                          cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    const int vpl = (int)(cols / 128);
    const int64_t long_min = rows * cols < TM_LN_LONG_SMALL_N ? 0 : TM_LN_LONG_MIN;
    if (cols % 128 == 0 && (vpl == 6 || vpl == 8 || vpl == 4 || vpl == 2) &&
        cols <= long_min && use_vec(cols, x, y, gamma, beta, x)) {
        const size_t smem = warp_fwd_smem(vpl);
#define TB_LNW(V)                                                                            \
    case V: {                                                                                \
        auto k = ln_fwd_warp_kernel<V>;                                                      \
        int grid = grid_for((const void*)k, kWWarps * 32, smem, (rows + kWWarps - 1) / kWWarps, 0, TM_LN_WAVES); \
        launch(k, grid, kWWarps * 32, smem, st)(x, gamma, beta, eps, y, rstd, rows, dev_status); \
        break;                                                                               \
    }
        switch (vpl) {
            TB_LNW(2)
            TB_LNW(4)
            TB_LNW(6)
            TB_LNW(8)
        }
#undef TB_LNW
        return cudaGetLastError();
    }
    if (long_fwd_ok(cols, long_min) && aligned16(x) && aligned16(y) && aligned16(gamma) &&
        aligned16(beta))
        return launch_ln_long_fwd<0>(x, nullptr, nullptr, 1.0, 0, 0, 0, gamma, beta, eps, y, rstd,
                                     rows, cols, dev_status, st);
    if (use_vec(cols, x, y, gamma, beta, x)) {
        int block = vec_threads(cols);
        size_t smem = fwd_smem(cols);
        auto k = block <= 256 ? ln_fwd_vec_kernel<256> : ln_fwd_vec_kernel<kMaxThreads>;
        int grid = grid_for((const void*)k, block, smem, (rows + kRows - 1) / kRows);
        launch(k, grid, block, smem, st)(x, gamma, beta, eps, y, rstd, rows, (int)cols, dev_status);
    } else {
        int grid = grid_for((const void*)ln_fwd_generic_kernel, 256, 0, rows);
        launch(ln_fwd_generic_kernel, grid, 256, 0, st)(x, gamma, beta, eps, y, rstd, rows,
                                                     (int)cols, dev_status);
    }
    return cudaGetLastError();
}

size_t ln_peer_inbox_bytes(int world, int64_t cols) {
    const int64_t ncb = (2 * cols + kPeerCols - 1) / kPeerCols;
    return (size_t)2 * world * (size_t)(ncb * kPeerCols) * sizeof(double);
}
size_t ln_peer_flag_bytes(int world, int64_t cols) {
    const int64_t ncb = (2 * cols + kPeerCols - 1) / kPeerCols;
    return (size_t)2 * world * (size_t)ncb * sizeof(uint32_t);
}

cudaError_t launch_ln_param_reduce_peer(const double* partials, int64_t nparts, int64_t cols,
                                        const LnPeer& peer, float* dgamma, float* dbeta,
                                        cudaStream_t st) {
    if (cols == 0) return cudaSuccess;
    const int ncb = (int)((2 * cols + kPeerCols - 1) / kPeerCols);
    const uint64_t tmo = peer.timeout_ms ? (uint64_t)peer.timeout_ms * 1000000ull
                                         : kPeerDefaultTimeoutNs;
    return launch_pdl((const void*)ln_param_reduce_peer_kernel, ncb, kPeerCols * kPeerRowGroups, 0,
                      st, partials, (int)nparts, (int)cols, peer.rank, peer.world, peer.inbox,
                      peer.flags, peer.epoch, tmo, dgamma, dbeta, peer.status);
}

size_t ln_bwd_workspace(int64_t rows, int64_t cols) {
    if (rows == 0 || cols == 0) return 0;
    // The vector/generic choice also depends on pointer alignment; size for
    // the larger of the two grids.
    int gv = (cols % 4 == 0 && cols <= kVecMaxCols) ? bwd_grid(rows, cols, true) : 0;
    int gg = bwd_grid(rows, cols, false);
    int gl = cluster_bwd_ok(cols) ? bwd_cluster_grid(rows, cols) / cluster_k(cols) : 0;
    int g = gv > gg ? gv : gg;
    g = gl > g ? gl : g;
    return (size_t)g * 2 * (size_t)cols * sizeof(double);
}

cudaError_t launch_ln_bwd(const float* dy, const float* y, const float* rstd, const float* gamma,
                          const float* beta, float* dx, float* dgamma, float* dbeta, void* ws,
                          int64_t rows, int64_t cols, cudaStream_t st, const LnPeer* peer,
                          const uint32_t* mask, double scale, float* dproj, int64_t* nparts_out) {
    if (nparts_out) *nparts_out = 0;
    if (cols == 0) return cudaSuccess;
    if (rows == 0 && nparts_out) return cudaSuccess;  // no partial rows
    if (rows == 0) {
        if (peer) return launch_ln_param_reduce_peer(nullptr, 0, cols, *peer, dgamma, dbeta, st);
        cudaMemsetAsync(dgamma, 0, cols * sizeof(float), st);
        cudaMemsetAsync(dbeta, 0, cols * sizeof(float), st);
        return cudaGetLastError();
    }
    const bool drop = dproj != nullptr;
    const bool aligned = aligned16(dy) && aligned16(y) && aligned16(dx) && aligned16(gamma) &&
                         aligned16(beta) && (!drop || aligned16(dproj));
    const bool clu = cluster_bwd_ok(cols) && aligned;
    const bool vec = !clu && use_vec(cols, dy, y, dx, gamma, beta, kVecMaxCols) &&
                     (!drop || aligned16(dproj));
    // the grid (= the workspace's partial rows) is the plain kernel's, also
    // for the fused variant, so one workspace query serves both
    const int grid = clu ? bwd_cluster_grid(rows, cols) / cluster_k(cols) : bwd_grid(rows, cols, vec);
    double* w = static_cast<double*>(ws);
    if (clu) {
        const int k = cluster_k(cols);
        using KFn = void (*)(const float*, const float*, const float*, const float*,
                             const float*, float*, double*, int64_t, int, int, const uint32_t*,
                             double, float*);
        KFn kf = reinterpret_cast<KFn>(const_cast<void*>(bwd_cluster_fn(cols, drop)));
        const int nt = cluster_nt(cols);
        const size_t smem = bwd_cluster_smem(cols);
        (void)grid_for((const void*)kf, nt, smem, grid * k);  // smem opt-in
        cudaError_t e = launch(kf, grid * k, nt, smem, st)
                            .cluster((unsigned)k)(dy, y, rstd, gamma, beta, dx, w, rows, (int)cols,
                                                  cluster_sw(cols), mask, scale, dproj);
        if (e != cudaSuccess) return e;
    } else if (vec) {
        using KFn = void (*)(const float*, const float*, const float*, const float*,
                             const float*, float*, double*, int64_t, int, const uint32_t*, double,
                             float*);
        KFn k = reinterpret_cast<KFn>(const_cast<void*>(bwd_vec_fn(cols, drop)));
        // grid_for also opts the kernel into its dynamic smem size
        if (drop) (void)grid_for((const void*)k, bwd_threads(cols), bwd_smem(cols), grid);
        launch(k, grid, bwd_threads(cols), bwd_smem(cols), st)(dy, y, rstd, gamma, beta, dx, w, rows,
                                                           (int)cols, mask, scale, dproj);
    } else {
        const size_t smem = generic_bwd_smem(cols);
        launch(ln_bwd_generic_kernel, grid, 256, smem, st)(dy, y, rstd, gamma, beta, dx, w, rows,
                                                       (int)cols, mask, scale, dproj,
                                                       smem == 0 ? 1 : 0);
    }
    if (nparts_out) {
        *nparts_out = grid;
        return cudaGetLastError();
    }
    if (peer) return launch_ln_param_reduce_peer(w, grid, cols, *peer, dgamma, dbeta, st);
    return launch_ln_param_reduce(w, grid, cols, dgamma, dbeta, st);
}

cudaError_t launch_ln_param_reduce(const double* partials, int64_t nparts, int64_t cols,
                                   float* dgamma, float* dbeta, cudaStream_t st) {
    if (cols == 0) return cudaSuccess;
    if (nparts == 0) {
        cudaMemsetAsync(dgamma, 0, cols * sizeof(float), st);
        cudaMemsetAsync(dbeta, 0, cols * sizeof(float), st);
        return cudaGetLastError();
    }
    if (TM_LN_REDUCE_NARROW)
        return launch_pdl((const void*)ln_param_reduce8_kernel,
                          (int)((2 * cols + kRedCols - 1) / kRedCols), kRedCols * kRedSlices, 0,
                          st, partials, (int)nparts, (int)cols, dgamma, dbeta);
    const int rgrid = (int)((2 * cols + 31) / 32);
    return launch_pdl((const void*)ln_param_reduce_kernel, rgrid, 1024, 0, st, partials,
                      (int)nparts, (int)cols, dgamma, dbeta);
}

cudaError_t launch_dal_fwd(const float* proj, const float* res, double scale, uint64_t thresh,
                           int philox, uint32_t* mask, uint64_t seed, uint64_t offset,
                           const float* gamma, const float* beta, double eps, float* y,
                           float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                           cudaStream_t st) {
    if (rows == 0) return cudaSuccess;
    const int vpl = (int)(cols / 128);
    const bool warp_ok = cols % 128 == 0 && vpl >= 1 && vpl <= 8 && cols <= TM_DAL_LONG_MIN &&
                         aligned16(proj) &&
                         aligned16(res) && aligned16(y) && aligned16(gamma) && aligned16(beta) &&
                         (offset & 3u) == 0;
    if (warp_ok) {
        const size_t smem = dal_fwd_smem(vpl);
#define TB_DAL(V)                                                                            \
    case V: {                                                                                \
        auto k = philox ? dal_fwd_warp_kernel<V, 2> : dal_fwd_warp_kernel<V, 1>;              \
        int grid = grid_for((const void*)k, kWWarps * 32, smem, (rows + kWWarps - 1) / kWWarps, 0, TM_LN_WAVES); \
        launch(k, grid, kWWarps * 32, smem, st)(proj, res, mask, scale, thresh, seed, offset,    \
                                                gamma, beta, eps, y, rstd, rows, dev_status);    \
        break;                                                                               \
    }
        switch (vpl) {
            TB_DAL(1)
            TB_DAL(2)
            TB_DAL(3)
            TB_DAL(4)
            TB_DAL(5)
            TB_DAL(6)
            TB_DAL(7)
            TB_DAL(8)
        }
#undef TB_DAL
        return cudaGetLastError();
    }
    if (long_fwd_ok(cols, TM_DAL_LONG_MIN) && aligned16(proj) && aligned16(res) && aligned16(y) &&
        aligned16(gamma) && aligned16(beta) && (offset & 3u) == 0) {
        return philox ? launch_ln_long_fwd<2>(proj, res, mask, scale, thresh, seed, offset, gamma,
                                              beta, eps, y, rstd, rows, cols, dev_status, st)
                      : launch_ln_long_fwd<1>(proj, res, mask, scale, thresh, seed, offset, gamma,
                                              beta, eps, y, rstd, rows, cols, dev_status, st);
    }
    const size_t smem = (size_t)cols * sizeof(float) <= 160 * 1024 ? (size_t)cols * sizeof(float) : 0;
    int grid = grid_for((const void*)dal_fwd_generic_kernel, 256, smem, rows);
    launch(dal_fwd_generic_kernel, grid, 256, smem, st)(proj, res, mask, philox ? 2 : 1, scale,
                                                        thresh, seed, offset, gamma, beta, eps, y,
                                                        rstd, rows, (int)cols, dev_status,
                                                        smem == 0 ? 1 : 0);
    return cudaGetLastError();
}

}  // namespace tb
