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
// Layout: a warp owns 128-element chunks (one float4 per lane, 128-bit
// coalesced); the chunk's 4 mask words are packed with warp ballots.  A
// ragged tail (< 128 elements) or unaligned pointers take the scalar path
// (32 elements per warp step, one ballot = one mask word).
#include "common.cuh"
#include "gelu_math.h"
#include "gelu_fwd_slow.h"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kBlock = 256;
constexpr int kUnroll = 2;  // chunks in flight per warp

// ---------------------------------------------------------------- forward
__device__ __forceinline__ void gelu_fwd_scalar_words(const float* __restrict__ x,
                                                      float* __restrict__ y,
                                                      uint32_t* __restrict__ mask, int64_t n,
                                                      float xstar_gt, int64_t w_begin,
                                                      int64_t w_step, int lane) {
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = w_begin; w < nwords; w += w_step) {
        int64_t i = (w << 5) + lane;
        bool in = i < n;
        float xv = in ? x[i] : 0.0f;
        bool m = in && (xv >= xstar_gt);
        uint32_t bits = __ballot_sync(kFull, m);
        if (in) y[i] = tm_gelu_fwd(xv);
        if (lane == 0) mask[w] = bits;
    }
}

__global__ void __launch_bounds__(kBlock) gelu_fwd_vec_kernel(const float* __restrict__ x,
                                                              float* __restrict__ y,
                                                              uint32_t* __restrict__ mask,
                                                              int64_t n, float xstar_gt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 7;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    for (int64_t c0 = warp * kUnroll; c0 < nchunks; c0 += nwarps * kUnroll) {
        float4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (c0 + u < nchunks) v[u] = ld_stream(x4 + ((c0 + u) << 5) + lane);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (c0 + u < nchunks) {  // warp-uniform
                float4 o;
                o.x = tm_gelu_fwd(v[u].x);
                o.y = tm_gelu_fwd(v[u].y);
                o.z = tm_gelu_fwd(v[u].z);
                o.w = tm_gelu_fwd(v[u].w);
                uint32_t word = pack_chunk_bits(v[u].x >= xstar_gt, v[u].y >= xstar_gt,
                                                v[u].z >= xstar_gt, v[u].w >= xstar_gt, lane);
                st_stream(y4 + ((c0 + u) << 5) + lane, o);
                if (lane < 4) st_stream(mask + ((c0 + u) << 2) + lane, word);
            }
        }
    }
    // Ragged tail: words [4*nchunks, ceil(n/32)) on the last warp.
    if (warp == nwarps - 1) {
        gelu_fwd_scalar_words(x, y, mask, n, xstar_gt, nchunks << 2, 1, lane);
    }
}

__global__ void __launch_bounds__(kBlock) gelu_fwd_scalar_kernel(const float* __restrict__ x,
                                                                 float* __restrict__ y,
                                                                 uint32_t* __restrict__ mask,
                                                                 int64_t n, float xstar_gt) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    gelu_fwd_scalar_words(x, y, mask, n, xstar_gt, warp, nwarps, lane);
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
    __shared__ SmemTable st;
    extern __shared__ float coef[];
    load_table(t, st, coef);
    const int maxseg = max(t.nseg[0], t.nseg[1]);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    gelu_bwd_scalar_words(dy, y, mask, dx, n, t, st, coef, maxseg, warp, nwarps, lane);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

cudaError_t launch_gelu_fwd(const float* x, float* y, uint32_t* mask, int64_t n, float xstar_gt,
                            cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(x) && aligned16(y) && aligned16(mask);
    const void* k = vec ? (const void*)gelu_fwd_vec_kernel : (const void*)gelu_fwd_scalar_kernel;
    const int64_t warps_needed = vec ? ((n >> 7) + kUnroll - 1) / kUnroll + 1 : (n + 31) >> 5;
    int grid = grid_for(k, kBlock, 0, (warps_needed * 32 + kBlock - 1) / kBlock);
    if (vec) {
        gelu_fwd_vec_kernel<<<grid, kBlock, 0, st>>>(x, y, mask, n, xstar_gt);
    } else {
        gelu_fwd_scalar_kernel<<<grid, kBlock, 0, st>>>(x, y, mask, n, xstar_gt);
    }
    return cudaGetLastError();
}

cudaError_t launch_gelu_bwd(const float* dy, const float* y, const uint32_t* mask,
                            const GeluDevTable& t, float* dx, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const bool vec = aligned16(dy) && aligned16(y) && aligned16(dx) && aligned16(mask);
    const size_t smem = (size_t)(t.nseg[0] + t.nseg[1]) * t.stride * sizeof(float);
    const void* k = vec ? (const void*)gelu_bwd_vec_kernel : (const void*)gelu_bwd_scalar_kernel;
    const int64_t warps_needed = vec ? ((n >> 7) + kUnroll - 1) / kUnroll + 1 : (n + 31) >> 5;
    int grid = grid_for(k, kBlock, smem, (warps_needed * 32 + kBlock - 1) / kBlock);
    if (vec) {
        gelu_bwd_vec_kernel<<<grid, kBlock, smem, st>>>(dy, y, mask, dx, n, t);
    } else {
        gelu_bwd_scalar_kernel<<<grid, kBlock, smem, st>>>(dy, y, mask, dx, n, t);
    }
    return cudaGetLastError();
}

}  // namespace tb
