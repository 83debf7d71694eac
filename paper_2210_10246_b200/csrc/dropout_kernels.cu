// dropout_kernels.cu -- elementwise dropout with bit-packed masks (sm_100a).
//
// dropout_apply / dropout_backward (ops_reference.cpp:147-161 -> mask_scale
// kernels.cpp:285-295): out = mask ? in * (1/(1-p)) : 0, the product taken
// in fp64 and rounded once, so results are bit-exact with the reference on
// the same inputs.  Used for the hidden dropouts (ref_ops::dropout,
// ops_reference.cpp:214-225; encoder.cpp:180-184, 200-203) and as the
// "dropout-rescale" recompute rule (ops_tempo.cpp:17-26).
// HBM: read 4 B + write 4 B + 1 bit  = 8.125 B/elem each direction.
//
// Plus the BoolMask byte <-> bit converters (tensor.cpp:205-220).
#include "common.cuh"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kBlock = 256;
constexpr int kUnroll = 4;
#ifndef TM_DROPOUT_V8
#define TM_DROPOUT_V8 1
#endif
#ifndef TM_DROPOUT_PHILOX_WAVES
#define TM_DROPOUT_PHILOX_WAVES 1
#endif
#ifndef TM_DROPOUT_WAVES
#define TM_DROPOUT_WAVES 8
#endif
#ifndef TM_DROPOUT_U8
#define TM_DROPOUT_U8 2  // re-tuned at r1l: bwd 49.8 -> 47.3 us, bit-identical
#endif
#ifndef TM_DROPOUT_PHILOX_MINB
#define TM_DROPOUT_PHILOX_MINB 2  // min resident CTAs/SM for the Philox kernel (<= 128 regs; 1 lets ptxas take 138 and halves occupancy: 49 -> 58 us)
#endif
#ifndef TM_DROPOUT_PHILOX_U8
#define TM_DROPOUT_PHILOX_U8 TM_DROPOUT_U8
#endif

__device__ __forceinline__ float dscale(float v, double s) { return (float)((double)v * s); }

// PHILOX: generate + write the mask; otherwise read it.
template <bool PHILOX>
__device__ __forceinline__ void dropout_scalar_words(const float* __restrict__ x,
                                                     uint32_t* __restrict__ mask, double scale,
                                                     uint64_t thresh, uint64_t seed,
                                                     uint64_t offset, float* __restrict__ y,
                                                     int64_t n, int64_t w_begin, int64_t w_step,
                                                     int lane) {
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = w_begin; w < nwords; w += w_step) {
        const int64_t i = (w << 5) + lane;
        const bool in = i < n;
        bool keep;
        if (PHILOX) {
            keep = in && (uint64_t)philox_at(seed, offset + (uint64_t)i) >= thresh;
            uint32_t bits = __ballot_sync(kFull, keep);
            if (lane == 0) mask[w] = bits;
        } else {
            keep = (mask[w] >> lane) & 1u;
        }
        if (in) y[i] = keep ? dscale(x[i], scale) : 0.0f;
    }
}

template <bool PHILOX>
__global__ void __launch_bounds__(kBlock) dropout_fwd_vec_kernel(
    const float* __restrict__ x, uint32_t* __restrict__ mask, double scale, uint64_t thresh,
    uint64_t seed, uint64_t offset, float* __restrict__ y, int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 7;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    struct Group {
        float4 v[kUnroll];
        uint32_t nib[kUnroll];
    };
    auto load = [&](Group& G, int64_t c0, int uu) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (u < uu) {
                G.v[u] = ld_stream(x4 + ((c0 + u) << 5) + lane);
                if (!PHILOX) G.nib[u] = chunk_nibble(mask + ((c0 + u) << 2), lane);
            }
        }
    };
    auto compute = [&](Group& G, int64_t c0, int uu) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (u < uu) {
                if (PHILOX) {
                    const uint64_t e0 = ((uint64_t)(c0 + u) << 7) + (uint64_t)lane * 4;
                    U4 r = philox_quad(seed, (offset + e0) >> 2);
                    G.nib[u] = nibble4((uint64_t)r.x >= thresh, (uint64_t)r.y >= thresh,
                                       (uint64_t)r.z >= thresh, (uint64_t)r.w >= thresh);
                    store_chunk_mask(mask + ((c0 + u) << 2), G.nib[u], lane);
                }
                float4 o;
                o.x = (G.nib[u] & 1u) ? dscale(G.v[u].x, scale) : 0.0f;
                o.y = (G.nib[u] & 2u) ? dscale(G.v[u].y, scale) : 0.0f;
                o.z = (G.nib[u] & 4u) ? dscale(G.v[u].z, scale) : 0.0f;
                o.w = (G.nib[u] & 8u) ? dscale(G.v[u].w, scale) : 0.0f;
                st_stream(y4 + ((c0 + u) << 5) + lane, o);
            }
        }
    };
    // whole groups, next group's loads in flight during this group's work
    const int64_t ngroups = nchunks / kUnroll;
    Group nxt;
    if (warp < ngroups) load(nxt, warp * kUnroll, kUnroll);
    for (int64_t gi = warp; gi < ngroups; gi += nwarps) {
        Group cur = nxt;
        if (gi + nwarps < ngroups) load(nxt, (gi + nwarps) * kUnroll, kUnroll);
        compute(cur, gi * kUnroll, kUnroll);
    }
    for (int64_t c = ngroups * kUnroll + warp; c < nchunks; c += nwarps) {
        Group one;
        load(one, c, 1);
        compute(one, c, 1);
    }
    if (warp == nwarps - 1)
        dropout_scalar_words<PHILOX>(x, mask, scale, thresh, seed, offset, y, n, nchunks << 2, 1,
                                     lane);
}

// 256-bit variant: lane L owns elements 8L..8L+7 of each 256-element chunk
// (one LDG/STG.256) and byte L of the chunk's mask (read or written
// directly); Philox draws by global element index as above (same bits);
// U chunks per group, ping-pong register buffers.
template <bool PHILOX, int U>
__global__ void __launch_bounds__(kBlock, PHILOX ? TM_DROPOUT_PHILOX_MINB : 1) dropout_fwd8_kernel(
    const float* __restrict__ x, uint32_t* __restrict__ mask, double scale, uint64_t thresh,
    uint64_t seed, uint64_t offset, float* __restrict__ y, int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    if (PHILOX) grid_dep_launch_persistent();  // Philox: one persistent wave
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    uint8_t* mask8 = reinterpret_cast<uint8_t*>(mask);
    const int64_t nchunks = n >> 8;
    const int64_t ngroups = nchunks / U;
    struct Group {
        F8 v[U];
        uint32_t mb[U];
    };
    auto load = [&](Group& G, int64_t c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            G.v[u] = ld_stream8(x + ((c0 + u) << 8) + 8 * lane);
            if (!PHILOX) G.mb[u] = ld_byte(mask8 + ((c0 + u) << 5) + lane);
        }
    };
    auto compute = [&](Group& G, int64_t c0) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e0 = ((c0 + u) << 8) + 8 * lane;
            uint32_t bits;
            if (PHILOX) {
                const uint64_t q = (offset + (uint64_t)e0) >> 2;
                const U4 a = philox_quad(seed, q), b = philox_quad(seed, q + 1);
                bits = ((uint64_t)a.x >= thresh ? 1u : 0u) | ((uint64_t)a.y >= thresh ? 2u : 0u) |
                       ((uint64_t)a.z >= thresh ? 4u : 0u) | ((uint64_t)a.w >= thresh ? 8u : 0u) |
                       ((uint64_t)b.x >= thresh ? 16u : 0u) | ((uint64_t)b.y >= thresh ? 32u : 0u) |
                       ((uint64_t)b.z >= thresh ? 64u : 0u) | ((uint64_t)b.w >= thresh ? 128u : 0u);
                st_stream(mask8 + (e0 >> 3), bits);
            } else {
                bits = G.mb[u];
            }
            F8 o;
#pragma unroll
            for (int j = 0; j < 8; ++j) o.v[j] = ((bits >> j) & 1u) ? dscale(G.v[u].v[j], scale) : 0.0f;
            st_stream8(y + e0, o);
        }
    };
    Group a, b;
    if (warp < ngroups) load(a, warp * U);
    for (int64_t gi = warp; gi < ngroups; gi += 2 * nwarps) {
        const int64_t g1 = gi + nwarps, g2 = gi + 2 * nwarps;
        if (g1 < ngroups) load(b, g1 * U);
        compute(a, gi * U);
        if (g1 >= ngroups) break;
        if (g2 < ngroups) load(a, g2 * U);
        compute(b, g1 * U);
    }
    // leftover chunks (< U per warp), then the ragged tail on the last warp
    for (int64_t c = ngroups * U + warp; c < nchunks; c += nwarps) {
        const F8 v = ld_stream8(x + (c << 8) + 8 * lane);
        const int64_t e0 = (c << 8) + 8 * lane;
        uint32_t bits;
        if (PHILOX) {
            const uint64_t q = (offset + (uint64_t)e0) >> 2;
            const U4 ra = philox_quad(seed, q), rb = philox_quad(seed, q + 1);
            bits = ((uint64_t)ra.x >= thresh ? 1u : 0u) | ((uint64_t)ra.y >= thresh ? 2u : 0u) |
                   ((uint64_t)ra.z >= thresh ? 4u : 0u) | ((uint64_t)ra.w >= thresh ? 8u : 0u) |
                   ((uint64_t)rb.x >= thresh ? 16u : 0u) | ((uint64_t)rb.y >= thresh ? 32u : 0u) |
                   ((uint64_t)rb.z >= thresh ? 64u : 0u) | ((uint64_t)rb.w >= thresh ? 128u : 0u);
            st_stream(mask8 + (e0 >> 3), bits);
        } else {
            bits = ld_byte(mask8 + (e0 >> 3));
        }
        F8 o;
#pragma unroll
        for (int j = 0; j < 8; ++j) o.v[j] = ((bits >> j) & 1u) ? dscale(v.v[j], scale) : 0.0f;
        st_stream8(y + e0, o);
    }
    if (warp == nwarps - 1)
        dropout_scalar_words<PHILOX>(x, mask, scale, thresh, seed, offset, y, n, nchunks << 3, 1,
                                     lane);
}

template <bool PHILOX>
__global__ void __launch_bounds__(kBlock) dropout_fwd_scalar_kernel(
    const float* __restrict__ x, uint32_t* __restrict__ mask, double scale, uint64_t thresh,
    uint64_t seed, uint64_t offset, float* __restrict__ y, int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    dropout_scalar_words<PHILOX>(x, mask, scale, thresh, seed, offset, y, n, warp, nwarps, lane);
}

// Byte mask -> bits; a byte > 1 is a ParamError (BoolMask::from_bytes).
__global__ void __launch_bounds__(kBlock) mask_pack_kernel(const uint8_t* __restrict__ bytes,
                                                           uint32_t* __restrict__ bits, int64_t n,
                                                           int32_t* __restrict__ status) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = warp; w < nwords; w += nwarps) {
        const int64_t i = (w << 5) + lane;
        uint8_t b = i < n ? bytes[i] : 0;
        if (b > 1 && status) *status = TEMPO_ERR_PARAM;
        uint32_t word = __ballot_sync(kFull, b != 0);
        if (lane == 0) bits[w] = word;
    }
}

__global__ void __launch_bounds__(kBlock) mask_unpack_kernel(const uint32_t* __restrict__ bits,
                                                             uint8_t* __restrict__ bytes,
                                                             int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride)
        bytes[i] = (bits[i >> 5] >> (i & 31)) & 1u;
}

// out = float(double(a) * c) -- tempo::scale (kernels.cpp:209-213).
__global__ void __launch_bounds__(kBlock) scale_kernel(const float* __restrict__ a, double c,
                                                       float* __restrict__ out, int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride)
        out[i] = dscale(a[i], c);
}

__global__ void __launch_bounds__(kBlock) add_kernel(const float* __restrict__ a,
                                                     const float* __restrict__ b,
                                                     float* __restrict__ out, int64_t n) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    const int64_t stride = (int64_t)gridDim.x * kBlock;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride)
        out[i] = a[i] + b[i];
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }

template <bool PHILOX>
cudaError_t fwd(const float* x, double scale, uint64_t thresh, uint32_t* mask, uint64_t seed,
                uint64_t offset, float* y, int64_t n, cudaStream_t st) {
    if (TM_DROPOUT_V8 && aligned32(x) && aligned32(y) && aligned16(mask) && (offset & 7u) == 0) {
        constexpr int U = PHILOX ? TM_DROPOUT_PHILOX_U8 : TM_DROPOUT_U8;
        auto k = dropout_fwd8_kernel<PHILOX, U>;
        const int64_t warps = ((n >> 8) + U - 1) / U + 1;
        // supplied masks: several waves of CTAs balance better; Philox (more
        // work per element) keeps one persistent wave
        int grid = grid_for((const void*)k, kBlock, 0, (warps * 32 + kBlock - 1) / kBlock, 0,
                            PHILOX ? TM_DROPOUT_PHILOX_WAVES : TM_DROPOUT_WAVES);
        launch(k, grid, kBlock, 0, st)(x, mask, scale, thresh, seed, offset, y, n);
        return cudaGetLastError();
    }
    const bool vec = aligned16(x) && aligned16(y) && aligned16(mask) && (offset & 3u) == 0;
    if (vec) {
        auto k = dropout_fwd_vec_kernel<PHILOX>;
        const int64_t warps = ((n >> 7) + kUnroll - 1) / kUnroll + 1;
        int grid = grid_for((const void*)k, kBlock, 0, (warps * 32 + kBlock - 1) / kBlock);
        launch(k, grid, kBlock, 0, st)(x, mask, scale, thresh, seed, offset, y, n);
    } else {
        auto k = dropout_fwd_scalar_kernel<PHILOX>;
        const int64_t warps = (n + 31) >> 5;
        int grid = grid_for((const void*)k, kBlock, 0, (warps * 32 + kBlock - 1) / kBlock);
        launch(k, grid, kBlock, 0, st)(x, mask, scale, thresh, seed, offset, y, n);
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dropout_fwd(const float* x, double scale, uint64_t thresh, int philox,
                               uint32_t* mask, uint64_t seed, uint64_t offset, float* y, int64_t n,
                               cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    return philox ? fwd<true>(x, scale, thresh, mask, seed, offset, y, n, st)
                  : fwd<false>(x, scale, thresh, mask, seed, offset, y, n, st);
}

cudaError_t launch_dropout_bwd(const float* dy, const uint32_t* mask, double scale, float* dx,
                               int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    // dropout_backward is mask_scale on the gradient: the SUPPLIED forward.
    return fwd<false>(dy, scale, 0, const_cast<uint32_t*>(mask), 0, 0, dx, n, st);
}

cudaError_t launch_mask_pack(const uint8_t* bytes, uint32_t* bits, int64_t n, int32_t* status,
                             cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const int64_t warps = (n + 31) >> 5;
    int grid = grid_for((const void*)mask_pack_kernel, kBlock, 0, (warps * 32 + kBlock - 1) / kBlock);
    launch(mask_pack_kernel, grid, kBlock, 0, st)(bytes, bits, n, status);
    return cudaGetLastError();
}

cudaError_t launch_scale(const float* a, double c, float* out, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int grid = grid_for((const void*)scale_kernel, kBlock, 0, (n + kBlock - 1) / kBlock);
    launch(scale_kernel, grid, kBlock, 0, st)(a, c, out, n);
    return cudaGetLastError();
}

cudaError_t launch_add(const float* a, const float* b, float* out, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int grid = grid_for((const void*)add_kernel, kBlock, 0, (n + kBlock - 1) / kBlock);
    launch(add_kernel, grid, kBlock, 0, st)(a, b, out, n);
    return cudaGetLastError();
}

cudaError_t launch_mask_unpack(const uint32_t* bits, uint8_t* bytes, int64_t n, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    int grid = grid_for((const void*)mask_unpack_kernel, kBlock, 0, (n + kBlock - 1) / kBlock);
    launch(mask_unpack_kernel, grid, kBlock, 0, st)(bits, bytes, n);
    return cudaGetLastError();
}

}  // namespace tb
