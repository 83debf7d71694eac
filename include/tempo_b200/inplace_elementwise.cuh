// tempo_b200/inplace_elementwise.cuh -- the reference's generic in-place
// elementwise scheme (tempo_ops::inplace_elementwise, ops_tempo.hpp:21-35,
// ops_tempo.cpp:32-71; PAPER.md "differentiate from output + branch mask")
// as COMPILE-TIME functor kernels for sm_100a.
//
// The reference takes three std::function callbacks per element (fwd,
// branch, grad_from_output).  On the GPU the spec is a struct of __device__
// functions, instantiated into the same streaming kernels the GELU uses:
// float4 loads, register prefetch, the bit-packed branch mask (one bit per
// element, BoolMask order), and the backward reading only (y, mask):
//
//   struct ExpSpec {                                  // test_ops_tempo.cpp:291-316
//       __device__ static float fwd(float x) { return expf(x); }
//       __device__ static bool branch(float) { return true; }
//       __device__ static float grad_from_output(float y, bool) { return y; }
//   };
//   tempo_b200::ew::forward<ExpSpec>(x, y, mask, n, stream);
//   tempo_b200::ew::backward<ExpSpec>(dy, y, mask, dx, n, stream);
//
// Header-only; include it from a .cu compiled with
// -gencode arch=compute_100a,code=sm_100a.  With tempo.hpp included first,
// tempo_ops::inplace_elementwise<Spec>(Graph&, ...) records the op on the
// device Tape exactly like the reference builder (stash: y + mask).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tempo_b200 {
namespace ew {

namespace detail {
constexpr int kBlock = 256;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t nibble(bool a, bool b, bool c, bool d) {
    return (uint32_t)a | ((uint32_t)b << 1) | ((uint32_t)c << 2) | ((uint32_t)d << 3);
}
// Lane L owns elements 4L..4L+3 of a 128-element chunk; word w of the chunk
// holds lanes 8w..8w+7 (bit 4j+k = element 4(8w+j)+k, BoolMask order).
__device__ __forceinline__ void store_chunk_mask(uint32_t* words, uint32_t nib, int lane) {
    uint32_t v = nib << ((lane & 7) << 2);
    v |= __shfl_xor_sync(kFull, v, 1);
    v |= __shfl_xor_sync(kFull, v, 2);
    v |= __shfl_xor_sync(kFull, v, 4);
    if ((lane & 7) == 0) words[lane >> 3] = v;
}

template <class Spec>
__global__ void __launch_bounds__(kBlock) fwd_kernel(const float* __restrict__ x,
                                                     float* __restrict__ y,
                                                     uint32_t* __restrict__ mask, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 7;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    float4 nxt = make_float4(0.f, 0.f, 0.f, 0.f);
    if (warp < nchunks) nxt = __ldg(x4 + (warp << 5) + lane);
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const float4 v = nxt;
        if (c + nwarps < nchunks) nxt = __ldg(x4 + ((c + nwarps) << 5) + lane);
        y4[(c << 5) + lane] = make_float4(Spec::fwd(v.x), Spec::fwd(v.y), Spec::fwd(v.z),
                                          Spec::fwd(v.w));
        store_chunk_mask(mask + (c << 2),
                         nibble(Spec::branch(v.x), Spec::branch(v.y), Spec::branch(v.z),
                                Spec::branch(v.w)),
                         lane);
    }
    if (warp == nwarps - 1) {  // ragged tail: one ballot per mask word
        const int64_t nwords = (n + 31) >> 5;
        for (int64_t w = nchunks << 2; w < nwords; ++w) {
            const int64_t i = (w << 5) + lane;
            const bool in = i < n;
            const float xv = in ? x[i] : 0.0f;
            const uint32_t bits = __ballot_sync(kFull, in && Spec::branch(xv));
            if (in) y[i] = Spec::fwd(xv);
            if (lane == 0) mask[w] = bits;
        }
    }
}

template <class Spec>
__global__ void __launch_bounds__(kBlock) bwd_kernel(const float* __restrict__ dy,
                                                     const float* __restrict__ y,
                                                     const uint32_t* __restrict__ mask,
                                                     float* __restrict__ dx, int64_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = n >> 7;
    const float4* g4 = reinterpret_cast<const float4*>(dy);
    const float4* y4 = reinterpret_cast<const float4*>(y);
    float4* d4 = reinterpret_cast<float4*>(dx);
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const float4 g = __ldg(g4 + (c << 5) + lane), v = __ldg(y4 + (c << 5) + lane);
        const uint32_t nib = (__ldg(mask + (c << 2) + (lane >> 3)) >> (4 * (lane & 7))) & 0xfu;
        d4[(c << 5) + lane] = make_float4(g.x * Spec::grad_from_output(v.x, nib & 1u),
                                          g.y * Spec::grad_from_output(v.y, (nib >> 1) & 1u),
                                          g.z * Spec::grad_from_output(v.z, (nib >> 2) & 1u),
                                          g.w * Spec::grad_from_output(v.w, (nib >> 3) & 1u));
    }
    if (warp == nwarps - 1) {
        for (int64_t i = (nchunks << 7) + lane; i < n; i += 32)
            dx[i] = dy[i] * Spec::grad_from_output(y[i], (mask[i >> 5] >> (i & 31)) & 1u);
    }
}

inline int grid_of(const void* k, int64_t n) {
    int dev = 0, sms = 1, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kBlock, 0);
    const int64_t need = (((n >> 7) + 1) * 32 + kBlock - 1) / kBlock;
    const int64_t full = (int64_t)sms * (per > 0 ? per : 1);
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace detail

// y = Spec::fwd(x), mask bit = Spec::branch(x).  x, y 16-byte aligned.
template <class Spec>
cudaError_t forward(const float* x, float* y, uint32_t* mask, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (!detail::aligned16(x) || !detail::aligned16(y)) return cudaErrorMisalignedAddress;
    auto k = detail::fwd_kernel<Spec>;
    k<<<detail::grid_of((const void*)k, n), detail::kBlock, 0, st>>>(x, y, mask, n);
    return cudaGetLastError();
}

// dx = dy * Spec::grad_from_output(y, mask bit).
template <class Spec>
cudaError_t backward(const float* dy, const float* y, const uint32_t* mask, float* dx, int64_t n,
                     cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (!detail::aligned16(dy) || !detail::aligned16(y) || !detail::aligned16(dx))
        return cudaErrorMisalignedAddress;
    auto k = detail::bwd_kernel<Spec>;
    k<<<detail::grid_of((const void*)k, n), detail::kBlock, 0, st>>>(dy, y, mask, dx, n);
    return cudaGetLastError();
}

}  // namespace ew

#ifdef TEMPO_B200_HAS_GRAPH_API
namespace tempo_ops {
// tempo_ops::inplace_elementwise (ops_tempo.cpp:32-71) with a device spec:
// stashes its output (shared with downstream) and the bit mask, not x.
template <class Spec>
NodeId inplace_elementwise(Graph& g, NodeId x, std::string tag, std::string mask_tag) {
    const Tensor& vx = g.value(x);
    Tensor y = Tensor::empty(vx.shape());
    BoolMask mask = BoolMask::empty(vx.shape());
    cudaStream_t st = static_cast<cudaStream_t>(g.stream);
    cudaError_t e = ew::forward<Spec>(vx.data(), y.data(), mask.words(), vx.numel(), st);
    if (e != cudaSuccess) throw CudaError(std::string("inplace_elementwise: ") + cudaGetErrorString(e));
    NodeId id = g.tape.record(
        "inplace_ew", tag, {x}, y, {LazyStash::materialized(tag, StashRole::OpOwnStash, y)},
        [mask, st](BackwardCtx& ctx) -> std::vector<Tensor> {
            const Tensor& gy = ctx.grad_out();
            const Tensor& yv = ctx.stash(0);
            Tensor dx = Tensor::empty(yv.shape());
            cudaError_t e2 = ew::backward<Spec>(gy.data(), yv.data(), mask.words(), dx.data(),
                                                yv.numel(), st);
            if (e2 != cudaSuccess)
                throw CudaError(std::string("inplace_elementwise bwd: ") + cudaGetErrorString(e2));
            return {dx};
        });
    g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
    return id;
}
}  // namespace tempo_ops
#endif

}  // namespace tempo_b200
