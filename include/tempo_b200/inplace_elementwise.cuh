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

// Lane L owns elements 8L..8L+7 of a 256-element chunk: one 256-bit load or
// store per tensor and a whole byte of the bit-packed mask (byte L of the
// chunk's 32 bytes = BoolMask order), written or read directly.
struct F8 {
    float v[8];
};
__device__ __forceinline__ F8 ld8(const float* p) {
    F8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float* p, const F8& r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
                 "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]),
                 "f"(r.v[7])
                 : "memory");
}

// vec = 0 (pointers not 32-byte aligned): everything through the scalar
// loops (same per-element functions, so the same bits).
template <class Spec>
__global__ void __launch_bounds__(kBlock) fwd_kernel(const float* __restrict__ x,
                                                     float* __restrict__ y,
                                                     uint32_t* __restrict__ mask, int64_t n,
                                                     int vec) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = vec ? (n >> 8) : 0;
    uint8_t* mask8 = reinterpret_cast<uint8_t*>(mask);
    F8 nxt;
    if (warp < nchunks) nxt = ld8(x + (warp << 8) + 8 * lane);
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const F8 v = nxt;
        if (c + nwarps < nchunks) nxt = ld8(x + ((c + nwarps) << 8) + 8 * lane);
        F8 o;
        uint32_t b = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            o.v[k] = Spec::fwd(v.v[k]);
            b |= (uint32_t)Spec::branch(v.v[k]) << k;
        }
        st8(y + (c << 8) + 8 * lane, o);
        mask8[(c << 5) + lane] = (uint8_t)b;
    }
    // the rest (ragged tail, or everything when unaligned): one ballot per word
    const int64_t nwords = (n + 31) >> 5;
    for (int64_t w = (nchunks << 3) + warp; w < nwords; w += nwarps) {
        const int64_t i = (w << 5) + lane;
        const bool in = i < n;
        const float xv = in ? x[i] : 0.0f;
        const uint32_t bits = __ballot_sync(kFull, in && Spec::branch(xv));
        if (in) y[i] = Spec::fwd(xv);
        if (lane == 0) mask[w] = bits;
    }
}

template <class Spec>
__global__ void __launch_bounds__(kBlock) bwd_kernel(const float* __restrict__ dy,
                                                     const float* __restrict__ y,
                                                     const uint32_t* __restrict__ mask,
                                                     float* __restrict__ dx, int64_t n, int vec) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nchunks = vec ? (n >> 8) : 0;
    const uint8_t* mask8 = reinterpret_cast<const uint8_t*>(mask);
    for (int64_t c = warp; c < nchunks; c += nwarps) {
        const F8 g = ld8(dy + (c << 8) + 8 * lane), v = ld8(y + (c << 8) + 8 * lane);
        const uint32_t b = __ldg(mask8 + (c << 5) + lane);
        F8 o;
#pragma unroll
        for (int k = 0; k < 8; ++k) o.v[k] = g.v[k] * Spec::grad_from_output(v.v[k], (b >> k) & 1u);
        st8(dx + (c << 8) + 8 * lane, o);
    }
    for (int64_t i = (nchunks << 8) + warp * 32 + lane; i < n; i += nwarps * 32)
        dx[i] = dy[i] * Spec::grad_from_output(y[i], (mask[i >> 5] >> (i & 31)) & 1u);
}

inline int grid_of(const void* k, int64_t n) {
    int dev = 0, sms = 1, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kBlock, 0);
    const int64_t need = (((n >> 5) + 1) * 32 + kBlock - 1) / kBlock;
    const int64_t full = (int64_t)sms * (per > 0 ? per : 1);
    return (int)(need < full ? (need > 0 ? need : 1) : full);
}

inline bool aligned32(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
}  // namespace detail

// y = Spec::fwd(x), mask bit = Spec::branch(x).  Any alignment (32-byte
// aligned x and y take the 256-bit path).
template <class Spec>
cudaError_t forward(const float* x, float* y, uint32_t* mask, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int vec = detail::aligned32(x) && detail::aligned32(y) ? 1 : 0;
    auto k = detail::fwd_kernel<Spec>;
    k<<<detail::grid_of((const void*)k, n), detail::kBlock, 0, st>>>(x, y, mask, n, vec);
    return cudaGetLastError();
}

// dx = dy * Spec::grad_from_output(y, mask bit).  dx may alias dy.
template <class Spec>
cudaError_t backward(const float* dy, const float* y, const uint32_t* mask, float* dx, int64_t n,
                     cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int vec = detail::aligned32(dy) && detail::aligned32(y) && detail::aligned32(dx) ? 1 : 0;
    auto k = detail::bwd_kernel<Spec>;
    k<<<detail::grid_of((const void*)k, n), detail::kBlock, 0, st>>>(dy, y, mask, dx, n, vec);
    return cudaGetLastError();
}

}  // namespace ew

#ifdef TEMPO_B200_HAS_GRAPH_API
namespace tempo_ops {
// tempo_ops::inplace_elementwise (ops_tempo.cpp:32-71) with a device spec:
// stashes its output (shared with downstream) and the bit mask, not x.
template <class Spec>
NodeId inplace_elementwise(Graph& g, NodeId x, std::string tag, std::string mask_tag) {
    // allocate y / the mask on the graph's stream, where the kernel runs
    // (as every builder in tempo_host.cpp does)
    tempo_b200::StreamScope scope_(g.stream);
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
