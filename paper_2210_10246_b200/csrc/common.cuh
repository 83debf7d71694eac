// common.cuh -- device helpers shared by the Tempo in-place operator kernels.
//
// All kernels here are HBM-streaming kernels: 128-bit
// coalesced loads/stores, read-once data loaded with L1::no_allocate and
// written with the streaming (.cs) hint, grids sized as a multiple of the SM
// count x resident CTAs per SM (grid-stride persistent loops).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tb {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;

// ---- streaming global memory access -------------------------------------
__device__ __forceinline__ float4 ld_stream(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// 256-bit accesses (sm_100: LDG/STG .256): eight consecutive floats per lane,
// so a lane owns a whole byte of a bit-packed mask.
struct F8 {
    float v[8];
};
__device__ __forceinline__ F8 ld_stream8(const float* p) {
    F8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]),
                   "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream8(float* p, const F8& r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
                 "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]),
                 "f"(r.v[7])
                 : "memory");
}
__device__ __forceinline__ void st_stream(uint8_t* p, uint32_t v) {
    asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_byte(const uint8_t* p) {
    uint16_t v;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
}
// (acc << 1) | sign(v): one funnel shift collects a sign bit.
__device__ __forceinline__ uint32_t push_sign(uint32_t acc, float v) {
    return __funnelshift_l(__float_as_uint(v), acc, 1);
}

// Plain cached load (data read by several lanes / re-read from L2).
__device__ __forceinline__ uint32_t ld_cached(const uint32_t* p) { return __ldg(p); }

__device__ __forceinline__ void st_stream(float4* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};"
                 :
                 : "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}
__device__ __forceinline__ void st_stream(float* p, float v) {
    asm volatile("st.global.cs.f32 [%0], %1;" : : "l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void st_stream(uint32_t* p, uint32_t v) {
    asm volatile("st.global.cs.u32 [%0], %1;" : : "l"(p), "r"(v) : "memory");
}

// ---- bit-packed masks ----------------------------------------------------
// Chunk = 128 consecutive elements handled by one warp, lane L owning
// elements 4L..4L+3 (one float4).  The chunk's mask is 4 words; word w holds
// lanes 8w..8w+7, bit (4j + k) = element 4(8w+j) + k: the linear BoolMask
// order (tensor.cpp:199-201).
//
// pack: lane L contributes the nibble of its 4 elements; three xor-shuffles
// OR the 8 nibbles of each 8-lane group into that group's word, which lane
// 8w stores (the 4 words of a chunk are contiguous: one 16-byte sector).
__device__ __forceinline__ uint32_t nibble4(bool k0, bool k1, bool k2, bool k3) {
    return (uint32_t)k0 | ((uint32_t)k1 << 1) | ((uint32_t)k2 << 2) | ((uint32_t)k3 << 3);
}
__device__ __forceinline__ void store_chunk_mask(uint32_t* chunk_words, uint32_t nib, int lane) {
    uint32_t v = nib << ((lane & 7) << 2);
    v |= __shfl_xor_sync(kFull, v, 1);
    v |= __shfl_xor_sync(kFull, v, 2);
    v |= __shfl_xor_sync(kFull, v, 4);
    if ((lane & 7) == 0) st_stream(chunk_words + (lane >> 3), v);
}
// unpack: the 4 bits of lane L's float4 from the chunk's word (L >> 3).
__device__ __forceinline__ uint32_t chunk_nibble(const uint32_t* chunk_words, int lane) {
    uint32_t w = ld_cached(chunk_words + (lane >> 3));
    return (w >> (4 * (lane & 7))) & 0xfu;
}

// ---- Philox4x32-10 (Salmon et al., SC'11) --------------------------------
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += W0;
        k1 += W1;
    }
    return c;
}
// Four uniform draws for elements 4q..4q+3 of a tensor whose element 0 has
// global index `offset` (offset % 4 == 0 required for the vector paths; the
// scalar path draws per element with the same counter mapping).
__device__ __forceinline__ U4 philox_quad(uint64_t seed, uint64_t quad_index) {
    U4 c{(uint32_t)quad_index, (uint32_t)(quad_index >> 32), 0x7e3a1b5du, 0x0u};
    return philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
}
__device__ __forceinline__ uint32_t philox_at(uint64_t seed, uint64_t global_index) {
    U4 r = philox_quad(seed, global_index >> 2);
    switch (global_index & 3) {
        case 0: return r.x;
        case 1: return r.y;
        case 2: return r.z;
        default: return r.w;
    }
}

// ---- TMA bulk copies + mbarriers (cp.async.bulk, sm_90+/sm_100a) ---------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Arrive (count 1) and add `bytes` to the barrier's expected transaction count.
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// Plain arrive (count 1, release at CTA scope).
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "TB_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra TB_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// Order this thread's generic-proxy smem accesses before later async-proxy
// (TMA) writes to the same smem (stage reuse).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global -> shared bulk copy (16-byte aligned, size % 16 == 0), completing
// `bytes` transactions on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Named barrier over `nthreads` threads (a multiple of 32) of the CTA: the
// warps of one row group synchronise without stalling the CTA's other groups.
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---- programmatic dependent launch (PDL) --------------------------------
// A kernel launched with the programmatic-stream-serialization attribute may
// start while its predecessor drains; it must call grid_dep_wait() before
// touching the predecessor's outputs (waits for its completion + memory
// flush).  grid_dep_launch() lets the dependent grid launch early.
__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
#ifndef TM_PDL_TRIGGER
#define TM_PDL_TRIGGER 0  // 1: early trigger (measured -7 %: dependents steal slots from multi-wave grids)
#endif
__device__ __forceinline__ void grid_dep_launch() {
#if TM_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// Early trigger for single-wave persistent grids: all their CTAs are already
// resident, so the dependent's CTAs can only take leftover slots (no slot
// stealing) and start the moment this grid's memory is flushed.
#ifndef TM_PDL_TRIGGER_PERSISTENT
#define TM_PDL_TRIGGER_PERSISTENT 1
#endif
__device__ __forceinline__ void grid_dep_launch_persistent() {
#if TM_PDL_TRIGGER_PERSISTENT
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// ---- warp reductions -----------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ float warp_sumf(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(kFull, v, o));
    return v;
}

}  // namespace tb
