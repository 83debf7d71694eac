// umma_rate.cu -- tcgen05.mma issue rate probe (cycles per instruction) for
// kind::tf32 / kind::f16, M = 128, N in {64, 128, 256}, K-major SW128
// operands resident in smem (contents irrelevant), one accumulator.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((a >> 4) & 0x3fff);
    d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

template <int N, bool TF32>
__global__ void rate(long long* cyc, int iters) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 65536 / 4; i += blockDim.x) ((float*)base)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tm = tbase;
    // f16 kind: a/b format 0 (F16), K = 16 per MMA (32 bytes); tf32: K = 8 (32 bytes)
    uint32_t idesc = (1u << 4) | ((TF32 ? 2u : 0u) << 7) | ((TF32 ? 2u : 0u) << 10) |
                     ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    if (t == 0) {
        uint32_t a = su32(base), b = su32(base + 16384);
        long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                uint64_t da = desc(a + kk * 32, 16, 1024), db = desc(b + kk * 32, 16, 1024);
                uint32_t acc = (it | kk) != 0;
                if (TF32)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
        long long c1 = clock64();
        *cyc = c1 - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm) : "memory");
}

template <int N, bool TF32>
void run() {
    long long* d;
    cudaMalloc(&d, 8);
    auto k = rate<N, TF32>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    int iters = 2000;
    k<<<1, 128, 70000>>>(d, iters);
    cudaDeviceSynchronize();
    k<<<1, 128, 70000>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    double per = (double)c / (iters * 4);
    double flop = 2.0 * 128 * N * (TF32 ? 8 : 16);
    printf("%s M=128 N=%d: %.1f cycles/MMA, %.0f FLOP/cycle/SM (%s)\n", TF32 ? "tf32" : "f16 ", N, per,
           flop / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<64, true>();
    run<128, true>();
    run<256, true>();
    run<64, false>();
    run<256, false>();
    return 0;
}
