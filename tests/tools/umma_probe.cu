// umma_probe.cu -- checks the tcgen05 kind::tf32 operand layouts used by
// dv_gemm_kernels.cu on one 128 x 64 x 32 tile with small-integer data
// (exact in TF32): variant bit 0: A MN-major, bit 1: B MN-major, bit 2: LBO/SBO swapped
// for the MN-major operands (else K-major SWIZZLE_128B).  Prints max |err|.
#include <cstdio>
#include <cstdint>
#include <vector>
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
__device__ __forceinline__ uint32_t mn_off(int mn, int k, int groups) {
    int chunk = (mn >> 2) & 7, row = k & 7;
    return (uint32_t)(((k >> 3) * groups + (mn >> 5)) * 1024 + row * 128 + ((chunk ^ row) << 4) + (mn & 3) * 4);
}
// K-major SW128: row mn has 32 K-elements (128 B); 8 rows per 1 KB atom; atoms along MN
__device__ __forceinline__ uint32_t k_off(int mn, int k) {
    int chunk = (k >> 2) & 7, row = mn & 7;
    return (uint32_t)((mn >> 3) * 1024 + row * 128 + ((chunk ^ row) << 4) + (k & 3) * 4);
}

__global__ void probe(const float* A, const float* B, float* D, int variant) {
    // A [128][32] (m,k), B [32][64] (k,n), D [128][64]
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char* sa = base;            // 16 KB
    unsigned char* sb = base + 16384;    // 8 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < 128 * 32; i += blockDim.x) {
        int m = i / 32, k = i % 32;
        uint32_t o = (variant & 1) ? mn_off(m, k, 4) : k_off(m, k);
        *(float*)(sa + o) = A[m * 32 + k];
    }
    for (int i = t; i < 32 * 64; i += blockDim.x) {
        int k = i / 64, n = i % 64;
        uint32_t o = (variant & 2) ? mn_off(n, k, 2) : k_off(n, k);
        *(float*)(sb + o) = B[k * 64 + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t tm = tbase;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(variant & 1) << 15) |
                     ((uint32_t)((variant >> 1) & 1) << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    const bool sw = variant & 4;
    if (t == 0) {
        for (int kk = 0; kk < 4; ++kk) {
            uint64_t da, db;
            if (variant & 1) da = sw ? desc(su32(sa) + kk * 4 * 1024, 4 * 1024, 1024)
                                     : desc(su32(sa) + kk * 4 * 1024, 1024, 4 * 1024);
            else da = desc(su32(sa) + kk * 32, 16, 1024);
            if (variant & 2) db = sw ? desc(su32(sb) + kk * 2 * 1024, 2 * 1024, 1024)
                                     : desc(su32(sb) + kk * 2 * 1024, 1024, 2 * 1024);
            else db = desc(su32(sb) + kk * 32, 16, 1024);
            uint32_t acc = kk > 0;
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                         ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    __syncwarp();
    // wait
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4) {
        for (int c0 = 0; c0 < 64; c0 += 16) {
            uint32_t r[16];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(tm + ((uint32_t)(warp * 32) << 16) + c0));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            for (int i = 0; i < 16; ++i) D[(warp * 32 + lane) * 64 + c0 + i] = __uint_as_float(r[i]);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tm) : "memory");
}

int main() {
    std::vector<float> A(128 * 32), B(32 * 64), R(128 * 64);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) A[m * 32 + k] = (float)((m * 3 + k * 7) % 11 - 5);
    for (int k = 0; k < 32; ++k) for (int n = 0; n < 64; ++n) B[k * 64 + n] = (float)((k * 5 + n * 3) % 9 - 4);
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n) {
        double s = 0; for (int k = 0; k < 32; ++k) s += (double)A[m * 32 + k] * B[k * 64 + n];
        R[m * 64 + n] = (float)s;
    }
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, R.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int v = 0; v < 8; ++v) {
        if (v == 4) continue;
        cudaMemset(dD, 0, R.size() * 4);
        probe<<<1, 256, 32768>>>(dA, dB, dD, v);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> G(R.size());
        cudaMemcpy(G.data(), dD, G.size() * 4, cudaMemcpyDeviceToHost);
        double mx = 0; int nz = 0;
        for (size_t i = 0; i < G.size(); ++i) { double d = G[i] - R[i]; if (d < 0) d = -d; if (d > mx) mx = d; nz += G[i] != 0; }
        printf("variant %d (A %s, B %s, %s): err=%s max|err|=%g nonzero=%d  D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", v,
               (v & 1) ? "MN" : "K", (v & 2) ? "MN" : "K", (v & 4) ? "lbo<->sbo" : "lbo=mn-step",
               cudaGetErrorString(e), mx, nz, G[0], G[1], G[2], G[3], R[0], R[1], R[2], R[3]);
    }
    return 0;
}
