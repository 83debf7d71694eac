// tmem_a_probe.cu -- checks tcgen05.mma kind::tf32 with the A operand in TMEM
// (written by tcgen05.st, lane = row m, one 32-bit column per K element) and B
// K-major SWIZZLE_128B in shared memory, on one 128 x 64 x 32 tile with
// small-integer data (exact in TF32).  Then times back-to-back MMAs
// (M=128, N=64, K=8) with A from TMEM vs A from shared memory.  Prints max |err|
// and cycles per MMA.
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
__device__ __forceinline__ uint32_t k_off(int mn, int k) {
    int chunk = (k >> 2) & 7, row = mn & 7;
    return (uint32_t)((mn >> 3) * 1024 + row * 128 + ((chunk ^ row) << 4) + (k & 3) * 4);
}

__global__ void probe(const float* A, const float* B, float* D, int reps, long long* cyc, int mode) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    unsigned char* sa = base;            // 16 KB (A K-major, smem mode timing)
    unsigned char* sb = base + 16384;    // 8 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < 128 * 32; i += blockDim.x) {
        int m = i / 32, k = i % 32;
        *(float*)(sa + k_off(m, k)) = A[m * 32 + k];
    }
    for (int i = t; i < 32 * 64; i += blockDim.x) {
        int k = i / 64, n = i % 64;
        *(float*)(sb + k_off(n, k)) = B[k * 64 + n];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase, ta = tbase + 64;
    if (warp < 4) {  // row m = warp*32+lane -> TMEM lane m, columns 64 + k
        const int m = warp * 32 + lane;
        for (int c0 = 0; c0 < 32; c0 += 16) {
            uint32_t r[16];
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(A[m * 32 + c0 + i]);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                ::"r"(ta + ((uint32_t)(warp * 32) << 16) + c0),
                  "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                  "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    long long t0 = 0, t1 = 0;
    if (t == 0) {
        t0 = clock64();
        for (int rep = 0; rep < reps; ++rep) {
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t db = desc(su32(sb) + kk * 32, 16, 1024);
                const uint32_t acc = (rep > 0 || kk > 0);
                if (mode == 0) {
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "r"(ta + kk * 8), "l"(db), "r"(idesc), "r"(acc));
                } else {
                    const uint64_t da = desc(su32(sa) + kk * 32, 16, 1024);
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
    if (t == 0) { t1 = clock64(); cyc[blockIdx.x] = t1 - t0; }
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp < 4 && blockIdx.x == 0) {
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
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm) : "memory");
}

// issue rate: back-to-back M=128 x N x K=8 tf32 MMAs into one accumulator,
// A from TMEM (TA) or from a K-major SW128 smem tile, contents irrelevant
template <int N, bool TA>
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
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase, ta = tbase + 256;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    if (t == 0) {
        const uint32_t a = su32(base), b = su32(base + 16384);
        long long c0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t db = desc(b + kk * 32, 16, 1024);
                const uint32_t acc = (it | kk) != 0;
                if (TA)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "r"(ta + kk * 8), "l"(db), "r"(idesc), "r"(acc));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
                                 ::"r"(tm), "l"(desc(a + kk * 32, 16, 1024)), "l"(db), "r"(idesc), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
        asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
        cyc[blockIdx.x] = clock64() - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

// the dV / ctx GEMM's per-slice issue pattern: 4 K-steps x 2 M-blocks x 3
// products (lo.hi, hi.lo, hi.hi), A from TMEM, two B tiles (hi, lo) in
// SWIZZLE_128B smem, accumulators rotating over 2 sets; one commit per slice
__global__ void pattern(long long* cyc, int slices, int commit_each) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* base = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 32768 / 4; i += blockDim.x) ((float*)base)[i] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tm = tbase;
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    if (t == 0) {
        const uint32_t bhi = su32(base), blo = su32(base + 8192);
        long long c0 = clock64();
        int phase = 0;
        for (int sl = 0; sl < slices; ++sl) {
            const uint32_t a0 = tm + (sl & 1) * 128;  // A stage
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t bh = desc(bhi + kk * 32, 16, 1024), bl = desc(blo + kk * 32, 16, 1024);
                const int set = (sl * 4 + kk) & 1;
                const uint32_t fresh = (sl == 0 && kk < 2);
                if (!(commit_each & 2)) {  // the GEMM's order: 3 products per accumulator in a row
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb) {
                        const uint32_t ah = a0 + mb * 64 + kk * 8;
                        const uint32_t acc = tm + 256 + set * 128 + mb * 64;
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                     ::"r"(acc), "r"(ah + 32), "l"(bh), "r"(idesc), "r"(1u - fresh));
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                     ::"r"(acc), "r"(ah), "l"(bl), "r"(idesc), "r"(1u));
                        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                     ::"r"(acc), "r"(ah), "l"(bh), "r"(idesc), "r"(1u));
                    }
                } else {  // interleaved over the two M-blocks
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
#pragma unroll
                        for (int mb = 0; mb < 2; ++mb) {
                            const uint32_t ah = a0 + mb * 64 + kk * 8;
                            const uint32_t acc = tm + 256 + set * 128 + mb * 64;
                            const uint32_t aa = q == 0 ? ah + 32 : ah;
                            const uint64_t bb = q == 1 ? bl : bh;
                            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n"
                                         ::"r"(acc), "r"(aa), "l"(bb), "r"(idesc), "r"(q == 0 ? 1u - fresh : 1u));
                        }
                    }
                }
            }
            if (commit_each & 1) {  // commit + wait per slice: the round trip the GEMM pays
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
                asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)), "r"(phase) : "memory");
                phase ^= 1;
            }
        }
        if (!(commit_each & 1)) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
            asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar)) : "memory");
        }
        cyc[blockIdx.x] = clock64() - c0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

template <int N, bool TA>
void run_rate(long long* dc, int ctas) {
    auto k = rate<N, TA>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    const int iters = 2000;
    k<<<ctas, 128, 70000>>>(dc, iters);
    cudaDeviceSynchronize();
    k<<<ctas, 128, 70000>>>(dc, iters);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<long long> c(ctas);
    cudaMemcpy(c.data(), dc, ctas * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (auto v : c) mx = v > mx ? v : mx;
    const double per = (double)mx / (iters * 4);
    printf("rate tf32 M=128 N=%d A=%s ctas=%d: %.1f cycles/MMA, %.0f FLOP/cycle/SM (%s)\n", N,
           TA ? "tmem" : "smem", ctas, per, 2.0 * 128 * N * 8 / per, cudaGetErrorString(e));
}

int main() {
    std::vector<float> A(128 * 32), B(32 * 64), R(128 * 64);
    for (int m = 0; m < 128; ++m) for (int k = 0; k < 32; ++k) A[m * 32 + k] = (float)((m * 3 + k * 7) % 11 - 5);
    for (int k = 0; k < 32; ++k) for (int n = 0; n < 64; ++n) B[k * 64 + n] = (float)((k * 5 + n * 3) % 9 - 4);
    for (int m = 0; m < 128; ++m) for (int n = 0; n < 64; ++n) {
        double s = 0; for (int k = 0; k < 32; ++k) s += (double)A[m * 32 + k] * B[k * 64 + n];
        R[m * 64 + n] = (float)s;
    }
    float *dA, *dB, *dD; long long* dc;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, R.size() * 4);
    cudaMalloc(&dc, 148 * 8);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(dD, 0, R.size() * 4);
        probe<<<1, 256, 32768>>>(dA, dB, dD, 1, dc, mode);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> G(R.size());
        cudaMemcpy(G.data(), dD, G.size() * 4, cudaMemcpyDeviceToHost);
        double mx = 0; int nz = 0;
        for (size_t i = 0; i < G.size(); ++i) { double d = G[i] - R[i]; if (d < 0) d = -d; if (d > mx) mx = d; nz += G[i] != 0; }
        printf("A from %s: err=%s max|err|=%g nonzero=%d D[0][0..3]=%g %g %g %g ref=%g %g %g %g\n",
               mode ? "smem" : "TMEM", cudaGetErrorString(e), mx, nz, G[0], G[1], G[2], G[3], R[0], R[1], R[2], R[3]);
        const int reps = 4096;
        probe<<<148, 256, 32768>>>(dA, dB, dD, reps, dc, mode);
        e = cudaDeviceSynchronize();
        std::vector<long long> c(148);
        cudaMemcpy(c.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mxc = 0; for (auto v : c) mxc = v > mxc ? v : mxc;
        printf("  rate (148 CTAs, %d MMAs of 128x64x8 each): %s, %.2f cycles/MMA\n", reps * 4,
               cudaGetErrorString(e), (double)mxc / (reps * 4));
    }
    for (int ctas : {1, 148}) {
        run_rate<64, true>(dc, ctas); run_rate<64, false>(dc, ctas);
        run_rate<128, true>(dc, ctas); run_rate<128, false>(dc, ctas);
        run_rate<256, true>(dc, ctas); run_rate<256, false>(dc, ctas);
    }
    cudaFuncSetAttribute(pattern, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    for (int ce = 0; ce < 4; ++ce) {
        const int slices = 512;
        pattern<<<148, 128, 40000>>>(dc, slices, ce);
        cudaDeviceSynchronize();
        pattern<<<148, 128, 40000>>>(dc, slices, ce);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<long long> c(148);
        cudaMemcpy(c.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
        long long mx = 0; for (auto v : c) mx = v > mx ? v : mx;
        printf("GEMM slice pattern (24 MMAs N=64, A tmem, 2 sets)%s%s: %.1f cycles/slice, %.1f cycles/MMA (%s)\n",
               (ce & 2) ? ", M-blocks interleaved" : "", (ce & 1) ? " + commit/wait per slice" : "", (double)mx / slices, (double)mx / (slices * 24), cudaGetErrorString(e));
    }
    return 0;
}
