// dv_gemm_kernels.cu -- the attention-dropout recompute fused into its
// consumer, the dV GEMM, on the 5th-generation tensor cores (sm_100a).
//
// The reference's Sub-Layer Dropout Recomputation keeps only P and the mask;
// when the backward reaches the consumer of the dropped-out map D -- the
// attention-context GEMM ctx = D @ V, whose backward needs D for
// dV = D^T @ dO -- the consumer asks for D and the recompute rule
// "dropout-rescale" rebuilds it (graph.cpp:46-50 -> BackwardCtx::stash,
// tape.cpp:244-264; rule ops_tempo.cpp:17-26 = dropout_apply,
// ops_reference.cpp:147-153).  Here D never exists in HBM: the producer warps
// rebuild each tile of D from P and the mask bits (D = keep ? float(double(P)
// * s) : 0, the same rounding as mask_scale, kernels.cpp:285-295, so the
// tile is bitwise the D the forward produced) directly in shared memory, in
// the UMMA operand layout, and tcgen05.mma consumes it.  HBM traffic per
// attention element: P (4 B) + the mask bit, instead of writing D (4 B) in
// attn_probs_bwd and reading it back (4 B) in a separate GEMM.
//
// GEMM per (batch, head): dV[j, c] = sum_i D[i, j] dO[i, c]
//   M = s_k (j), N = d (c), K = s_q (i).  P / D are row-major [i][j] and dO
//   [i][c], i.e. both operands are MN-major in HBM; tcgen05 kind::tf32 gives
//   no result for MN-major operands on this part (measured,
//   tests/tools/umma_probe.cu: every a_major/b_major = MN variant returns 0,
//   K-major is exact), so the producers transpose while staging: a thread
//   owns one M (or N) index, reads it down 32 K-rows (each warp load is a
//   coalesced 128-byte row segment) and writes 16-byte K-chunks into the
//   canonical K-major SWIZZLE_128B layout (128-byte rows, 8-row 1 KB atoms,
//   chunk index XOR row: conflict-free).
// fp32 accuracy from TF32 tensor cores: 3xTF32 -- x = hi + lo with hi, lo
//   TF32 (round-to-nearest), D^T dO ~ hi*hi + hi*lo + lo*hi, all three
//   products accumulated in one fp32 TMEM accumulator (relative error ~2^-21
//   per product vs fp32's 2^-24; dV within 1e-6 of the fp64 product).
//
// CTA = one (head, 256-row block of dV): 8 producer warps + 1 MMA warp.
//   producers: global P (+mask words) and dO -> registers (the next K-chunk
//     of 32 rows loads while this one is staged) -> D, hi/lo split ->
//     st.shared into stage s of a 2-deep ring -> fence.proxy.async +
//     mbarrier arrive (full[s]);
//   MMA warp (one elected lane): per stage, 4 K-steps x 2 M-blocks x 3
//     tcgen05.mma.kind::tf32 (M=128, N=d, K=8) into two TMEM accumulators,
//     tcgen05.commit -> empty[s] (the stage may be overwritten) and, after
//     the last stage, -> acc_full;
//   epilogue: the producer warps tcgen05.ld their TMEM lane quadrant
//     (warp w: accumulator w/4, lanes 32*(w%4)..) and store dV rows.
#include "common.cuh"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kBM = 256;             // dV rows per CTA (two M=128 accumulators)
constexpr int kBK = 32;              // K rows (query positions) per stage
constexpr int kStagesG = 2;
constexpr int kProducers = 256;      // 8 warps
constexpr int kThreadsG = kProducers + 32;

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ uint32_t sw128_k_offset(int mn, int kchunk) {
    // byte offset of the 16-byte K-chunk `kchunk` (K = 4*kchunk..+3, < 32) of
    // row mn in a K-major SWIZZLE_128B tile: [mn/8][mn%8][128 B], chunk ^ row
    const int row = mn & 7;
    return (uint32_t)((mn >> 3) * 1024 + row * 128 + ((kchunk ^ row) << 4));
}

// UMMA shared-memory descriptor (sm_100): start, LBO, SBO in 16-byte units,
// version 1, SWIZZLE_128B (layout type 2).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3fff);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3fff) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)2 << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, M x N.
__host__ __device__ constexpr uint32_t idesc_tf32_k(int m, int n) {
    return (1u << 4)                      // c_format = F32
           | (2u << 7) | (2u << 10)       // a_format, b_format = TF32
           | ((uint32_t)(n >> 3) << 17)   // N >> 3
           | ((uint32_t)(m >> 4) << 24);  // M >> 4
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <int N>  // head dim d
__global__ void __launch_bounds__(kThreadsG, 1) dv_recompute_gemm_kernel(
    const float* __restrict__ P, const uint32_t* __restrict__ mask, double scale,
    const float* __restrict__ dO, float* __restrict__ dV, int s_q, int s_k) {
    static_assert(N % 32 == 0 && N >= 32 && N <= 128, "head dim");
    constexpr int kAbytes = kBM * kBK * 4;          // one of A_hi / A_lo per stage
    constexpr int kBbytes = N * kBK * 4;            // one of B_hi / B_lo per stage
    constexpr int kStageBytes = 2 * kAbytes + 2 * kBbytes;
    // kSets accumulator sets (K-steps round-robin, summed in the epilogue):
    // the tensor core's fp32 accumulation truncates, so its error grows with
    // the number of MMAs per accumulator (K = 1024 in one set: 1.7e-5)
    constexpr int kSets = 512 / (2 * N) >= 4 ? 4 : 512 / (2 * N);
    constexpr int kTmemCols = kSets * 2 * N;  // 512 for N = 64 / 128, 256 for N = 32
    grid_dep_wait();
    grid_dep_launch();
    extern __shared__ __align__(1024) unsigned char gsm[];
    // 1 KB alignment for the swizzled operand tiles
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(gsm) + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[kStagesG], empty[kStagesG], acc_full;
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jblocks = s_k / kBM;
    const int64_t head = blockIdx.x / jblocks;
    const int j0 = (blockIdx.x % jblocks) * kBM;
    const int nk = s_q / kBK;
    const float* Ph = P + head * (int64_t)s_q * s_k;
    const float* dOh = dO + head * (int64_t)s_q * N;
    const uint32_t* mh_base = mask;  // word index uses the global element index
    const int64_t e_head = head * (int64_t)s_q * s_k;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesG; ++s) {
            mbar_init(&full[s], kProducers);
            mbar_init(&empty[s], 1);
        }
        mbar_init(&acc_full, 1);
        mbar_fence_init();
    }
    if (warp == kProducers / 32) {  // the MMA warp allocates the accumulators
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(&tmem_base_sh)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp < kProducers / 32) {
        // ---------------- producers ----------------
        // A: thread t owns dV row m = t (j0 + t); per stage it reads P[i][j0+t]
        //    down the 32 K-rows (a warp = one coalesced 128-byte segment per
        //    row) and the keep bit from the row's mask word (lane l loads row
        //    l's word, shuffled per row).
        // B: thread t owns dO column n = t % N over K-rows 8*(t/N)..+7 (and
        //    further K-groups when N < 64).
        const int t = threadIdx.x;
        constexpr int kBK8 = kBK * N / kProducers;  // dO elements per thread per stage
        static_assert(kBK8 % 4 == 0, "dO chunk");
        const int bn = t % N, bk0 = (t / N) * kBK8;
        float pv[kBK], ov[kBK8];
        uint32_t mword;
        const int jcol = j0 + t;
        auto load = [&](int ks) {
            const int i0 = ks * kBK;
#pragma unroll
            for (int k = 0; k < kBK; ++k) pv[k] = ld_stream(Ph + (int64_t)(i0 + k) * s_k + jcol);
            // row (i0 + lane)'s mask word covering columns j0 + 32*(t/32) ..
            const int64_t e = e_head + (int64_t)(i0 + lane) * s_k + j0 + (t & ~31);
            mword = __ldg(mh_base + (e >> 5));
#pragma unroll
            for (int k = 0; k < kBK8; ++k) ov[k] = ld_stream(dOh + (int64_t)(i0 + bk0 + k) * N + bn);
        };
        load(0);
        for (int ks = 0; ks < nk; ++ks) {
            const int s = ks % kStagesG;
            if (ks >= kStagesG) mbar_wait(&empty[s], (uint32_t)(((ks / kStagesG) + 1) & 1));
            unsigned char* st = base + s * kStageBytes;
            unsigned char* a_hi = st;
            unsigned char* a_lo = st + kAbytes;
            unsigned char* b_hi = st + 2 * kAbytes;
            unsigned char* b_lo = b_hi + kBbytes;
#pragma unroll
            for (int q = 0; q < kBK / 4; ++q) {
                float hi[4], lo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = 4 * q + u;
                    const uint32_t w = __shfl_sync(kFull, mword, k);
                    // D exactly as dropout_apply / the forward's D (one fp64 rounding)
                    const float d = ((w >> lane) & 1u) ? (float)((double)pv[k] * scale) : 0.0f;
                    hi[u] = tf32_rna(d);
                    lo[u] = tf32_rna(d - hi[u]);
                }
                const uint32_t off = sw128_k_offset(t, q);
                *reinterpret_cast<float4*>(a_hi + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(a_lo + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
#pragma unroll
            for (int q = 0; q < kBK8 / 4; ++q) {
                float hi[4], lo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const float o = ov[4 * q + u];
                    hi[u] = tf32_rna(o);
                    lo[u] = tf32_rna(o - hi[u]);
                }
                const uint32_t off = sw128_k_offset(bn, (bk0 >> 2) + q);
                *reinterpret_cast<float4*>(b_hi + off) = make_float4(hi[0], hi[1], hi[2], hi[3]);
                *reinterpret_cast<float4*>(b_lo + off) = make_float4(lo[0], lo[1], lo[2], lo[3]);
            }
            if (ks + 1 < nk) load(ks + 1);  // next chunk's loads in flight during the MMAs
            fence_proxy_async_smem();       // generic-proxy writes -> visible to tcgen05
            mbar_arrive(&full[s]);
        }
        // ---------------- epilogue ----------------
        mbar_wait(&acc_full, 0);
        tc_fence_after();
        const int mb = warp / 4, quad = warp % 4;
        const int row = j0 + mb * 128 + quad * 32 + lane;
        float* out = dV + head * (int64_t)s_k * N + (int64_t)row * N;
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
            float v[16];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mb * N + c0);
            tmem_ld16(ta, v);
#pragma unroll
            for (int set = 1; set < kSets; ++set) {  // fixed order: bitwise reproducible
                float w[16];
                tmem_ld16(ta + (uint32_t)(set * 2 * N), w);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += w[i];
            }
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                st_stream(reinterpret_cast<float4*>(out + c0 + i),
                          make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]));
        }
    } else if (lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_tf32_k(128, N);
        for (int ks = 0; ks < nk; ++ks) {
            const int s = ks % kStagesG;
            mbar_wait(&full[s], (uint32_t)((ks / kStagesG) & 1));
            tc_fence_after();
            const uint32_t st = smem_u32(base + s * kStageBytes);
            const uint32_t a_hi = st, a_lo = st + kAbytes;
            const uint32_t b_hi = st + 2 * kAbytes, b_lo = b_hi + kBbytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 8; ++kk) {  // K = 8 per MMA: +32 bytes along the rows
                const uint64_t bh = umma_desc_sw128(b_hi + kk * 32, 16, 1024);
                const uint64_t bl = umma_desc_sw128(b_lo + kk * 32, 16, 1024);
#pragma unroll
                for (int mb = 0; mb < 2; ++mb) {
                    const uint32_t ao = mb * 128 * 128 + kk * 32;  // 128 rows x 128 B per M-block
                    const uint64_t ah = umma_desc_sw128(a_hi + ao, 16, 1024);
                    const uint64_t al = umma_desc_sw128(a_lo + ao, 16, 1024);
                    const int set = kk % kSets;
                    const uint32_t acc = tmem + (uint32_t)(set * 2 * N + mb * N);
                    mma_tf32(acc, al, bh, idesc, ks != 0 || kk >= kSets);  // small terms first
                    mma_tf32(acc, ah, bl, idesc, 1);
                    mma_tf32(acc, ah, bh, idesc, 1);
                }
            }
            mma_commit(&empty[s]);  // stage s may be refilled once these MMAs retire
        }
        mma_commit(&acc_full);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kProducers / 32) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

template <int N>
size_t dv_smem() {
    return 1024 + (size_t)kStagesG * (2 * kBM * kBK * 4 + 2 * N * kBK * 4);
}

template <int N>
cudaError_t launch_dv(const float* P, const uint32_t* mask, double scale, const float* dO, float* dV,
                      int64_t heads, int64_t s_q, int64_t s_k, cudaStream_t st) {
    auto k = dv_recompute_gemm_kernel<N>;
    const size_t smem = dv_smem<N>();
    (void)grid_for((const void*)k, kThreadsG, smem, 1);  // opts the kernel into its smem size
    const int64_t grid = heads * (s_k / kBM);
    launch(k, (int)grid, kThreadsG, smem, st)(P, mask, scale, dO, dV, (int)s_q, (int)s_k);
    return cudaGetLastError();
}

}  // namespace

bool dv_gemm_supported(int64_t s_q, int64_t s_k, int64_t d) {
    return s_q > 0 && s_k > 0 && s_q % kBK == 0 && s_k % kBM == 0 && (d == 32 || d == 64 || d == 128) &&
           s_q <= (1 << 20) && s_k <= (1 << 20);
}

cudaError_t launch_dv_recompute_gemm(const float* P, const uint32_t* mask, double scale,
                                     const float* dO, float* dV, int64_t heads, int64_t s_q,
                                     int64_t s_k, int64_t d, cudaStream_t st) {
    if (heads == 0) return cudaSuccess;
    switch (d) {
        case 32: return launch_dv<32>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        case 64: return launch_dv<64>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        case 128: return launch_dv<128>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tb
