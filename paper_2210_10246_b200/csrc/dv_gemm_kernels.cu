// dv_gemm_kernels.cu -- the attention-dropout recompute fused into its
// consumers, the attention-context GEMM ctx = D @ V (forward) and its
// backward's dV = D^T @ dO, on the 5th-generation tensor cores (sm_100a).
//
// The reference's Sub-Layer Dropout Recomputation keeps only P and the mask;
// the consumer of the dropped-out map D gets it from the recompute rule
// "dropout-rescale" (graph.cpp:46-50 -> BackwardCtx::stash, tape.cpp:244-264;
// rule ops_tempo.cpp:17-26 = dropout_apply, ops_reference.cpp:147-153), and
// the forward materialises D for ctx (ops_tempo.cpp:196-210).  Here D never
// exists in memory at all: the producer warps rebuild D' = keep ? P : 0 (the
// 1/(1-p) is applied in the epilogue) tile by tile and write it, split into
// TF32 hi + lo, straight into TMEM as the A operand of tcgen05.mma.  HBM
// traffic per attention element: P (4 B) + the mask bit.
//
// The product kernel is ctx_recompute_gemm_ta_kernel<N, DRAIN, DV> (below,
// "ctx with the A operand in TMEM"): persistent, warp-specialised (TMA
// loader lane, 16 producer warps in two alternating halves, one MMA lane),
// 32-wide K slices through a 4-deep TMA ring, 3xTF32 (hi*hi + hi*lo + lo*hi
// -- lo*hi first), accumulation error flat in K (set rotation up to K = 1024,
// drained ping-pong accumulators beyond).  Why A in TMEM: tcgen05 kind::tf32
// takes no MN-major smem operands on this part (tests/tools/umma_probe.cu),
// so D^T needs a transpose anyway; a producer thread that owns one output
// row = one TMEM lane does it on the way in, and the MMA then reads A from
// TMEM instead of 12 B per element of smem (tests/tools/tmem_a_probe.cu).
//
// Kept as A/B baselines and fallbacks (DESIGN 3d has the measured history):
// dv_recompute_gemm_kernel (register-prefetch producers, smem operands; also
// d = 128 and the path without tensor maps), dv_recompute_gemm_staged_kernel
// and ctx_recompute_gemm_kernel (TMA staging, smem operands; TM_DV_TA=0 /
// TM_CTX_TA=0).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kBM = 256;             // dV rows per CTA (two M=128 accumulators)
constexpr int kBK = 32;              // K rows (query positions) per stage
constexpr int kStagesG = 2;
constexpr int kProducers = 256;      // 8 warps
constexpr int kThreadsG = kProducers + 32;

#ifndef TM_DV_FAST_RNA
#define TM_DV_FAST_RNA 1
#endif
// Round to TF32 (10 explicit mantissa bits), nearest, ties away from zero:
// cvt.rna.tf32.f32.  On sm_100 that conversion is a multi-instruction
// sequence (inf/NaN check, integer rounding, mask), the producers' largest
// ALU cost (ncu).  On the sign-magnitude bit pattern, adding half a TF32 ulp
// (bit 12) and clearing the 13 low bits IS that rounding for finite values;
// inf/NaN keep their bits (a NaN payload could carry into the sign).  The
// split's low part x - hi is always finite and small, so it skips the check.
#ifndef TM_DV_SPLIT
#define TM_DV_SPLIT 1
#endif
#if !TM_DV_SPLIT
__device__ __forceinline__ float tf32_rna(float x) {
#if TM_DV_FAST_RNA
    const uint32_t u = __float_as_uint(x);
    const uint32_t r = (u + 0x1000u) & 0xffffe000u;
    return __uint_as_float((u & 0x7f800000u) == 0x7f800000u ? u : r);
#else
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
#endif
}
__device__ __forceinline__ float tf32_rna_finite(float x) {  // x finite
#if TM_DV_FAST_RNA
    return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
#else
    return tf32_rna(x);
#endif
}
#endif

// 3xTF32 operand split x = hi + lo.  hi = x rounded to TF32 (nearest, ties
// away: the integer form, which keeps +-inf and turns a NaN into a NaN or, for
// a NaN with the top mantissa bits set, -0 -- its lo is then NaN, so NaN still
// propagates through the hi*lo products); lo = x - hi is exact and left
// unrounded: the tensor core reads the top 19 bits of an fp32 TF32 operand,
// so lo is truncated there (error < 2^-21 |x| per element, vs 2^-22 with a
// rounded lo) at 3 instructions instead of ~10.  TM_DV_SPLIT=0: both parts
// rounded with the inf/NaN guards.
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
#if TM_DV_SPLIT
    hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
    lo = x - hi;
#else
    hi = tf32_rna(x);
    lo = isfinite(x) ? tf32_rna_finite(x - hi) : x - hi;
#endif
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
                    split_tf32(d, hi[u], lo[u]);
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
                    split_tf32(o, hi[u], lo[u]);
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

// ---- v2: bulk-copy staging ----------------------------------------------
// The register-prefetch producers above keep only ~40 KB per SM in flight
// (one K-chunk of 32 rows per thread): the kernel waits on DRAM latency
// (2.1 TB/s).  Here a loader lane streams 16-row slices of P, their mask
// words and dO into a kSS-deep shared-memory staging ring with cp.async.bulk
// (mbarrier completion, ~100 KB in flight per SM), 16 producer warps
// transpose each slice from the ring (a warp reads 32 consecutive floats of a
// row: conflict-free) into a kOS-deep ring of K-major SWIZZLE_64B operand
// tiles (16 K-rows = 64-byte rows, 8-row 512-byte atoms), and the MMA lane
// issues 2 K-steps x 2 M-blocks x 3 products per slice.  The dropout scale
// 1/(1-p) is applied to dV in the epilogue, so staging D' = keep ? P : 0 is
// a select.
constexpr int kBKs = 16;  // K rows per staging slice = per operand stage

__device__ __forceinline__ uint32_t sw64_k_offset(int mn, int kchunk) {
    // byte offset of 16-byte K-chunk `kchunk` (< 4) of row mn, K-major
    // SWIZZLE_64B: [mn/8][mn%8][64 B], chunk ^ ((mn%8) >> 1) (Swizzle<2,4,3>)
    const int row = mn & 7;
    return (uint32_t)((mn >> 3) * 512 + row * 64 + ((kchunk ^ (row >> 1)) << 4));
}
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t smem_addr, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3fff);
    d |= (uint64_t)1 << 16;  // LBO (unused for swizzled K-major)
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3fff) << 32;
    d |= (uint64_t)1 << 46;  // version
    d |= (uint64_t)4 << 61;  // SWIZZLE_64B
    return d;
}
__device__ __forceinline__ void sts128(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(a), "f"(b), "f"(c),
                 "f"(d)
                 : "memory");
}
__device__ __forceinline__ void sts64(uint32_t addr, float a, float b) {
    asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, float a) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(a) : "memory");
}
__device__ __forceinline__ float lds32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ldsu32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

#ifndef TM_DV_SS
#define TM_DV_SS 5
#endif
#ifndef TM_DV_OS
#define TM_DV_OS 3
#endif
#ifndef TM_DV_BM
// dV rows per CTA: 256 (1 CTA/SM) or 128 (2 CTAs/SM, 8 producer warps each).
// A/B at BERT-large: 414 vs 449 us, bit-identical -- two CTAs per SM hide no
// latency that matters and each loads the head's dO slices once per 128
// rows (twice the dO traffic): the producers' issue rate is the limit.
#define TM_DV_BM 256
#endif
template <int N, int BM>
struct StagedCfg {
    static constexpr int kSS = BM == 256 ? TM_DV_SS : 4;           // staging slices in flight
    static constexpr int kOS = BM == 256 ? TM_DV_OS : 2;           // operand stages
    static constexpr int kSP = 2 * BM;                             // producer threads
    static constexpr int kPbytes = kBKs * BM * 4;                  // 16 / 8 KB
    static constexpr int kObytes = kBKs * N * 4;                   // 2 / 4 KB
    static constexpr int kMbytes = kBKs * (BM / 32) * 4;           // 512 / 256 B of mask words
    static constexpr int kSlice = kPbytes + kObytes + kMbytes;
    static constexpr int kAbytes = BM * kBKs * 4;                  // 16 / 8 KB
    static constexpr int kBbytes = N * kBKs * 4;
    static constexpr int kOpStage = 2 * kAbytes + 2 * kBbytes;
    static constexpr size_t kSmem = 1024 + (size_t)kOS * kOpStage + (size_t)kSS * kSlice;
    static_assert(kSmem <= (BM == 256 ? 227 : 110) * 1024, "smem");
};

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

template <int N, int BM>
__global__ void __launch_bounds__(2 * BM + 64, BM == 256 ? 1 : 2) dv_recompute_gemm_staged_kernel(
    const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_m,
    const __grid_constant__ CUtensorMap tm_o, double scale, float* __restrict__ dV, int s_q,
    int s_k) {
    using Cfg = StagedCfg<N, BM>;
    constexpr int kSP = Cfg::kSP;
    constexpr int kMB = BM / 128;  // M = 128 blocks (TMEM accumulators per set)
    constexpr int kSets = 512 / (2 * N) >= 4 ? 4 : 512 / (2 * N);
    constexpr int kTmemCols = kSets * kMB * N < 32 ? 32 : kSets * kMB * N;
    constexpr int kSS = Cfg::kSS, kOS = Cfg::kOS;
    grid_dep_wait();
    grid_dep_launch();
    extern __shared__ __align__(1024) unsigned char gsm[];
    const uint32_t base = (smem_u32(gsm) + 1023u) & ~1023u;      // shared-space addresses
    const uint32_t stage_base = base + kOS * Cfg::kOpStage;       // staging ring after the operands
    unsigned char* stage_ptr = gsm + (stage_base - smem_u32(gsm)); // generic view (bulk copies)
    __shared__ uint64_t full[kOS], empty[kOS], acc_full, sfull[kSS], sempty[kSS];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jblocks = s_k / BM;
    const int64_t head = blockIdx.x / jblocks;
    const int j0 = (blockIdx.x % jblocks) * BM;
    const int nsl = s_q / kBKs;  // slices = operand stages
    constexpr int kMMAWarp = kSP / 32, kLoadWarp = kSP / 32 + 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kOS; ++s) {
            mbar_init(&full[s], kSP / 32);  // one arrival per producer warp
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kSS; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], kSP / 32);
        }
        mbar_init(&acc_full, 1);
        mbar_fence_init();
    }
    if (warp == kMMAWarp) {
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

    if (warp < kMMAWarp) {
        // ---------------- producers: staging slice -> K-major operands ----
        // A: thread t owns dV row m = t % 256 and K-rows 8*(t/256)..+7 of the
        //    slice: D' = keep ? P : 0, split hi/lo TF32.  B: dO column
        //    bn = t % N, K-rows bk.. (1 or 2 per thread).
        const int t = threadIdx.x;
        const int m = t % BM, kh = t / BM;
        constexpr int kOPT = kBKs * N / kSP;  // 1, 2 or 4 dO values per thread
        static_assert(kOPT == 1 || kOPT == 2 || kOPT == 4, "dO slice split");
        const int bn = t % N, bk = (t / N) * kOPT;
        for (int sl = 0; sl < nsl; ++sl) {
            const int ss = sl % kSS, s = sl % kOS;
            mbar_wait(&sfull[ss], (uint32_t)((sl / kSS) & 1));
            const uint32_t sp = stage_base + ss * Cfg::kSlice;
            float pv[8];
            uint32_t w[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                pv[k] = lds32(sp + (uint32_t)(((kh * 8 + k) * BM + m) * 4));
                w[k] = ldsu32(sp + Cfg::kPbytes + Cfg::kObytes + (uint32_t)(((kh * 8 + k) * (BM / 32) + (m >> 5)) * 4));
            }
            float ov[kOPT];
#pragma unroll
            for (int k = 0; k < kOPT; ++k) ov[k] = lds32(sp + Cfg::kPbytes + (uint32_t)(((bk + k) * N + bn) * 4));
            __syncwarp();  // the warp is done reading slice ss: one arrival for it
            if (lane == 0) mbar_arrive(&sempty[ss]);
            if (sl >= kOS) mbar_wait(&empty[s], (uint32_t)(((sl / kOS) + 1) & 1));
            const uint32_t a_hi = base + s * Cfg::kOpStage, a_lo = a_hi + Cfg::kAbytes;
            const uint32_t b_hi = a_lo + Cfg::kAbytes, b_lo = b_hi + Cfg::kBbytes;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                float hi[4], lo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = 4 * q + u;
                    const float d = ((w[k] >> lane) & 1u) ? pv[k] : 0.0f;
                    split_tf32(d, hi[u], lo[u]);
                }
                const uint32_t off = sw64_k_offset(m, kh * 2 + q);
                sts128(a_hi + off, hi[0], hi[1], hi[2], hi[3]);
                sts128(a_lo + off, lo[0], lo[1], lo[2], lo[3]);
            }
            {
                float hi[kOPT], lo[kOPT];
#pragma unroll
                for (int u = 0; u < kOPT; ++u) {
                    split_tf32(ov[u], hi[u], lo[u]);
                }
                const uint32_t off = sw64_k_offset(bn, bk >> 2) + (uint32_t)((bk & 3) * 4);
                if (kOPT == 4) {
                    sts128(b_hi + off, hi[0], hi[1 % kOPT], hi[2 % kOPT], hi[3 % kOPT]);
                    sts128(b_lo + off, lo[0], lo[1 % kOPT], lo[2 % kOPT], lo[3 % kOPT]);
                } else if (kOPT == 2) {
                    sts64(b_hi + off, hi[0], hi[kOPT - 1]);
                    sts64(b_lo + off, lo[0], lo[kOPT - 1]);
                } else {
                    sts32(b_hi + off, hi[0]);
                    sts32(b_lo + off, lo[0]);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();  // every lane fenced its operand stores: one arrival per warp
            if (lane == 0) mbar_arrive(&full[s]);
        }
        // ---------------- epilogue: dV = (1/(1-p)) * sum of the sets ----------
        mbar_wait(&acc_full, 0);
        tc_fence_after();
        const int quad = warp % 4, mb = (warp / 4) % kMB, half = warp / (4 * kMB);  // 2 column halves
        const int row = j0 + mb * 128 + quad * 32 + lane;
        float* out = dV + head * (int64_t)s_k * N + (int64_t)row * N;
        const float sc = (float)scale;
#pragma unroll
        for (int c0 = half * (N / 2); c0 < (half + 1) * (N / 2); c0 += 16) {
            float v[16];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mb * N + c0);
            static_assert(kSP / 32 == 8 * kMB, "two warps per (TMEM lane quadrant, M-block)");
            tmem_ld16(ta, v);
#pragma unroll
            for (int set = 1; set < kSets; ++set) {
                float wv[16];
                tmem_ld16(ta + (uint32_t)(set * kMB * N), wv);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += wv[i];
            }
#pragma unroll
            for (int i = 0; i < 16; i += 4)
                st_stream(reinterpret_cast<float4*>(out + c0 + i),
                          make_float4(v[i] * sc, v[i + 1] * sc, v[i + 2] * sc, v[i + 3] * sc));
        }
    } else if (warp == kMMAWarp && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_tf32_k(128, N);
        for (int sl = 0; sl < nsl; ++sl) {
            const int s = sl % kOS;
            mbar_wait(&full[s], (uint32_t)((sl / kOS) & 1));
            tc_fence_after();
            const uint32_t a_hi = base + s * Cfg::kOpStage, a_lo = a_hi + Cfg::kAbytes;
            const uint32_t b_hi = a_lo + Cfg::kAbytes, b_lo = b_hi + Cfg::kBbytes;
#pragma unroll
            for (int kk = 0; kk < kBKs / 8; ++kk) {  // K = 8 per MMA: +32 bytes along 64-byte rows
                const uint64_t bh = umma_desc_sw64(b_hi + kk * 32, 512);
                const uint64_t bl = umma_desc_sw64(b_lo + kk * 32, 512);
                const int gk = sl * (kBKs / 8) + kk;  // global K-step
                const int set = gk % kSets;
#pragma unroll
                for (int mb = 0; mb < kMB; ++mb) {
                    const uint32_t ao = mb * 128 * 64 + kk * 32;  // 128 rows x 64 B per M-block
                    const uint64_t ah = umma_desc_sw64(a_hi + ao, 512);
                    const uint64_t al = umma_desc_sw64(a_lo + ao, 512);
                    const uint32_t acc = tmem + (uint32_t)(set * kMB * N + mb * N);
                    mma_tf32(acc, al, bh, idesc, gk >= kSets);
                    mma_tf32(acc, ah, bl, idesc, 1);
                    mma_tf32(acc, ah, bh, idesc, 1);
                }
            }
            mma_commit(&empty[s]);
        }
        mma_commit(&acc_full);
    } else if (warp == kLoadWarp && lane == 0) {
        // ---------------- loader: three 2D TMA loads per slice ---------------
        // (P rows [16 x 256], their mask words [16 x 8], dO rows [16 x N]);
        // 33 one-dimensional bulk copies per slice were the limiter
        const int y0 = (int)(head * s_q);
        for (int sl = 0; sl < nsl; ++sl) {
            const int ss = sl % kSS;
            if (sl >= kSS) mbar_wait(&sempty[ss], (uint32_t)(((sl / kSS) + 1) & 1));
            unsigned char* sp = stage_ptr + ss * Cfg::kSlice;
            mbar_expect_tx(&sfull[ss], Cfg::kSlice);
            const int y = y0 + sl * kBKs;
            tma_load_2d(sp, &tm_p, j0, y, &sfull[ss]);
            tma_load_2d(sp + Cfg::kPbytes + Cfg::kObytes, &tm_m, j0 / 32, y, &sfull[ss]);
            tma_load_2d(sp + Cfg::kPbytes, &tm_o, 0, y, &sfull[ss]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMMAWarp) {
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

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2D row-major tensor [rows][cols] of 4-byte elements, box [box_rows][box_cols]
bool make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dt, const void* ptr, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols,
                  CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
    auto enc = tmap_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 4};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N>
cudaError_t launch_dv_staged(const float* P, const uint32_t* mask, double scale, const float* dO,
                             float* dV, int64_t heads, int64_t s_q, int64_t s_k, cudaStream_t st) {
    constexpr int BM = TM_DV_BM;
    CUtensorMap tp, tmk, to;
    const uint64_t rows = (uint64_t)(heads * s_q);
    if (!make_tmap_2d(&tp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, P, rows, (uint64_t)s_k, kBKs, BM) ||
        !make_tmap_2d(&tmk, CU_TENSOR_MAP_DATA_TYPE_UINT32, mask, rows, (uint64_t)(s_k / 32), kBKs,
                      BM / 32) ||
        !make_tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dO, rows, (uint64_t)N, kBKs, N))
        return launch_dv<N>(P, mask, scale, dO, dV, heads, s_q, s_k, st);  // no tensor maps
    auto k = dv_recompute_gemm_staged_kernel<N, BM>;
    const size_t smem = StagedCfg<N, BM>::kSmem;
    constexpr int threads = StagedCfg<N, BM>::kSP + 64;
    (void)grid_for((const void*)k, threads, smem, 1);
    const int64_t grid = heads * (s_k / BM);
    launch(k, (int)grid, threads, smem, st)(tp, tmk, to, scale, dV, (int)s_q, (int)s_k);
    return cudaGetLastError();
}

// ---- the FORWARD consumer: ctx = D @ V with D rebuilt from P + mask -------
// The attention forward's consumer of the dropped-out map (tempo_ops::sdpa,
// ops_tempo.cpp:196-210: matmul(dropout_recompute(probs), v)) as one tcgen05
// GEMM that never reads D: per (head, 128-query block), ctx[i, c] = (1/(1-p))
// * sum_j keep[i, j] P[i, j] V[j, c] -- M = s_q (i), N = d (c), K = s_k (j).
// Here P's rows are already K-major, so the loader's 2D TMA stages each
// 256 x 16 P tile with SWIZZLE_64B, which IS the UMMA K-major SWIZZLE_64B
// operand layout: the producers split every element in place (select on the
// keep bit, 3xTF32 hi/lo) at the same smem offset, vectorised and
// conflict-free; only V (row-major [j][c], MN-major) is transposed by the
// producers, as dO is in the dV GEMM.  (A first version with 128-row CTAs and
// 32-column SWIZZLE_128B slices took 0.53 ms at BERT-large: each head's V was
// read by four CTAs.)  With the dV GEMM, D exists in neither
// pass: the softmax forward writes P and the mask bits only (8.125 B/elem
// instead of 12.125).
constexpr int kCM = 256;        // query rows per CTA (two M = 128 accumulators)
constexpr int kCK = 16;         // key columns per slice (64-byte operand rows, SWIZZLE_64B)
constexpr int kCSP = 512;       // 16 producer warps: 2 per query row
constexpr int kCThreads = kCSP + 64;

template <int N>
struct CtxCfg {
    static constexpr int kSS = 4, kOS = 3;
    static constexpr int kPbytes = kCM * kCK * 4;   // 16 KB, swizzled
    static constexpr int kVbytes = kCK * N * 4;     // 4 KB (N = 64)
    static constexpr int kSlice = kPbytes + kVbytes;
    static constexpr int kAbytes = kCM * kCK * 4;
    static constexpr int kBbytes = N * kCK * 4;
    static constexpr int kOpStage = 2 * kAbytes + 2 * kBbytes;
    static constexpr size_t kSmem = 1024 + (size_t)kOS * kOpStage + (size_t)kSS * kSlice;
    static_assert(kSmem <= 227 * 1024, "smem");
};

template <int N>
__global__ void __launch_bounds__(kCThreads, 1) ctx_recompute_gemm_kernel(
    const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_v,
    const uint32_t* __restrict__ mask, double scale, float* __restrict__ ctx, int s_q, int s_k) {
    using Cfg = CtxCfg<N>;
    constexpr int kSets = 512 / (2 * N) >= 4 ? 4 : 512 / (2 * N);
    constexpr int kTmemCols = kSets * 2 * N;
    constexpr int kSS = Cfg::kSS, kOS = Cfg::kOS;
    grid_dep_wait();
    grid_dep_launch();
    extern __shared__ __align__(1024) unsigned char gsm[];
    const uint32_t base = (smem_u32(gsm) + 1023u) & ~1023u;
    const uint32_t stage_base = base + kOS * Cfg::kOpStage;
    unsigned char* stage_ptr = gsm + (stage_base - smem_u32(gsm));
    __shared__ uint64_t full[kOS], empty[kOS], acc_full, sfull[kSS], sempty[kSS];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int iblocks = (s_q + kCM - 1) / kCM;  // a ragged last block: rows >= s_q are
    const int64_t head = blockIdx.x / iblocks;  // computed on the next head's (or zero-
    const int i0 = (blockIdx.x % iblocks) * kCM;  // filled) P rows and not stored
    const int nsl = s_k / kCK;
    constexpr int kMMAWarp = kCSP / 32, kLoadWarp = kCSP / 32 + 1;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kOS; ++s) {
            mbar_init(&full[s], kCSP / 32);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kSS; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], kCSP / 32);
        }
        mbar_init(&acc_full, 1);
        mbar_fence_init();
    }
    if (warp == kMMAWarp) {
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

    if (warp < kMMAWarp) {
        // ---------------- producers ----------------
        // A: thread t owns query row m = t % 256 and the two 16-byte K-chunks
        //    2h, 2h+1 (h = t / 256) of the slice, at the same swizzled offset
        //    in staging and operand.
        // B: thread t owns V column n = t % N, K-rows kq*KV..+KV-1.
        const int t = threadIdx.x;
        const int m = t % kCM, h = t / kCM;
        constexpr int kKV = kCK * N / kCSP;  // V values per thread per slice (2 for N = 64)
        static_assert(kKV == 1 || kKV == 2, "V chunk");
        const int bn = t % N, bk = (t / N) * kKV;
        const bool row_in = i0 + m < s_q;
        const uint32_t* mrow = mask + (((head * (int64_t)s_q + i0 + m) * s_k) >> 5);
        // the mask word of columns 32*(sl/2).. serves two slices; the next
        // one is loaded a slice pair ahead (a per-row word: 32 sectors/warp)
        uint32_t w = 0, w_next = row_in ? __ldg(mrow) : 0u;
        for (int sl = 0; sl < nsl; ++sl) {
            const int ss = sl % kSS, s = sl % kOS;
            if ((sl & 1) == 0) {
                w = w_next;
                if (row_in && sl + 2 < nsl) w_next = __ldg(mrow + (sl >> 1) + 1);
            }
            mbar_wait(&sfull[ss], (uint32_t)((sl / kSS) & 1));
            const uint32_t sp = stage_base + ss * Cfg::kSlice;
            float4 pv[2];
#pragma unroll
            for (int c = 0; c < 2; ++c)
                asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                             : "=f"(pv[c].x), "=f"(pv[c].y), "=f"(pv[c].z), "=f"(pv[c].w)
                             : "r"(sp + sw64_k_offset(m, 2 * h + c)));
            float ov[kKV];
#pragma unroll
            for (int k = 0; k < kKV; ++k)
                ov[k] = lds32(sp + Cfg::kPbytes + (uint32_t)(((bk + k) * N + bn) * 4));
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[ss]);
            if (sl >= kOS) mbar_wait(&empty[s], (uint32_t)(((sl / kOS) + 1) & 1));
            const uint32_t a_hi = base + s * Cfg::kOpStage, a_lo = a_hi + Cfg::kAbytes;
            const uint32_t b_hi = a_lo + Cfg::kAbytes, b_lo = b_hi + Cfg::kBbytes;
            const uint32_t wsl = w >> (16 * (sl & 1));  // this slice's 16 keep bits
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const float e[4] = {pv[c].x, pv[c].y, pv[c].z, pv[c].w};
                float hi[4], lo[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int k = 4 * (2 * h + c) + u;  // column 16*sl + k
                    const float d = ((wsl >> k) & 1u) ? e[u] : 0.0f;
                    split_tf32(d, hi[u], lo[u]);
                }
                const uint32_t off = sw64_k_offset(m, 2 * h + c);
                sts128(a_hi + off, hi[0], hi[1], hi[2], hi[3]);
                sts128(a_lo + off, lo[0], lo[1], lo[2], lo[3]);
            }
            {
                float hi[kKV], lo[kKV];
#pragma unroll
                for (int u = 0; u < kKV; ++u) {
                    split_tf32(ov[u], hi[u], lo[u]);
                }
                const uint32_t off = sw64_k_offset(bn, bk >> 2) + (uint32_t)((bk & 3) * 4);
                if (kKV == 2) {
                    sts64(b_hi + off, hi[0], hi[kKV - 1]);
                    sts64(b_lo + off, lo[0], lo[kKV - 1]);
                } else {
                    sts32(b_hi + off, hi[0]);
                    sts32(b_lo + off, lo[0]);
                }
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[s]);
        }
        // ---------------- epilogue: ctx = (1/(1-p)) * sum of the sets ------
        mbar_wait(&acc_full, 0);
        tc_fence_after();
        const int quad = warp % 4, mb = (warp / 4) % 2, half = warp / 8;
        const int row = i0 + mb * 128 + quad * 32 + lane;
        float* out = ctx + (head * (int64_t)s_q + row) * N;
        const float sc = (float)scale;
        const bool store = row < s_q;
#pragma unroll
        for (int c0 = half * (N / 2); c0 < (half + 1) * (N / 2); c0 += 16) {
            float v[16];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(mb * N + c0);
            tmem_ld16(ta, v);
#pragma unroll
            for (int set = 1; set < kSets; ++set) {
                float wv[16];
                tmem_ld16(ta + (uint32_t)(set * 2 * N), wv);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] += wv[i];
            }
            if (store) {  // (the tcgen05.ld above stays warp-uniform)
#pragma unroll
                for (int i = 0; i < 16; i += 4)
                    st_stream(reinterpret_cast<float4*>(out + c0 + i),
                              make_float4(v[i] * sc, v[i + 1] * sc, v[i + 2] * sc, v[i + 3] * sc));
            }
        }
    } else if (warp == kMMAWarp && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = idesc_tf32_k(128, N);
        for (int sl = 0; sl < nsl; ++sl) {
            const int s = sl % kOS;
            mbar_wait(&full[s], (uint32_t)((sl / kOS) & 1));
            tc_fence_after();
            const uint32_t a_hi = base + s * Cfg::kOpStage, a_lo = a_hi + Cfg::kAbytes;
            const uint32_t b_hi = a_lo + Cfg::kAbytes, b_lo = b_hi + Cfg::kBbytes;
#pragma unroll
            for (int kk = 0; kk < kCK / 8; ++kk) {  // K = 8 per MMA: +32 bytes along 64-byte rows
                const uint64_t bh = umma_desc_sw64(b_hi + kk * 32, 512);
                const uint64_t bl = umma_desc_sw64(b_lo + kk * 32, 512);
                const int gk = sl * (kCK / 8) + kk;
                const int set = gk % kSets;
#pragma unroll
                for (int mb = 0; mb < 2; ++mb) {
                    const uint32_t ao = mb * 128 * 64 + kk * 32;  // 128 rows x 64 B per M-block
                    const uint64_t ah = umma_desc_sw64(a_hi + ao, 512);
                    const uint64_t al = umma_desc_sw64(a_lo + ao, 512);
                    const uint32_t acc = tmem + (uint32_t)(set * 2 * N + mb * N);
                    mma_tf32(acc, al, bh, idesc, gk >= kSets);  // small terms first
                    mma_tf32(acc, ah, bl, idesc, 1);
                    mma_tf32(acc, ah, bh, idesc, 1);
                }
            }
            mma_commit(&empty[s]);
        }
        mma_commit(&acc_full);
    } else if (warp == kLoadWarp && lane == 0) {
        // ---------------- loader: the P tile (swizzled) and the V rows ------
        const int y_p = (int)(head * s_q + i0), y_v0 = (int)(head * s_k);
        for (int sl = 0; sl < nsl; ++sl) {
            const int ss = sl % kSS;
            if (sl >= kSS) mbar_wait(&sempty[ss], (uint32_t)(((sl / kSS) + 1) & 1));
            unsigned char* sp = stage_ptr + ss * Cfg::kSlice;
            mbar_expect_tx(&sfull[ss], Cfg::kSlice);
            tma_load_2d(sp, &tm_p, sl * kCK, y_p, &sfull[ss]);
            tma_load_2d(sp + Cfg::kPbytes, &tm_v, 0, y_v0 + sl * kCK, &sfull[ss]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMMAWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                     "n"(kTmemCols)
                     : "memory");
    }
}

// ---- ctx with the A operand in TMEM ----------------------------------------
// The producers above write every A element twice to shared memory (hi, lo),
// fence the generic->async proxy per slice, and the MMA reads A back from smem
// three times (al.bh, ah.bl, ah.bh): ~34 B of smem traffic per P element.
// tcgen05.mma also takes A from TMEM (tests/tools/tmem_a_probe.cu: exact for
// kind::tf32, lane = row, one column per K element), and a producer thread
// owns one query row = one TMEM lane: it splits its 8 P values of the slice
// and tcgen05.st's them (hi, lo: 8 columns each) straight into the A stage.
// Only V's K-major B tile still goes through smem, written by warps 0-3 (the
// only ones that fence the async proxy).  TMEM: kSets accumulator sets x 2
// M-blocks x N columns + kAS A stages x 2 M-blocks x 32 columns = 512.
#ifndef TM_CTX_TA
#define TM_CTX_TA 1
#endif
#ifndef TM_CTX_TA_SS
#define TM_CTX_TA_SS 4
#endif
#ifndef TM_CTX_TA_SETS
#define TM_CTX_TA_SETS 2
#endif
#ifndef TM_CTX_TA_K
#define TM_CTX_TA_K 32   // key columns per slice: 32 (SWIZZLE_128B) or 16 (SWIZZLE_64B)
#endif
#ifndef TM_CTX_DRAIN
#define TM_CTX_DRAIN 8   // slices per drained segment of the drained instantiation
#endif
#ifndef TM_CTX_DRAIN_MIN_SK
#define TM_CTX_DRAIN_MIN_SK 1024  // s_k above which the drained instantiation runs
#endif
#ifndef TM_CTX_DBG_NOMMA  // timing experiments only: issue no MMAs (producer-bound time)
#define TM_CTX_DBG_NOMMA 0
#endif
#ifndef TM_CTX_DBG_NOPROD  // timing experiments only: no A split / TMEM stores
#define TM_CTX_DBG_NOPROD 0
#endif
#ifndef TM_CTX_TA_AS
#define TM_CTX_TA_AS 2
#endif
#ifndef TM_CTX_A_FIRST
#define TM_CTX_A_FIRST 1
#endif
#ifndef TM_GEMM_PERSIST
#define TM_GEMM_PERSIST 1  // undrained instantiation: one CTA per SM looping over tiles
#endif
#ifndef TM_GEMM_BALL
#define TM_GEMM_BALL 1
#endif
#ifndef TM_GEMM_ALT
#define TM_GEMM_ALT 1  // undrained instantiation: the producer halves alternate slices
#endif
template <int N, bool DRAIN, bool DV = false>
struct CtxTaCfg {
    static constexpr int kTK = TM_CTX_TA_K;             // key columns per slice
    // kG > 0: the accumulation runs in segments of kG slices into two
    // ping-pong TMEM accumulators; the producers drain each finished segment
    // into fp32 registers (round-to-nearest adds), so the tensor core's
    // truncating accumulation spans at most 3 * kTK/8 * kG products whatever
    // s_k is.  kG = 0: kSets accumulator sets in rotation.
    static constexpr int kG = DRAIN ? TM_CTX_DRAIN : 0;
    static constexpr int kSets = kG > 0 ? 2 : (N == 64 ? TM_CTX_TA_SETS : 4);
    static constexpr int kAcc = kSets * 2 * N;         // accumulator columns
    static constexpr int kAcols = 2 * 2 * kTK;         // one A stage: 2 M-blocks x (hi, lo)
    static constexpr int kASmax = (512 - kAcc) / kAcols > 4 ? 4 : (512 - kAcc) / kAcols;
    static constexpr int kAS = TM_CTX_TA_AS < kASmax ? TM_CTX_TA_AS : kASmax;
    static_assert(kAS >= 2, "TMEM columns");
    // TMEM column map: A stages first, the accumulators at the top
    static constexpr int kA0 = TM_CTX_A_FIRST ? 0 : kAcc;
    static constexpr int kAcc0 = TM_CTX_A_FIRST ? 512 - kAcc : 0;
    static constexpr int kSS = TM_CTX_TA_SS;
    static constexpr int kPbytes = kCM * kTK * 4;      // 16 / 32 KB, swizzled
    static constexpr int kVbytes = kTK * N * 4;        // V (ctx) / dO (dV) rows
    static constexpr int kMbytes = DV ? kTK * (kCM / 32) * 4 : 0;  // dV: the slice's mask words
    static constexpr int kSlice = (kPbytes + kVbytes + kMbytes + 1023) / 1024 * 1024;
    static constexpr int kBbytes = N * kTK * 4;
    static constexpr int kOpStage = 2 * kBbytes;       // B hi, lo
    static constexpr size_t kSmem = 1024 + (size_t)kAS * kOpStage + (size_t)kSS * kSlice;
    static_assert(kSmem <= 227 * 1024, "smem");
};

__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "r"(tmem_a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]),
                 "f"(v[7])
                 : "memory");
}
template <int TK>
__device__ __forceinline__ uint32_t swz_k_offset(int mn, int kchunk) {
    return TK == 32 ? sw128_k_offset(mn, kchunk) : sw64_k_offset(mn, kchunk);
}
template <int TK>
__device__ __forceinline__ uint64_t umma_desc_k(uint32_t addr) {
    return TK == 32 ? umma_desc_sw128(addr, 16, 1024) : umma_desc_sw64(addr, 512);
}

// DV = true: the same pipeline for dV = D^T dO (M = s_k, N = d, K = s_q):
// the loader stages [kTK query rows x 256 key columns] of P row-major, their
// mask words and the dO rows; a producer thread owns key column m = one TMEM
// lane and reads its kTK/2 values down the slice (a warp reads 32 consecutive
// floats of a row: conflict-free) -- the transpose happens on the way into
// TMEM.  B = dO's K-major tile, exactly as V's for ctx.
template <int N, bool DRAIN, bool DV>
__global__ void __launch_bounds__(kCThreads, 1) ctx_recompute_gemm_ta_kernel(
    const __grid_constant__ CUtensorMap tm_p, const __grid_constant__ CUtensorMap tm_v,
    const __grid_constant__ CUtensorMap tm_m, const uint32_t* __restrict__ mask, double scale,
    float* __restrict__ ctx, int s_q, int s_k, int ntiles) {
    using Cfg = CtxTaCfg<N, DRAIN, DV>;
    constexpr int kSets = Cfg::kSets, kSS = Cfg::kSS, kAS = Cfg::kAS, kG = Cfg::kG;
    constexpr int kTK = Cfg::kTK;
    constexpr int kGd = kG > 0 ? kG : 1;  // (division-safe)
    constexpr bool kAlt = TM_GEMM_ALT && kG == 0 && kTK == 32;
    grid_dep_wait();
    grid_dep_launch();
    extern __shared__ __align__(1024) unsigned char gsm[];
    const uint32_t base = (smem_u32(gsm) + 1023u) & ~1023u;
    const uint32_t stage_base = base + kAS * Cfg::kOpStage;
    unsigned char* stage_ptr = gsm + (stage_base - smem_u32(gsm));
    __shared__ uint64_t full[kAS], empty[kAS], acc_full, acc_empty, sfull[kSS], sempty[kSS];
    __shared__ uint64_t seg_full[2], seg_empty[2];  // kG > 0: segment accumulators
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Tiles = (head, 256 output rows): ctx's query rows (ragged s_q allowed)
    // / dV's key rows.  Persistent: CTA b takes tiles b, b + grid, ...; the
    // slice ring, the operand stages and their barrier phases run on across
    // tiles (slice counter gs), so the next tile's loads stream in under the
    // current tile's epilogue.  (The drained instantiation is launched with
    // one tile per CTA.)
    const int n_rows = DV ? s_k : s_q;
    const int iblocks = (n_rows + kCM - 1) / kCM;
    const int nsl = (DV ? s_q : s_k) / kTK;
    const int myn = (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    constexpr int kMMAWarp = kCSP / 32, kLoadWarp = kCSP / 32 + 1;
    constexpr int kArrive = kCSP / 32 / (kAlt ? 2 : 1);  // producer warps per slice
    // ALT: each half must own its ring slots and operand stages (even ring
    // depths) -- a half waiting on a slot the other half has not drained yet
    // would wait two phases ahead, which an mbarrier parity wait cannot tell
    // from the phase just completed (measured: kSS = 3 corrupts and faults)
    static_assert(!kAlt || (kSS % 2 == 0 && kAS % 2 == 0), "ALT needs even ring depths");

    if (threadIdx.x == 0) {
        for (int s = 0; s < kAS; ++s) {
            mbar_init(&full[s], kArrive);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kSS; ++s) {
            mbar_init(&sfull[s], 1);
            mbar_init(&sempty[s], kArrive);
        }
        mbar_init(&acc_full, 1);
        mbar_init(&acc_empty, kCSP / 32);
        for (int g = 0; g < 2; ++g) {
            mbar_init(&seg_full[g], 1);
            mbar_init(&seg_empty[g], kCSP / 32);
        }
        mbar_fence_init();
    }
    if (warp == kMMAWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&tmem_base_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp < kMMAWarp) {
        // ---------------- producers ----------------
        // A: thread t owns output row m = t % 256 of the tile (TMEM lane
        //    32*(warp%4) + lane of M-block m / 128).  ALT (the undrained
        //    instantiation): the two 8-warp halves take alternate slices
        //    (slice counter parity), a thread covering all kTK K values of
        //    its row; else both halves share every slice, half the K values
        //    each (h = t / 256).
        // B: 4 warps per half, thread tb < 128 owns V / dO column n = tb % N,
        //    K-rows kb..kb+kKV-1.
        constexpr int kGrp = kAlt ? 2 : 1;
        constexpr int kColsT = (kTK / 2) * kGrp;  // K values per thread per slice
        const int t = threadIdx.x;
        const int m = t % kCM, mb = m >> 7;
        const int grp = kAlt ? t / kCM : 0, h = kAlt ? 0 : t / kCM;
        const int tb = kAlt ? t % kCM : t;
        // B producers: 4 warps of the slice's half, or for dV (TM_GEMM_BALL)
        // all 8 (A/B: dV 289 -> 285 us, ctx 294 -> 296: ctx keeps 4)
        constexpr int kBThreads = (TM_GEMM_BALL && kAlt && DV) ? kCM : 128;
        const bool bwarp = tb < kBThreads;
        constexpr int kKV = kTK * N / kBThreads;  // V / dO values per B thread
        const int bn = tb % N, kb = (tb / N) * kKV;
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        constexpr int kSlPerWord = 32 / kTK;  // slices per mask word (2 or 1)
        static_assert(!kAlt || kSlPerWord == 1, "alternating halves need a mask word per slice");
        const int quad = warp % 4, emb = (warp / 4) % 2, half = warp / 8;
        const uint32_t acc_lane = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(Cfg::kAcc0 + emb * N + half * (N / 2));
        const float sc = (float)scale;
        float racc[N / 2];
        auto drain = [&](int j) {  // segment j: wait for its MMAs, add, free the buffer
            mbar_wait(&seg_full[j & 1], (uint32_t)((j >> 1) & 1));
            tc_fence_after();
#pragma unroll
            for (int c0 = 0; c0 < N / 2; c0 += 16) {
                float v[16];
                tmem_ld16(acc_lane + (uint32_t)((j & 1) * 2 * N + c0), v);
#pragma unroll
                for (int i = 0; i < 16; ++i) racc[c0 + i] += v[i];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&seg_empty[j & 1]);
        };
        for (int k = 0; k < myn; ++k) {
            const int tile = (int)blockIdx.x + k * (int)gridDim.x;
            const int64_t head = tile / iblocks;
            const int i0 = (tile % iblocks) * kCM;
            const int64_t gs0 = (int64_t)k * nsl;
            const bool row_in = !DV && i0 + m < s_q;
            const uint32_t* mrow = mask + (((head * (int64_t)s_q + i0 + m) * s_k) >> 5);
            // this thread's first slice of the tile (ALT: slice-counter parity)
            const int sl0 = kAlt ? (int)((grp + gs0) & 1) : 0;
            uint32_t w = 0, w_next = (row_in && sl0 < nsl) ? __ldg(mrow + sl0 / kSlPerWord) : 0u;
#pragma unroll
            for (int i = 0; i < N / 2; ++i) racc[i] = 0.0f;
            constexpr int kLag = 2;  // drain segment j while producing slice (j+1)*kG + kLag
            int drained = 0;
            for (int sl = sl0; sl < nsl; sl += kGrp) {
                const int64_t gs = gs0 + sl;
                const int ss = (int)(gs % kSS), s = (int)(gs % kAS);
                if (kG > 0 && sl >= kG + kLag && (sl - kLag) % kGd == 0) drain(drained++);
                if (!DV && sl % kSlPerWord == 0) {
                    w = w_next;
                    const int nx = sl / kSlPerWord + kGrp;  // this thread's next mask word
                    if (row_in && nx * kSlPerWord < nsl) w_next = __ldg(mrow + nx);
                }
                mbar_wait(&sfull[ss], (uint32_t)((gs / kSS) & 1));
                const uint32_t sp = stage_base + ss * Cfg::kSlice;
                float e[kColsT];
                uint32_t dvw[DV ? kColsT : 1];
                if (!DV) {
#pragma unroll
                    for (int c = 0; c < kColsT / 4; ++c)
                        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                                     : "=f"(e[4 * c]), "=f"(e[4 * c + 1]), "=f"(e[4 * c + 2]), "=f"(e[4 * c + 3])
                                     : "r"(sp + swz_k_offset<kTK>(m, (kColsT / 4) * h + c)));
                } else {
                    // query rows h*kColsT + k of key column m, and their mask words
#pragma unroll
                    for (int q = 0; q < kColsT; ++q) {
                        const int r = h * kColsT + q;
                        e[q] = lds32(sp + (uint32_t)((r * kCM + m) * 4));
                        dvw[q % (DV ? kColsT : 1)] =
                            ldsu32(sp + Cfg::kPbytes + Cfg::kVbytes + (uint32_t)((r * (kCM / 32) + (m >> 5)) * 4));
                    }
                }
                float ov[kKV];
                if (bwarp) {
#pragma unroll
                    for (int q = 0; q < kKV; ++q)
                        ov[q] = lds32(sp + Cfg::kPbytes + (uint32_t)(((kb + q) * N + bn) * 4));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sempty[ss]);
                if (gs >= kAS) mbar_wait(&empty[s], (uint32_t)(((gs / kAS) + 1) & 1));
                tc_fence_after();
                // this thread's keep bits: columns kTK*sl + h*kColsT ..
                const uint32_t wsl = w >> (kTK * (sl % kSlPerWord) + kColsT * h);
                const uint32_t ta = lane_base + (uint32_t)(Cfg::kA0 + s * Cfg::kAcols + mb * 2 * kTK + kColsT * h);
#pragma unroll
                for (int q = 0; q < (TM_CTX_DBG_NOPROD ? 0 : kColsT / 16); ++q) {  // 16 values: hi, lo -> TMEM
                    float hi[16], lo[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) {
                        const int kk = 16 * q + u;
                        const bool keep = DV ? ((dvw[kk % (DV ? kColsT : 1)] >> lane) & 1u) : ((wsl >> kk) & 1u);
                        split_tf32(keep ? e[kk] : 0.0f, hi[u], lo[u]);
                    }
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        tmem_st8(ta + 16 * q + 8 * c, hi + 8 * c);
                        tmem_st8(ta + kTK + 16 * q + 8 * c, lo + 8 * c);
                    }
                }
                if (bwarp) {
                    const uint32_t b_hi = base + s * Cfg::kOpStage, b_lo = b_hi + Cfg::kBbytes;
                    float bh[kKV], bl[kKV];
#pragma unroll
                    for (int u = 0; u < kKV; ++u) split_tf32(ov[u], bh[u], bl[u]);
#pragma unroll
                    for (int c = 0; c < kKV / 4; ++c) {
                        const uint32_t off = swz_k_offset<kTK>(bn, (kb >> 2) + c);
                        sts128(b_hi + off, bh[4 * c], bh[4 * c + 1], bh[4 * c + 2], bh[4 * c + 3]);
                        sts128(b_lo + off, bl[4 * c], bl[4 * c + 1], bl[4 * c + 2], bl[4 * c + 3]);
                    }
                    fence_proxy_async_smem();
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
            // ---------------- epilogue: out = (1/(1-p)) * the accumulation ----
            const int row = i0 + emb * 128 + quad * 32 + lane;
            float* out = ctx + (head * (int64_t)n_rows + row) * N;
            const bool store = row < n_rows;
            if (kG > 0) {  // (one tile per CTA)
                const int nseg = (nsl + kGd - 1) / kGd;
                while (drained < nseg) drain(drained++);
                if (store) {
#pragma unroll
                    for (int i = 0; i < N / 2; i += 4)
                        st_stream(reinterpret_cast<float4*>(out + half * (N / 2) + i),
                                  make_float4(racc[i] * sc, racc[i + 1] * sc, racc[i + 2] * sc,
                                              racc[i + 3] * sc));
                }
            } else {
                mbar_wait(&acc_full, (uint32_t)(k & 1));
                tc_fence_after();
                // all of this thread's sums into registers first, then free
                // the accumulators (the MMA lane starts the next tile) and
                // store while it runs
                float* v = racc;  // N/2 columns
#pragma unroll
                for (int c0 = 0; c0 < N / 2; c0 += 16) {
                    float w16[16];
                    const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) +
                                        (uint32_t)(Cfg::kAcc0 + emb * N + half * (N / 2) + c0);
                    tmem_ld16(ta, w16);
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[c0 + i] = w16[i];
#pragma unroll
                    for (int set = 1; set < kSets; ++set) {
                        tmem_ld16(ta + (uint32_t)(set * 2 * N), w16);
#pragma unroll
                        for (int i = 0; i < 16; ++i) v[c0 + i] += w16[i];
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty);
                if (store) {
#pragma unroll
                    for (int i = 0; i < N / 2; i += 4)
                        st_stream(reinterpret_cast<float4*>(out + half * (N / 2) + i),
                                  make_float4(v[i] * sc, v[i + 1] * sc, v[i + 2] * sc, v[i + 3] * sc));
                }
            }
        }
    } else if (warp == kMMAWarp && lane == 0) {
        // ---------------- MMA issuer: A from TMEM, B from smem ----------
        constexpr uint32_t idesc = idesc_tf32_k(128, N);
        for (int k = 0; k < myn; ++k) {
            if (kG == 0 && k > 0) {  // the producers have read the previous tile's sums
                mbar_wait(&acc_empty, (uint32_t)((k - 1) & 1));
                tc_fence_after();
            }
            for (int sl = 0; sl < nsl; ++sl) {
                const int64_t gs = (int64_t)k * nsl + sl;
                const int s = (int)(gs % kAS);
                const int seg = sl / kGd;
                const bool seg_first = kG > 0 && sl % kGd == 0;
                if (seg_first && seg >= 2) {  // the producers drained segment seg - 2
                    mbar_wait(&seg_empty[seg & 1], (uint32_t)(((seg >> 1) + 1) & 1));
                }
                mbar_wait(&full[s], (uint32_t)((gs / kAS) & 1));
                tc_fence_after();
                const uint32_t b_hi = base + s * Cfg::kOpStage, b_lo = b_hi + Cfg::kBbytes;
#pragma unroll
                for (int kk = 0; kk < kTK / 8; ++kk) {  // K = 8 per MMA: +32 bytes along the rows
                    const uint64_t bh = umma_desc_k<kTK>(b_hi + kk * 32);
                    const uint64_t bl = umma_desc_k<kTK>(b_lo + kk * 32);
                    const int gk = sl * (kTK / 8) + kk;
                    const int set = kG > 0 ? (seg & 1) : gk % kSets;
                    const bool fresh = kG > 0 ? (seg_first && kk == 0) : (gk < kSets);
#pragma unroll
                    for (int mbk = 0; mbk < 2; ++mbk) {
                        const uint32_t ah = tmem + (uint32_t)(Cfg::kA0 + s * Cfg::kAcols + mbk * 2 * kTK + kk * 8);
                        const uint32_t acc = tmem + (uint32_t)(Cfg::kAcc0 + set * 2 * N + mbk * N);
#if !TM_CTX_DBG_NOMMA
                        mma_tf32_ta(acc, ah + kTK, bh, idesc, !fresh);  // small terms first
                        mma_tf32_ta(acc, ah, bl, idesc, 1);
                        mma_tf32_ta(acc, ah, bh, idesc, 1);
#else
                        (void)acc; (void)ah; (void)bh; (void)bl; (void)fresh;
#endif
                    }
                }
                mma_commit(&empty[s]);
                if (kG > 0 && (sl % kGd == kGd - 1 || sl == nsl - 1)) mma_commit(&seg_full[seg & 1]);
            }
            mma_commit(&acc_full);
        }
    } else if (warp == kLoadWarp && lane == 0) {
        // ---------------- loader: the P tile and the V / dO rows -------------
        for (int k = 0; k < myn; ++k) {
            const int tile = (int)blockIdx.x + k * (int)gridDim.x;
            const int64_t head = tile / iblocks;
            const int i0 = (tile % iblocks) * kCM;
            const int y_p = (int)(head * s_q + i0), y_v0 = (int)(head * s_k);
            for (int sl = 0; sl < nsl; ++sl) {
                const int64_t gs = (int64_t)k * nsl + sl;
                const int ss = (int)(gs % kSS);
                if (gs >= kSS) mbar_wait(&sempty[ss], (uint32_t)(((gs / kSS) + 1) & 1));
                unsigned char* sp = stage_ptr + ss * Cfg::kSlice;
                mbar_expect_tx(&sfull[ss], Cfg::kPbytes + Cfg::kVbytes + Cfg::kMbytes);
                if (!DV) {
                    tma_load_2d(sp, &tm_p, sl * kTK, y_p, &sfull[ss]);
                    tma_load_2d(sp + Cfg::kPbytes, &tm_v, 0, y_v0 + sl * kTK, &sfull[ss]);
                } else {  // P rows [kTK x 256], dO rows [kTK x N], mask words [kTK x 8]
                    const int y = (int)(head * s_q) + sl * kTK;
                    tma_load_2d(sp, &tm_p, i0, y, &sfull[ss]);
                    tma_load_2d(sp + Cfg::kPbytes, &tm_v, 0, y, &sfull[ss]);
                    tma_load_2d(sp + Cfg::kPbytes + Cfg::kVbytes, &tm_m, i0 / 32, y, &sfull[ss]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == kMMAWarp) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem)
                     : "memory");
    }
}

template <int N>
cudaError_t launch_ctx(const float* P, const uint32_t* mask, double scale, const float* V,
                       float* ctx, int64_t heads, int64_t s_q, int64_t s_k, cudaStream_t st) {
    CUtensorMap tp, tv;
    constexpr int tk = TM_CTX_TA ? CtxTaCfg<N, false>::kTK : kCK;
    if (!make_tmap_2d(&tp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, P, (uint64_t)(heads * s_q),
                      (uint64_t)s_k, kCM, tk,
                      tk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_tmap_2d(&tv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, V, (uint64_t)(heads * s_k),
                      (uint64_t)N, tk, N))
        return cudaErrorNotSupported;
    // long rows: the drained accumulation (bounded truncation error); up to
    // TM_CTX_DRAIN_MIN_SK the set rotation, ~10 % faster (see CtxTaCfg)
    const bool drain = s_k > TM_CTX_DRAIN_MIN_SK;
    const int64_t grid = heads * ((s_q + kCM - 1) / kCM);
    if (!TM_CTX_TA) {
        auto k = ctx_recompute_gemm_kernel<N>;
        const size_t smem = CtxCfg<N>::kSmem;
        (void)grid_for((const void*)k, kCThreads, smem, 1);
        launch(k, (int)grid, kCThreads, smem, st)(tp, tv, mask, scale, ctx, (int)s_q, (int)s_k);
        return cudaGetLastError();
    }
    auto k = drain ? ctx_recompute_gemm_ta_kernel<N, true, false>
                   : ctx_recompute_gemm_ta_kernel<N, false, false>;
    const size_t smem = drain ? CtxTaCfg<N, true>::kSmem : CtxTaCfg<N, false>::kSmem;
    // persistent (one CTA per SM) unless drained (one tile per CTA)
    const int g = drain || !TM_GEMM_PERSIST ? (int)grid : grid_for((const void*)k, kCThreads, smem, grid);
    (void)grid_for((const void*)k, kCThreads, smem, 1);
    launch(k, g, kCThreads, smem, st)(tp, tv, tv, mask, scale, ctx, (int)s_q, (int)s_k, (int)grid);
    return cudaGetLastError();
}

// dV = D^T dO through the TMEM-A pipeline (DV instantiation above)
#ifndef TM_DV_TA
#define TM_DV_TA 1
#endif
template <int N>
cudaError_t launch_dv_ta(const float* P, const uint32_t* mask, double scale, const float* dO,
                         float* dV, int64_t heads, int64_t s_q, int64_t s_k, cudaStream_t st) {
    constexpr int tk = CtxTaCfg<N, false, true>::kTK;
    CUtensorMap tp, tmk, to;
    const uint64_t rows = (uint64_t)(heads * s_q);
    if (!make_tmap_2d(&tp, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, P, rows, (uint64_t)s_k, tk, kCM) ||
        !make_tmap_2d(&tmk, CU_TENSOR_MAP_DATA_TYPE_UINT32, mask, rows, (uint64_t)(s_k / 32), tk,
                      kCM / 32) ||
        !make_tmap_2d(&to, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dO, rows, (uint64_t)N, tk, N))
        return launch_dv<N>(P, mask, scale, dO, dV, heads, s_q, s_k, st);  // no tensor maps
    const bool drain = s_q > TM_CTX_DRAIN_MIN_SK;
    auto k = drain ? ctx_recompute_gemm_ta_kernel<N, true, true>
                   : ctx_recompute_gemm_ta_kernel<N, false, true>;
    const size_t smem = drain ? CtxTaCfg<N, true, true>::kSmem : CtxTaCfg<N, false, true>::kSmem;
    const int64_t grid = heads * (s_k / kCM);
    const int g = drain || !TM_GEMM_PERSIST ? (int)grid : grid_for((const void*)k, kCThreads, smem, grid);
    (void)grid_for((const void*)k, kCThreads, smem, 1);
    launch(k, g, kCThreads, smem, st)(tp, to, tmk, mask, scale, dV, (int)s_q, (int)s_k, (int)grid);
    return cudaGetLastError();
}

}  // namespace

bool ctx_gemm_supported(int64_t s_q, int64_t s_k, int64_t d) {
    return s_q > 0 && s_k > 0 && s_k % 32 == 0 && (d == 32 || d == 64) &&
           s_q <= (1 << 20) && s_k <= (1 << 20);
}

cudaError_t launch_ctx_recompute_gemm(const float* P, const uint32_t* mask, double scale,
                                      const float* V, float* ctx, int64_t heads, int64_t s_q,
                                      int64_t s_k, int64_t d, cudaStream_t st) {
    if (heads == 0) return cudaSuccess;
    switch (d) {
        case 32: return launch_ctx<32>(P, mask, scale, V, ctx, heads, s_q, s_k, st);
        case 64: return launch_ctx<64>(P, mask, scale, V, ctx, heads, s_q, s_k, st);
        default: return cudaErrorInvalidValue;
    }
}

bool dv_gemm_supported(int64_t s_q, int64_t s_k, int64_t d) {
    return s_q > 0 && s_k > 0 && s_q % kBK == 0 && s_k % kBM == 0 && (d == 32 || d == 64 || d == 128) &&
           s_q <= (1 << 20) && s_k <= (1 << 20);
}

cudaError_t launch_dv_recompute_gemm(const float* P, const uint32_t* mask, double scale,
                                     const float* dO, float* dV, int64_t heads, int64_t s_q,
                                     int64_t s_k, int64_t d, cudaStream_t st) {
    if (heads == 0) return cudaSuccess;
    switch (d) {
#ifndef TM_DV_STAGED
#define TM_DV_STAGED 1
#endif
        case 32: return TM_DV_TA ? launch_dv_ta<32>(P, mask, scale, dO, dV, heads, s_q, s_k, st)
                      : TM_DV_STAGED ? launch_dv_staged<32>(P, mask, scale, dO, dV, heads, s_q, s_k, st)
                                     : launch_dv<32>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        case 64: return TM_DV_TA ? launch_dv_ta<64>(P, mask, scale, dO, dV, heads, s_q, s_k, st)
                      : TM_DV_STAGED ? launch_dv_staged<64>(P, mask, scale, dO, dV, heads, s_q, s_k, st)
                                     : launch_dv<64>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        case 128: return launch_dv<128>(P, mask, scale, dO, dV, heads, s_q, s_k, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tb
