// mt19937_kernels.cu -- the reference's mask stream on the device.
//
// BoolMask::bernoulli_keep(shape, p, seed) (tensor.cpp:186-203) draws ONE
// sequential std::mt19937_64 stream per mask: element i is kept iff
// double(x_i) * 2^-64 >= p (uniform_real_distribution<double> over
// generate_canonical with a 64-bit engine), x_i the i-th tempered output.
// Reproducing it bit for bit in parallel (mt_jump.cpp has the math):
//
//   1. the stream is cut into chunks of kMtChunk = 2^18 outputs; chunk k's
//      starting state is T^(k * 2^18) s0, reached through base-32 digits of k
//      (levels 3..0): a jump by digit d at level l applies the polynomial
//      x^(d * 32^l * 2^18) mod P to a state;
//   2. mt_base_kernel: the 20248-word sequence started at each source state
//      (the recurrence, 128 words per step, ring buffer in smem);
//   3. mt_jump_kernel: a jumped state = XOR of the 312-word windows of that
//      sequence at the set bits of the polynomial (sequence in smem, one CTA
//      per (source, digit), thread j owns state word j);
//   4. mt_keep_kernel: one CTA per chunk runs the recurrence from its state
//      (128 outputs per step), tempers, compares with the integer threshold
//      and writes the keep bits with one ballot per 32 outputs (the packed
//      BoolMask order).
//
// The output of each step equals std::mt19937_64 after discard(offset) --
// the GPU tests check it against the host engine; nothing here depends on
// the device's float arithmetic (integer only).
#include <mutex>
#include <vector>

#include "common.cuh"
#include "mt19937.h"
#include "tempo_internal.h"

namespace tb {
namespace {

constexpr int kGenThreads = 128;  // outputs per recurrence step (<= 156)
constexpr int kRing = 512;        // ring buffer words (>= 312 + 128, power of two)
constexpr int kJumpThreads = 320;

// Sequence w_0 .. w_{kMtBaseWords-1} from each source state.
__global__ void __launch_bounds__(kGenThreads) mt_base_kernel(const uint64_t* __restrict__ src,
                                                              uint64_t* __restrict__ base) {
    __shared__ uint64_t ring[kRing];
    const uint64_t* st = src + (size_t)blockIdx.x * kMtN;
    uint64_t* out = base + (size_t)blockIdx.x * kMtBaseWords;
    for (int i = threadIdx.x; i < (int)kMtN; i += kGenThreads) {
        const uint64_t v = st[i];
        ring[i] = v;
        out[i] = v;
    }
    __syncthreads();
    for (int j0 = kMtN; j0 < kMtBaseWords; j0 += kGenThreads) {
        const int j = j0 + threadIdx.x;
        if (j < kMtBaseWords) {
            const uint64_t w = mt_next_word(ring[(j - 312) & (kRing - 1)],
                                            ring[(j - 311) & (kRing - 1)],
                                            ring[(j - 156) & (kRing - 1)]);
            ring[j & (kRing - 1)] = w;
            out[j] = w;
        }
        __syncthreads();
    }
}

// Children states: child c = child0 + s * 32 + d (d = 0: the source itself),
// stored at out[(c - child_lo) * 312] for c in [child_lo, child_hi].  The
// 312 polynomial words are split over kJumpParts CTAs (grid.x); each stages
// only the slice of the sequence its words touch in smem, accumulates the
// windows of its set bits (64 predicated loads per word, no serial bit
// scan) and XORs its partial state into the zeroed output.
constexpr int kJumpParts = 8;
constexpr int kJumpWordsPerPart = (kMtPolyWords + kJumpParts - 1) / kJumpParts;
constexpr int kJumpSlice = 64 * kJumpWordsPerPart + kMtN;  // staged words per CTA

__global__ void __launch_bounds__(kJumpThreads) mt_jump_kernel(const uint64_t* __restrict__ base,
                                                               const uint64_t* __restrict__ polys,
                                                               uint64_t* __restrict__ out,
                                                               int64_t child0, int64_t child_lo,
                                                               int64_t child_hi) {
    __shared__ uint64_t slice[kJumpSlice];
    const int part = blockIdx.x, d = blockIdx.y, s = blockIdx.z;
    const int64_t child = child0 + (int64_t)s * 32 + d;
    if (child < child_lo || child > child_hi) return;  // not needed
    const uint64_t* b = base + (size_t)s * kMtBaseWords;
    uint64_t* o = out + (size_t)(child - child_lo) * kMtN;
    const int j = threadIdx.x;
    if (d == 0) {
        if (part == 0 && j < (int)kMtN) atomicXor((unsigned long long*)(o + j), b[j]);
        return;
    }
    const int w0 = part * kJumpWordsPerPart;
    const int w1 = min(kMtPolyWords, w0 + kJumpWordsPerPart);
    if (w0 >= w1) return;
    const int lo = 64 * w0, hi = min(kMtBaseWords, 64 * w1 + (int)kMtN);
    for (int i = lo + j; i < hi; i += kJumpThreads) slice[i - lo] = b[i];
    __syncthreads();
    if (j >= (int)kMtN) return;
    const uint64_t* g = polys + (size_t)(d - 1) * kMtPolyWords;
    uint64_t acc = 0;
    for (int w = w0; w < w1; ++w) {
        const uint64_t bits = __ldg(g + w);  // uniform over the CTA
        const uint64_t* sb = slice + 64 * (w - w0) + j;
        const uint32_t blo = (uint32_t)bits, bhi = (uint32_t)(bits >> 32);
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if ((blo >> t) & 1u) acc ^= sb[t];
#pragma unroll
        for (int t = 0; t < 32; ++t)
            if ((bhi >> t) & 1u) acc ^= sb[32 + t];
    }
    atomicXor((unsigned long long*)(o + j), acc);
}

// Keep bits of elements [e_begin, e_end) of the stream; chunk k = k0 + blockIdx.x.
__global__ void __launch_bounds__(kGenThreads) mt_keep_kernel(const uint64_t* __restrict__ states,
                                                              int64_t k0, uint64_t e_begin,
                                                              uint64_t e_end, uint64_t xmin,
                                                              uint32_t* __restrict__ mask) {
    __shared__ uint64_t ring[kRing];
    const int64_t k = k0 + blockIdx.x;
    const uint64_t* st = states + (size_t)blockIdx.x * kMtN;
    for (int i = threadIdx.x; i < (int)kMtN; i += kGenThreads) ring[i] = st[i];
    __syncthreads();
    const uint64_t c0 = (uint64_t)k * (uint64_t)kMtChunk;  // global index of the chunk's output 0
    const uint64_t stop = min(c0 + (uint64_t)kMtChunk, e_end);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t t0 = c0; t0 < stop; t0 += kGenThreads) {
        const int j = (int)(t0 - c0) + kMtN + threadIdx.x;  // sequence index of this output
        const uint64_t w = mt_next_word(ring[(j - 312) & (kRing - 1)],
                                        ring[(j - 311) & (kRing - 1)],
                                        ring[(j - 156) & (kRing - 1)]);
        ring[j & (kRing - 1)] = w;
        const bool keep = mt_temper(w) >= xmin;
        uint32_t word = __ballot_sync(kFull, keep);
        const uint64_t e0 = t0 + 32 * warp;  // element of bit 0 of this warp's word
        if (lane == 0 && e0 >= e_begin && e0 < e_end) {
            if (e_end - e0 < 32) word &= (1u << (e_end - e0)) - 1u;
            mask[(e0 - e_begin) >> 5] = word;
        }
        __syncthreads();
    }
}

// std::mersenne_twister_engine::seed on the device (one thread, 312 steps).
__global__ void mt_seed_kernel(uint64_t seed, uint64_t* __restrict__ st) {
    if (threadIdx.x != 0) return;
    uint64_t v = seed;
    st[0] = v;
    for (uint64_t i = 1; i < kMtN; ++i) {
        v = 6364136223846793005ull * (v ^ (v >> 62)) + i;
        st[i] = v;
    }
}

struct DevPolys {
    std::mutex mu;
    std::vector<uint64_t*> ptr;  // per device
};
DevPolys& dev_polys() {
    static DevPolys d;
    return d;
}

const uint64_t* device_polys(cudaError_t& err) {
    const uint64_t* host = mt_jump_polys();
    if (!host) {
        err = cudaErrorUnknown;
        return nullptr;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    DevPolys& D = dev_polys();
    std::lock_guard<std::mutex> lock(D.mu);
    if ((int)D.ptr.size() <= dev) D.ptr.resize(dev + 1, nullptr);
    if (!D.ptr[dev]) {
        const size_t bytes = (size_t)kMtLevels * 31 * kMtPolyWords * sizeof(uint64_t);
        uint64_t* p = nullptr;
        err = cudaMalloc(&p, bytes);
        if (err != cudaSuccess) return nullptr;
        err = cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice);
        if (err != cudaSuccess) {
            cudaFree(p);
            return nullptr;
        }
        D.ptr[dev] = p;
    }
    err = cudaSuccess;
    return D.ptr[dev];
}

// Workspace layout (bytes, 256-aligned pieces): seed state, two state
// buffers of up to (ceil(K/32) + 1) * 32 states, base sequences of up to
// ceil(K/32) + 1 sources.
struct MtWs {
    size_t seed_off, sa_off, sb_off, base_off, total;
};
MtWs mt_ws_layout(uint64_t e_begin, int64_t n) {
    const int64_t k0 = (int64_t)(e_begin / kMtChunk);
    const int64_t k1 = (int64_t)((e_begin + (uint64_t)n - 1) / kMtChunk);
    const int64_t groups = (k1 >> 5) - (k0 >> 5) + 1;  // level-1 prefixes
    const size_t st = kMtN * sizeof(uint64_t);
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    MtWs L;
    L.seed_off = 0;
    L.sa_off = al(st);
    const size_t states = (size_t)(groups + 1) * 32 * st;
    L.sb_off = L.sa_off + al(states);
    L.base_off = L.sb_off + al(states);
    L.total = L.base_off + al((size_t)(groups + 1) * kMtBaseWords * sizeof(uint64_t));
    return L;
}

}  // namespace

size_t mt_keep_workspace(uint64_t e_begin, int64_t n) {
    if (n <= 0) return 0;
    return mt_ws_layout(e_begin, n).total;
}

cudaError_t launch_mt_keep_bits(uint64_t seed, double p, uint64_t e_begin, int64_t n,
                                uint32_t* mask, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const MtWs L = mt_ws_layout(e_begin, n);
    if (ws_bytes < L.total || (e_begin & 31u)) return cudaErrorInvalidValue;
    cudaError_t err = cudaSuccess;
    const uint64_t* polys = device_polys(err);
    if (!polys) return err;
    char* w = static_cast<char*>(ws);
    uint64_t* seed_st = reinterpret_cast<uint64_t*>(w + L.seed_off);
    uint64_t* sa = reinterpret_cast<uint64_t*>(w + L.sa_off);
    uint64_t* sb = reinterpret_cast<uint64_t*>(w + L.sb_off);
    uint64_t* base = reinterpret_cast<uint64_t*>(w + L.base_off);

    mt_seed_kernel<<<1, 32, 0, st>>>(seed, seed_st);

    const int64_t k0 = (int64_t)(e_begin / kMtChunk);
    const int64_t k1 = (int64_t)((e_begin + (uint64_t)n - 1) / kMtChunk);
    if ((k1 >> (5 * kMtLevels)) != 0) return cudaErrorInvalidValue;  // > 2^38 outputs

    // level states: prefixes [lo, hi] of k >> (5 * level), stored from `cur`
    const uint64_t* cur = seed_st;
    int64_t lo = 0, hi = 0;  // level kMtLevels: the single prefix 0
    uint64_t* bufs[2] = {sa, sb};
    int flip = 0;
    for (int l = kMtLevels - 1; l >= 0; --l) {
        const int64_t clo = k0 >> (5 * l), chi = k1 >> (5 * l);  // needed children
        const int64_t S = hi - lo + 1;                             // sources
        uint64_t* nxt = bufs[flip];
        flip ^= 1;
        const bool all_zero_digit = (clo == chi) && ((clo & 31) == 0);
        if (all_zero_digit) {  // child = source (digit 0): carry the state over
            err = cudaMemcpyAsync(nxt, cur + (size_t)(clo / 32 - lo) * kMtN,
                                  kMtN * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st);
            if (err != cudaSuccess) return err;
        } else {
            mt_base_kernel<<<(unsigned)S, kGenThreads, 0, st>>>(cur, base);
            err = cudaMemsetAsync(nxt, 0, (size_t)(chi - clo + 1) * kMtN * sizeof(uint64_t), st);
            if (err != cudaSuccess) return err;
            dim3 grid(kJumpParts, 32, (unsigned)S);
            mt_jump_kernel<<<grid, kJumpThreads, 0, st>>>(
                base, polys + (size_t)l * 31 * kMtPolyWords, nxt, lo * 32, clo, chi);
            err = cudaGetLastError();
            if (err != cudaSuccess) return err;
        }
        cur = nxt;
        lo = clo;
        hi = chi;
    }
    const uint64_t xmin = mt_keep_threshold(p);
    mt_keep_kernel<<<(unsigned)(k1 - k0 + 1), kGenThreads, 0, st>>>(cur, k0, e_begin,
                                                                   e_begin + (uint64_t)n, xmin,
                                                                   mask);
    return cudaGetLastError();
}

}  // namespace tb
