// mt19937_kernels.cu -- the reference's mask stream on the device.
//
// BoolMask::bernoulli_keep(shape, p, seed) (tensor.cpp:186-203) draws ONE
// sequential std::mt19937_64 stream per mask: element i is kept iff
// double(x_i) * 2^-64 >= p (uniform_real_distribution<double> over
// generate_canonical with a 64-bit engine), x_i the i-th tempered output.
// Reproducing it bit for bit in parallel (mt_jump.cpp has the math):
//
//   1. the stream is cut into chunks of kMtChunk = 2^19 outputs; chunk k's
//      starting state is T^(k * 2^19) s0, reached through base-32 digits of k
//      (levels 3..0): a jump by digit d at level l applies the polynomial
//      x^(d * 32^l * 2^19) mod P to a state;
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
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
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
// 312 polynomial words are split over kMtJumpParts CTAs (grid.x); each
// stages only the slice of the sequence its words touch (plus a zero tail
// for the list padding) in smem and walks the part's precomputed list of
// set-bit indices, four per uniform 64-bit load: per set bit one LDS and
// half a 3-input XOR; the partial state is XORed into the zeroed output.
constexpr int kJumpSlice = 64 * kMtJumpWords + 2 * (int)kMtN;  // words staged per CTA

__global__ void __launch_bounds__(kJumpThreads) mt_jump_kernel(
    const uint64_t* __restrict__ base, const uint16_t* __restrict__ idx,
    const int32_t* __restrict__ off, int poly0, uint64_t* __restrict__ out, int64_t child0,
    int64_t child_lo, int64_t child_hi) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
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
    const int g0 = 64 * part * kMtJumpWords;  // first sequence word of the slice
    const int real = 64 * kMtJumpWords + (int)kMtN;
    for (int i = j; i < kJumpSlice; i += kJumpThreads)
        slice[i] = (i < real && g0 + i < kMtBaseWords) ? b[g0 + i] : 0ull;
    __syncthreads();
    if (j >= (int)kMtN) return;
    const int pi = (poly0 + d - 1) * kMtJumpParts + part;
    const int k0 = __ldg(off + pi), k1 = __ldg(off + pi + 1);
    const uint64_t* L = reinterpret_cast<const uint64_t*>(idx + k0);
    const uint64_t* sj = slice + j;
    uint64_t acc = 0;
#pragma unroll 4
    for (int k = 0; k < (k1 - k0) >> 2; ++k) {
        const uint64_t q = __ldg(L + k);  // four indices, uniform over the CTA
        acc ^= sj[q & 0xffff] ^ sj[(q >> 16) & 0xffff] ^ sj[(q >> 32) & 0xffff] ^ sj[q >> 48];
    }
    atomicXor((unsigned long long*)(o + j), acc);
}

// Keep bits of elements [e_begin, e_end); chunk k = k0 + blockIdx.x.  Step t
// of a chunk produces outputs 128 t .. 128 t + 127 (all independent: the
// recurrence reaches back >= 156 words); warp w's ballot is the mask word of
// outputs 128 t + 32 w .. + 31.  Steps before the requested range only
// advance the recurrence (shard offsets that fall inside a chunk).
__global__ void __launch_bounds__(kGenThreads) mt_keep_kernel(const uint64_t* __restrict__ states,
                                                              int64_t k0, uint64_t e_begin,
                                                              uint64_t e_end, uint64_t xmin,
                                                              uint32_t* __restrict__ mask) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    __shared__ uint64_t ring[kRing];
    const int64_t k = k0 + blockIdx.x;
    const uint64_t* st = states + (size_t)blockIdx.x * kMtN;
    for (int i = threadIdx.x; i < (int)kMtN; i += kGenThreads) ring[i] = st[i];
    const uint64_t c0 = (uint64_t)k * (uint64_t)kMtChunk;  // global index of the chunk's output 0
    // chunk-relative output range [r0, r1) to store (r0 % 32 == 0)
    const uint32_t r0 = e_begin > c0 ? (uint32_t)(e_begin - c0) : 0u;
    const uint32_t r1 = (uint32_t)(min(c0 + (uint64_t)kMtChunk, e_end) - c0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* mrow = mask + ((c0 + r0 - e_begin) >> 5) - (r0 >> 5);  // word of chunk output 0
    // ring slots of this thread's operands, per phase of the 4-step (512-word)
    // cycle: loop-invariant, so a step costs no address arithmetic
    const int tid = threadIdx.x;
    int a312[4], a311[4], a156[4], aw[4];
#pragma unroll
    for (int ph = 0; ph < 4; ++ph) {
        const int j = ph * kGenThreads + kMtN + tid;  // sequence index mod 512
        a312[ph] = (j - 312) & (kRing - 1);
        a311[ph] = (j - 311) & (kRing - 1);
        a156[ph] = (j - 156) & (kRing - 1);
        aw[ph] = j & (kRing - 1);
    }
    __syncthreads();
    // batches of 32 steps: lane s keeps the ballot word of step s and the
    // warp stores its 32 words at once (words 4 t + w of the chunk)
    for (uint32_t tb = 0; tb < r1; tb += 32 * kGenThreads) {
        uint32_t mine = 0;
#pragma unroll 1
        for (int s4 = 0; s4 < 32; s4 += 4) {
#pragma unroll
            for (int ph = 0; ph < 4; ++ph) {
                const uint32_t t0 = tb + (s4 + ph) * kGenThreads;
                if (t0 < r1) {  // uniform
                    const uint64_t w = mt_next_word(ring[a312[ph]], ring[a311[ph]], ring[a156[ph]]);
                    ring[aw[ph]] = w;
                    __syncthreads();  // w is visible: the next step's loads overlap the tempering
                    const uint32_t word = __ballot_sync(kFull, mt_keep(w, xmin));
                    if (lane == s4 + ph) mine = word;
                }
            }
        }
        const uint32_t e = tb + lane * kGenThreads + 32 * warp;  // output of bit 0 of `mine`
        if (e >= r0 && e < r1) {
            if (r1 - e < 32) mine &= (1u << (r1 - e)) - 1u;  // ragged end
            mrow[e >> 5] = mine;
        }
    }
}

// std::mersenne_twister_engine::seed on the device (one thread, 312 steps).
__global__ void mt_seed_kernel(uint64_t seed, uint64_t* __restrict__ st) {
    grid_dep_wait();  // PDL: predecessor complete and visible
    grid_dep_launch();
    if (threadIdx.x != 0) return;
    uint64_t v = seed;
    st[0] = v;
    for (uint64_t i = 1; i < kMtN; ++i) {
        v = 6364136223846793005ull * (v ^ (v >> 62)) + i;
        st[i] = v;
    }
}

struct DevTables {
    std::mutex mu;
    std::vector<uint16_t*> idx;  // per device
    std::vector<int32_t*> off;
};
DevTables& dev_tables() {
    static DevTables d;
    return d;
}

// The jump index lists on this device (uploaded once per device).
cudaError_t device_index(const uint16_t** idx_out, const int32_t** off_out) {
    const int32_t* hoff = nullptr;
    size_t count = 0;
    const uint16_t* hidx = mt_jump_index(&hoff, &count);
    if (!hidx) return cudaErrorUnknown;
    int dev = 0;
    cudaGetDevice(&dev);
    DevTables& D = dev_tables();
    std::lock_guard<std::mutex> lock(D.mu);
    if ((int)D.idx.size() <= dev) {
        D.idx.resize(dev + 1, nullptr);
        D.off.resize(dev + 1, nullptr);
    }
    if (!D.idx[dev]) {
        const size_t noff = (size_t)kMtLevels * 31 * kMtJumpParts + 1;
        uint16_t* di = nullptr;
        int32_t* dof = nullptr;
        cudaError_t e = cudaMalloc(&di, count * sizeof(uint16_t));
        if (e == cudaSuccess) e = cudaMalloc(&dof, noff * sizeof(int32_t));
        if (e == cudaSuccess) e = cudaMemcpy(di, hidx, count * sizeof(uint16_t), cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaMemcpy(dof, hoff, noff * sizeof(int32_t), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(di);
            cudaFree(dof);
            return e;
        }
        D.idx[dev] = di;
        D.off[dev] = dof;
    }
    *idx_out = D.idx[dev];
    *off_out = D.off[dev];
    return cudaSuccess;
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

cudaError_t launch_mt_chunk_states(uint64_t seed, uint64_t e_begin, int64_t n, void* ws,
                                   size_t ws_bytes, const uint64_t** states, cudaStream_t st) {
    const MtWs L = mt_ws_layout(e_begin, n);
    if (n <= 0 || ws_bytes < L.total || (e_begin & 31u)) return cudaErrorInvalidValue;
    const uint16_t* jidx = nullptr;
    const int32_t* joff = nullptr;
    cudaError_t err = device_index(&jidx, &joff);
    if (err != cudaSuccess) return err;
    char* w = static_cast<char*>(ws);
    uint64_t* seed_st = reinterpret_cast<uint64_t*>(w + L.seed_off);
    uint64_t* sa = reinterpret_cast<uint64_t*>(w + L.sa_off);
    uint64_t* sb = reinterpret_cast<uint64_t*>(w + L.sb_off);
    uint64_t* base = reinterpret_cast<uint64_t*>(w + L.base_off);

    launch(mt_seed_kernel, 1, 32, 0, st)(seed, seed_st);

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
            launch(mt_base_kernel, (unsigned)S, kGenThreads, 0, st)(cur, base);
            err = cudaMemsetAsync(nxt, 0, (size_t)(chi - clo + 1) * kMtN * sizeof(uint64_t), st);
            if (err != cudaSuccess) return err;
            dim3 grid(kMtJumpParts, 32, (unsigned)S);
            launch(mt_jump_kernel, grid, kJumpThreads, 0, st)(base, jidx, joff, l * 31, nxt, lo * 32,
                                                          clo, chi);
            err = cudaGetLastError();
            if (err != cudaSuccess) return err;
        }
        cur = nxt;
        lo = clo;
        hi = chi;
    }
    *states = cur;
    return cudaGetLastError();
}

cudaError_t launch_mt_keep_bits(uint64_t seed, double p, uint64_t e_begin, int64_t n,
                                uint32_t* mask, void* ws, size_t ws_bytes, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const uint64_t* cur = nullptr;
    cudaError_t err = launch_mt_chunk_states(seed, e_begin, n, ws, ws_bytes, &cur, st);
    if (err != cudaSuccess) return err;
    const int64_t k0 = (int64_t)(e_begin / kMtChunk);
    const int64_t k1 = (int64_t)((e_begin + (uint64_t)n - 1) / kMtChunk);
    const uint64_t xmin = mt_keep_threshold(p);
    launch(mt_keep_kernel, (unsigned)(k1 - k0 + 1), kGenThreads, 0, st)(cur, k0, e_begin,
                                                                   e_begin + (uint64_t)n, xmin,
                                                                   mask);
    return cudaGetLastError();
}

}  // namespace tb
