// mt19937.h -- std::mt19937_64 (the reference's mask engine, tensor.cpp:197)
// pieces shared by the host jump-ahead code and the device generator.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define TB_HD __host__ __device__ __forceinline__
#else
#define TB_HD inline
#endif

#ifndef TM_MT_CHUNK_LOG2
#define TM_MT_CHUNK_LOG2 19
#endif

namespace tb {

constexpr unsigned kMtN = 312;                  // state words
constexpr int kMtDeg = 19937;                   // degree of the characteristic polynomial
constexpr int kMtPolyWords = (kMtDeg + 63) / 64;  // 312 words per jump polynomial
constexpr int kMtBaseWords = kMtDeg - 1 + kMtN;   // windows i <= 19936 of 312 words
constexpr int64_t kMtChunk = int64_t(1) << TM_MT_CHUNK_LOG2;  // outputs per device stream
constexpr int kMtLevels = 4;                    // 32^4 streams of kMtChunk: 2^38 outputs
// The device jump splits each polynomial's words over kMtJumpParts CTAs.
constexpr int kMtJumpParts = 8;
constexpr int kMtJumpWords = (kMtPolyWords + kMtJumpParts - 1) / kMtJumpParts;  // per part
// Sentinel index of the padded set-bit lists: points past the part's words
// and past the 312-word tail, into a zero region of the staged slice.
constexpr int kMtJumpSentinel = 64 * kMtJumpWords + (int)kMtN;

// w_{j} from w_{j-312}, w_{j-311}, w_{j-156} (mersenne_twister_engine::_M_gen_rand:
// upper 33 bits of w_{j-312}, lower 31 of w_{j-311}, twisted, xor w_{j-156}).
TB_HD uint64_t mt_next_word(uint64_t a, uint64_t b, uint64_t c) {
    const uint64_t y = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
    return c ^ (y >> 1) ^ ((y & 1u) ? 0xB5026F5AA96619E9ull : 0ull);
}

// Tempering of an output word (u=29 d=0x5555.. s=17 b t=37 c l=43).
TB_HD uint64_t mt_temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

#ifdef __CUDACC__
// keep <=> mt_temper(w) >= xmin, from the HIGH word of the tempered output
// alone except on a tie of the high words (probability 2^-32 per output):
// tempering is linear over GF(2), and its last step (z ^= z >> 43) and the
// low half of the third never reach the high word, so hi(temper(w)) =
// hi(y2) ^ ((lo(y2) << 5) & 0xFFF7EEE0) with y1, y2 the first two steps on
// 32-bit halves -- about half the integer work of the full 64-bit temper
// (the generators are issue-bound on it).
__device__ __forceinline__ bool mt_keep(uint64_t w, uint64_t xmin) {
    const uint32_t zl = (uint32_t)w, zh = (uint32_t)(w >> 32);
    const uint32_t y1l = zl ^ (__funnelshift_r(zl, zh, 29) & 0x55555555u);
    const uint32_t y1h = zh ^ ((zh >> 29) & 0x55555555u);
    const uint32_t y2l = y1l ^ ((y1l << 17) & 0xEDA60000u);
    const uint32_t y2h = y1h ^ (__funnelshift_l(y1l, y1h, 17) & 0x71D67FFFu);
    const uint32_t th = y2h ^ ((y2l << 5) & 0xFFF7EEE0u);
    const uint32_t xh = (uint32_t)(xmin >> 32);
    if (th != xh) return th > xh;
    return mt_temper(w) >= xmin;  // tie of the high words
}
#endif

// Host only.
void mt_seed_state(uint64_t seed, uint64_t* st312);
// Jump polynomials x^(d * 32^l * kMtChunk) mod P, layout [l][d-1][kMtPolyWords]
// (computed once per process; nullptr if the construction failed).
const uint64_t* mt_jump_polys();
// The same polynomials as lists of set-bit indices RELATIVE to their part's
// first bit (uint16), each part's list padded with kMtJumpSentinel to a
// multiple of 4; part (l, d-1, q) spans [off[i], off[i+1]) with
// i = (l * 31 + d - 1) * kMtJumpParts + q.
const uint16_t* mt_jump_index(const int32_t** off, size_t* count);
// Smallest 64-bit output x that the reference keeps at drop probability p.
uint64_t mt_keep_threshold(double p);

}  // namespace tb
