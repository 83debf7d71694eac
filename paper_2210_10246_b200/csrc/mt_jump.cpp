// mt_jump.cpp -- jump-ahead for std::mt19937_64 (host side).
//
// The reference draws every dropout mask from ONE sequential std::mt19937_64
// stream per tensor (BoolMask::bernoulli_keep, tensor.cpp:186-203, seeded by
// encoder::mask_stream_seed, encoder.cpp:39-46).  To reproduce that stream on
// the device in parallel, the stream is cut into chunks of kMtChunk outputs
// and every chunk's generator state is obtained by jumping ahead from the
// seeded state (Haramoto et al., "Efficient jump ahead for F2-linear random
// number generators", 2008):
//
//   * the transition T of the 19937-bit state is linear over GF(2); its
//     characteristic polynomial P (degree 19937) is the minimal polynomial of
//     any output bit sequence, found here once with Berlekamp-Massey;
//   * with g(x) = x^J mod P, T^J s = g(T) s = XOR of the windows
//     (w_i .. w_{i+311}) of the word sequence started at s, over the i with
//     g_i = 1 (only the low 31 bits of the first word, which never reach an
//     output, can differ);
//   * jump polynomials x^(d * 32^l * kMtChunk) mod P for digits d = 1..31 at
//     levels l = 0..kMtLevels-1 are computed once per process (GF(2)
//     polynomial arithmetic on 64-bit words) and uploaded once per device.
//
// This file also holds a host reference of the whole construction
// (tempo_mt_state_after_host), used by the CPU tests to pin the math against
// std::mt19937_64::discard.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <random>
#include <vector>

#include "mt19937.h"

namespace tb {
namespace {

using Poly = std::vector<uint64_t>;  // bit i of word i/64 = coefficient of x^i

int degree(const Poly& a) {
    for (int w = (int)a.size() - 1; w >= 0; --w)
        if (a[w]) return 64 * w + 63 - __builtin_clzll(a[w]);
    return -1;
}
inline int bit(const Poly& a, int i) { return (int)((a[i >> 6] >> (i & 63)) & 1u); }
inline void flip(Poly& a, int i) { a[i >> 6] ^= 1ull << (i & 63); }

// a ^= b << s
void xor_shifted(Poly& a, const Poly& b, int s) {
    const int ws = s >> 6, bs = s & 63;
    const int need = (int)b.size() + ws + 1;
    if ((int)a.size() < need) a.resize(need, 0);
    if (bs == 0) {
        for (size_t k = 0; k < b.size(); ++k) a[k + ws] ^= b[k];
    } else {
        for (size_t k = 0; k < b.size(); ++k) {
            a[k + ws] ^= b[k] << bs;
            a[k + ws + 1] ^= b[k] >> (64 - bs);
        }
    }
}

// Carry-less 64x64 -> 128 multiply (4-bit window), software.
inline void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
    uint64_t tab[16][2];
    tab[0][0] = tab[0][1] = 0;
    for (int i = 1; i < 16; ++i) {
        // tab[i] = i * a
        const int t = i & -i;  // lowest set bit
        const int sh = __builtin_ctz(t);
        tab[i][0] = tab[i ^ t][0] ^ (a << sh);
        tab[i][1] = tab[i ^ t][1] ^ (sh ? (a >> (64 - sh)) : 0);
    }
    lo = hi = 0;
    for (int k = 60; k >= 0; k -= 4) {
        hi = (hi << 4) | (lo >> 60);
        lo <<= 4;
        const int nib = (int)((b >> k) & 15u);
        lo ^= tab[nib][0];
        hi ^= tab[nib][1];
    }
}

Poly mul(const Poly& a, const Poly& b) {
    Poly r(a.size() + b.size() + 1, 0);
    for (size_t i = 0; i < a.size(); ++i) {
        if (!a[i]) continue;
        for (size_t j = 0; j < b.size(); ++j) {
            if (!b[j]) continue;
            uint64_t lo, hi;
            clmul64(a[i], b[j], lo, hi);
            r[i + j] ^= lo;
            r[i + j + 1] ^= hi;
        }
    }
    return r;
}

// a mod p (p monic of degree dp) through a table of x^(dp + k) mod p, k < 64.
struct Reducer {
    int dp;
    std::vector<Poly> hi;  // hi[k] = x^(dp + k) mod p, k < 64
    explicit Reducer(const Poly& p) : dp(degree(p)) {
        // x^dp mod p = p - x^dp
        Poly base = p;
        base.resize((dp >> 6) + 1, 0);
        flip(base, dp);
        hi.push_back(base);
        for (int k = 1; k < 64; ++k) {
            Poly v = hi.back();
            // multiply by x
            uint64_t carry = 0;
            for (auto& w : v) {
                const uint64_t nc = w >> 63;
                w = (w << 1) | carry;
                carry = nc;
            }
            if (carry) v.push_back(carry);
            v.resize((dp >> 6) + 2, 0);
            if (bit(v, dp)) {
                flip(v, dp);
                for (size_t q = 0; q < base.size(); ++q) v[q] ^= base[q];
            }
            v.resize((dp >> 6) + 1);
            hi.push_back(v);
        }
    }
    Poly reduce(Poly a) const {
        // x^i = x^(64 q) * x^(dp + k), i - dp = 64 q + k: clear bit i and xor
        // hi[k] in at word offset q (lower degree), from the top down.
        for (int i = degree(a); i >= dp; --i) {
            if (!bit(a, i)) continue;
            flip(a, i);
            const int q = (i - dp) >> 6, k = (i - dp) & 63;
            const Poly& h = hi[k];
            for (size_t w = 0; w < h.size(); ++w) a[w + q] ^= h[w];
        }
        a.resize((dp >> 6) + 1, 0);
        return a;
    }
};

// The word sequence w_0.. of std::mt19937_64 started at `state` (w_0..w_311 =
// state, then the recurrence), `count` words.
std::vector<uint64_t> word_sequence(const uint64_t* state, size_t count) {
    std::vector<uint64_t> w(count);
    for (size_t i = 0; i < kMtN && i < count; ++i) w[i] = state[i];
    for (size_t j = kMtN; j < count; ++j) w[j] = mt_next_word(w[j - 312], w[j - 311], w[j - 156]);
    return w;
}

// Berlekamp-Massey over GF(2) on the low bits of the word sequence of a
// seeded generator: the minimal polynomial = the characteristic polynomial
// of the transition (primitive of degree 19937).
Poly char_poly() {
    uint64_t st[kMtN];
    mt_seed_state(5489u, st);
    const int n2 = 2 * kMtDeg + 64;
    std::vector<uint64_t> w = word_sequence(st, (size_t)n2 + kMtN);
    // s_k = bit 0 of w_{312+k}; stored reversed r[n2-1-k] = s_k so that the
    // discrepancy sum_i C_i s_{N-i} is a bitwise dot product with C.
    const int nw = (n2 + 63) / 64 + 1;
    Poly r(nw + 1, 0);
    for (int k = 0; k < n2; ++k)
        if (w[kMtN + k] & 1u) flip(r, n2 - 1 - k);
    Poly C(nw, 0), B(nw, 0);
    C[0] = 1;
    B[0] = 1;
    int L = 0, m = 1;
    for (int N = 0; N < n2; ++N) {
        // d = sum_{i=0..L} C_i s_{N-i} = sum_i C_i r[base + i], base = n2-1-N
        const int base = n2 - 1 - N;
        const int bw = base >> 6, bb = base & 63;
        uint64_t acc = 0;
        const int cw = (L >> 6) + 1;
        for (int q = 0; q < cw; ++q) {
            uint64_t win = r[bw + q] >> bb;
            if (bb) win |= r[bw + q + 1] << (64 - bb);
            acc ^= win & C[q];
        }
        // mask C beyond L (C has no bits above L anyway)
        const int d = __builtin_popcountll(acc) & 1;
        if (!d) {
            ++m;
        } else if (2 * L <= N) {
            Poly T = C;
            xor_shifted(C, B, m);
            C.resize(nw, 0);
            L = N + 1 - L;
            B = T;
            m = 1;
        } else {
            xor_shifted(C, B, m);
            C.resize(nw, 0);
            ++m;
        }
    }
    // characteristic polynomial = reciprocal of the connection polynomial
    Poly P((L >> 6) + 1, 0);
    for (int i = 0; i <= L; ++i)
        if (bit(C, i)) flip(P, L - i);
    return P;
}

struct JumpTables {
    bool ok = false;
    Poly P;
    std::vector<uint64_t> polys;  // [kMtLevels][31][kMtPolyWords]
    std::vector<uint16_t> idx;    // set-bit lists per (poly, part), padded
    std::vector<int32_t> off;     // [kMtLevels * 31 * kMtJumpParts + 1]
};

void build_index(JumpTables& T) {
    const int npoly = kMtLevels * 31;
    T.off.assign((size_t)npoly * kMtJumpParts + 1, 0);
    T.idx.clear();
    for (int pi = 0; pi < npoly; ++pi) {
        const uint64_t* g = T.polys.data() + (size_t)pi * kMtPolyWords;
        for (int q = 0; q < kMtJumpParts; ++q) {
            T.off[(size_t)pi * kMtJumpParts + q] = (int32_t)T.idx.size();
            const int w0 = q * kMtJumpWords, w1 = std::min(kMtPolyWords, w0 + kMtJumpWords);
            for (int w = w0; w < w1; ++w)
                for (int b = 0; b < 64; ++b)
                    if ((g[w] >> b) & 1u) T.idx.push_back((uint16_t)(64 * (w - w0) + b));
            while ((T.idx.size() - T.off[(size_t)pi * kMtJumpParts + q]) % 4)
                T.idx.push_back((uint16_t)kMtJumpSentinel);
        }
    }
    T.off[(size_t)npoly * kMtJumpParts] = (int32_t)T.idx.size();
}

JumpTables& tables() {
    static JumpTables T;
    static std::once_flag once;
    std::call_once(once, [] {
        T.P = char_poly();
        if (degree(T.P) != kMtDeg) return;
        Reducer red(T.P);
        // x^kMtChunk mod P by repeated squaring of x
        Poly x((kMtDeg >> 6) + 1, 0);
        flip(x, 1);
        Poly step = x;
        for (int s = 0; (1ll << s) < kMtChunk; ++s) step = red.reduce(mul(step, step));
        T.polys.assign((size_t)kMtLevels * 31 * kMtPolyWords, 0);
        for (int l = 0; l < kMtLevels; ++l) {
            Poly cur = step;  // x^(1 * 32^l * chunk)
            for (int d = 1; d <= 31; ++d) {
                std::copy(cur.begin(), cur.begin() + kMtPolyWords,
                          T.polys.begin() + ((size_t)l * 31 + (d - 1)) * kMtPolyWords);
                if (d < 31 || l + 1 < kMtLevels) {
                    Poly nxt = red.reduce(mul(cur, step));
                    cur.swap(nxt);
                }
            }
            step = cur;  // x^(32 * 32^l * chunk)
        }
        build_index(T);
        T.ok = true;
    });
    return T;
}

}  // namespace

void mt_seed_state(uint64_t seed, uint64_t* st) {
    // std::mersenne_twister_engine::seed (f = 6364136223846793005, w = 64)
    st[0] = seed;
    for (uint64_t i = 1; i < kMtN; ++i)
        st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + i;
}

const uint64_t* mt_jump_polys() {
    JumpTables& T = tables();
    return T.ok ? T.polys.data() : nullptr;
}

const uint16_t* mt_jump_index(const int32_t** off, size_t* count) {
    JumpTables& T = tables();
    if (!T.ok) return nullptr;
    *off = T.off.data();
    *count = T.idx.size();
    return T.idx.data();
}

// Apply x^J mod P (given as kMtPolyWords words) to `state` on the host.
void mt_jump_host(const uint64_t* g, const uint64_t* state, uint64_t* out) {
    std::vector<uint64_t> w = word_sequence(state, kMtBaseWords);
    std::fill(out, out + kMtN, 0ull);
    for (int i = 0; i < kMtDeg; ++i)
        if ((g[i >> 6] >> (i & 63)) & 1u)
            for (int j = 0; j < (int)kMtN; ++j) out[j] ^= w[i + j];
}

uint64_t mt_keep_threshold(double p) {
    // keep <=> double(x) * 2^-64 >= p (generate_canonical<double, 53> with a
    // 64-bit engine, then uniform_real_distribution(0, 1)); double(x) rounds
    // to nearest, so keep <=> x >= the smallest x whose rounding is >= p*2^64.
    const double T = std::ldexp(p, 64);
    if (!(T > 0.0)) return 0;
    auto keep = [&](uint64_t x) { return (double)x >= T; };
    uint64_t lo = 0, hi = ~0ull;  // keep(hi) true since T < 2^64
    if (keep(0)) return 0;
    while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (keep(mid)) hi = mid; else lo = mid;
    }
    return hi;
}

}  // namespace tb

extern "C" {

// Host reference of the construction: `count` outputs of std::mt19937_64(seed)
// after discarding `steps`, obtained by jump-ahead (x^steps mod P applied to
// the seeded state) and the recurrence -- the CPU tests pin it against
// std::mt19937_64::discard.  Returns 0, or 9 if the tables failed.
int tempo_mt_outputs_after_host(uint64_t seed, uint64_t steps, int64_t count, uint64_t* out) {
    using namespace tb;
    JumpTables& T = tables();
    if (!T.ok) return 9;
    Reducer red(T.P);
    Poly g((kMtDeg >> 6) + 1, 0);
    flip(g, 0);
    for (int b = 63; b >= 0; --b) {  // left-to-right square and multiply by x
        g = red.reduce(mul(g, g));
        if ((steps >> b) & 1u) {
            Poly h((kMtDeg >> 6) + 2, 0);
            xor_shifted(h, g, 1);
            g = red.reduce(h);
        }
    }
    uint64_t st[kMtN], js[kMtN];
    mt_seed_state(seed, st);
    g.resize(kMtPolyWords, 0);
    mt_jump_host(g.data(), st, js);
    std::vector<uint64_t> w = word_sequence(js, kMtN + (size_t)count);
    for (int64_t j = 0; j < count; ++j) out[j] = mt_temper(w[kMtN + j]);
    return 0;
}

}  // extern "C"
