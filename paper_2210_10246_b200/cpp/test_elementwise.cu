// test_elementwise.cu -- GPU test of the compile-time in-place elementwise
// scheme (include/tempo_b200/inplace_elementwise.cuh), the analogue of the
// reference's test "the elementwise scheme extends beyond gelu"
// (proj/tests/test_ops_tempo.cpp:291-328).  Exit code = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../../include/tempo_b200/tempo.hpp"
#include "../../include/tempo_b200/inplace_elementwise.cuh"

using namespace tempo_b200;

// exp differentiates from its own output alone; constant branch.
struct ExpSpec {
    __device__ static float fwd(float x) { return expf(x); }
    __device__ static bool branch(float) { return true; }
    __device__ static float grad_from_output(float y, bool) { return y; }
};
// y = x|x| is invertible; the branch bit is not even needed, but the spec
// exercises it: dy/dx = 2|x| = 2 sqrt(|y|).
struct SignedSquareSpec {
    __device__ static float fwd(float x) { return x * fabsf(x); }
    __device__ static bool branch(float x) { return x > 0.0f; }
    __device__ static float grad_from_output(float y, bool) { return 2.0f * sqrtf(fabsf(y)); }
};
// leaky relu: branch = sign, gradient 1 or 0.1 from the branch alone.
struct LeakySpec {
    __device__ static float fwd(float x) { return x > 0.0f ? x : 0.1f * x; }
    __device__ static bool branch(float x) { return x > 0.0f; }
    __device__ static float grad_from_output(float, bool m) { return m ? 1.0f : 0.1f; }
    static bool branch_host(float x) { return x > 0.0f; }
};

static int fails = 0;
#define CHECK(c)                                                                     \
    do {                                                                             \
        if (!(c)) {                                                                  \
            std::printf("  check failed: %s (line %d)\n", #c, __LINE__);            \
            ++fails;                                                                 \
            return;                                                                  \
        }                                                                            \
    } while (0)

static double rel(double a, double b) { return std::abs(a - b) / std::max({1.0, std::abs(a), std::abs(b)}); }

template <class Spec, class F, class G, class B>
static void run(const char* name, std::int64_t n, F f, G grad, B br) {
    int before = fails;
    [&] {
        std::mt19937_64 rng(n);
        std::normal_distribution<double> d(0.0, 1.0);
        std::vector<float> xh(n), gh(n);
        for (auto& v : xh) v = (float)d(rng);
        for (auto& v : gh) v = (float)d(rng);
        Graph g;
        NodeId x = g.leaf(Tensor::from_host({n}, xh), "x");
        NodeId y = tempo_ops::inplace_elementwise<Spec>(g, x, "y", "y_mask");
        CHECK(g.ledger.live_by_tag().at("y") == n * 4);
        CHECK(g.ledger.live_by_tag().at("y_mask") == (n + 31) / 32 * 4);
        CHECK(g.ledger.live_by_tag().count("x") == 0);
        std::vector<float> yh = g.value(y).to_host();
        GradientMap gm = g.tape.backward(y, Tensor::from_host({n}, gh));
        std::vector<float> dx = gm.at(x).to_host();
        for (std::int64_t i = 0; i < n; ++i) {
            CHECK(rel(yh[i], f(xh[i])) <= 1e-6);
            CHECK(rel(dx[i], (double)gh[i] * grad(xh[i])) <= 1e-5);
        }
        (void)br;
    }();
    std::printf("%s %s (n=%lld)\n", fails == before ? "PASS" : "FAIL", name, (long long)n);
}

// Direct kernel calls: mask bits = Spec::branch(x) in BoolMask order, and the
// 256-bit path (32-byte aligned) and the scalar path (4-byte offset) agree
// bitwise on y, the mask and dx.
template <class Spec>
static void paths_agree(const char* name, std::int64_t n) {
    int before = fails;
    [&] {
        std::mt19937_64 rng(n + 7);
        std::normal_distribution<double> d(0.0, 1.0);
        std::vector<float> xh(n), gh(n);
        for (auto& v : xh) v = (float)d(rng);
        for (auto& v : gh) v = (float)d(rng);
        const std::int64_t words = (n + 31) / 32;
        float *xb, *yb, *gb, *db;
        uint32_t* mb;
        cudaMalloc(&xb, (n + 8) * 4); cudaMalloc(&yb, (n + 8) * 4); cudaMalloc(&gb, (n + 8) * 4);
        cudaMalloc(&db, (n + 8) * 4); cudaMalloc(&mb, 2 * words * 4);
        std::vector<float> y0, y1, d0, d1;
        std::vector<uint32_t> m0(words), m1(words);
        for (int off : {0, 1}) {
            cudaMemcpy(xb + off, xh.data(), n * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(gb + off, gh.data(), n * 4, cudaMemcpyHostToDevice);
            uint32_t* m = mb + off * words;
            CHECK(tempo_b200::ew::forward<Spec>(xb + off, yb + off, m, n, nullptr) == cudaSuccess);
            CHECK(tempo_b200::ew::backward<Spec>(gb + off, yb + off, m, db + off, n, nullptr) ==
                  cudaSuccess);
            std::vector<float> yh(n), dh(n);
            cudaMemcpy(yh.data(), yb + off, n * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(dh.data(), db + off, n * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy((off ? m1 : m0).data(), m, words * 4, cudaMemcpyDeviceToHost);
            (off ? y1 : y0) = yh;
            (off ? d1 : d0) = dh;
        }
        cudaFree(xb); cudaFree(yb); cudaFree(gb); cudaFree(db); cudaFree(mb);
        CHECK(y0 == y1 && d0 == d1 && m0 == m1);
        for (std::int64_t i = 0; i < n; ++i)
            CHECK(((m0[i / 32] >> (i % 32)) & 1u) == (uint32_t)Spec::branch_host(xh[i]));
        for (std::int64_t w = 0; w < words; ++w)  // bits past n are zero
            if (w == words - 1 && n % 32) CHECK((m0[w] >> (n % 32)) == 0u);
    }();
    std::printf("%s %s paths agree (n=%lld)\n", fails == before ? "PASS" : "FAIL", name, (long long)n);
}

int main() {
    for (std::int64_t n : {1, 255, 256, 4096 + 37, 1 << 20}) paths_agree<LeakySpec>("leaky relu", n);
    for (std::int64_t n : {1, 127, 128, 1000, 1 << 20}) {
        run<ExpSpec>("exp", n, [](double x) { return std::exp(x); },
                     [](double x) { return std::exp(x); }, 0);
        run<SignedSquareSpec>("signed square", n, [](double x) { return x * std::abs(x); },
                              [](double x) { return 2.0 * std::abs(x); }, 0);
        run<LeakySpec>("leaky relu", n, [](double x) { return x > 0 ? x : 0.1 * x; },
                       [](double x) { return x > 0 ? 1.0 : 0.1; }, 0);
    }
    std::printf("%d failure(s)\n", fails);
    return fails;
}
