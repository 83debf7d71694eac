// bench_graph.cpp -- the bench.py op chain driven through the C++ operator
// API (include/tempo_b200/tempo.hpp: Graph / Tape / tempo_ops builders), the
// drop-in a reference user would switch to, to measure what the API costs on
// top of the raw C-ABI chain: per step, four tapes (attention probs, hidden
// dropout + LN1, GELU, hidden dropout + LN2) are built on fresh graphs and
// run backward, with stream-ordered pooled allocation for every tensor.
// BERT-large layer shapes (BASELINE configs[3]); masks are inputs made once
// (the reference's mt19937_64 streams, on the device), like the reference.
// Prints one JSON line: ms/step over K steps (CUDA events around the whole
// step, host work included), the algorithmic bytes it moves and GB/s.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "../../include/tempo_b200/tempo.hpp"

using namespace tempo_b200;

static Tensor randn_dev(Shape s, unsigned seed, double scale = 1.0, double shift = 0.0) {
    std::int64_t n = 1;
    for (auto d : s) n *= d;
    std::vector<float> h((size_t)n);
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> nd(0.0, 1.0);
    for (auto& v : h) v = (float)(shift + scale * nd(rng));
    return Tensor::from_host(std::move(s), h);
}

int main(int argc, char** argv) {
    const int steps = argc > 1 ? std::atoi(argv[1]) : 20, warmup = argc > 2 ? std::atoi(argv[2]) : 3;
    // argv[3] == "async": Tape::backward(..., synchronize = false) -- every
    // tensor here lives on stream `st` or outlives the loop
    const bool kSync = !(argc > 3 && std::string(argv[3]) == "async");
    const std::int64_t B = 64, S = 512, H = 1024, A = 16, T = B * S, R = B * A * S;
    const double p = 0.1;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    // inputs (the GEMM outputs / input-gradients of a real layer), made once
    Tensor z = randn_dev({R, S}, 1), x1 = randn_dev({T, H}, 2), xg = randn_dev({T, 4 * H}, 3),
           x2 = randn_dev({T, H}, 4);
    Tensor g1 = randn_dev({H}, 5, 0.2, 1.0), b1 = randn_dev({H}, 6, 0.1),
           g2 = randn_dev({H}, 7, 0.2, 1.0), b2 = randn_dev({H}, 8, 0.1);
    Tensor dD = randn_dev({R, S}, 9), dy1 = randn_dev({T, H}, 10), dyg = randn_dev({T, 4 * H}, 11),
           dy2 = randn_dev({T, H}, 12);
    BoolMask m_att = BoolMask::bernoulli_keep({R, S}, p, tempo_mask_stream_seed(1234, 0, 0));
    BoolMask m1 = BoolMask::bernoulli_keep({T, H}, p, tempo_mask_stream_seed(1234, 0, 1));
    BoolMask m2 = BoolMask::bernoulli_keep({T, H}, p, tempo_mask_stream_seed(1234, 0, 2));
    GeluPolyTable table = GeluPolyTable::default_fit();
    cudaDeviceSynchronize();

    auto step = [&]() {
        {   // attention probabilities: fused softmax + dropout, fused backward
            Graph g;
            g.stream = st;
            NodeId zn = g.leaf(z, "z");
            NodeId d = tempo_ops::softmax_dropout(g, zn, p, m_att, 0, 0, "attn_probs",
                                                  "attn_drop_out", "attn_drop_mask", nullptr);
            g.tape.backward(d, dD, kSync);
        }
        {   // hidden dropout 1 -> LayerNorm 1
            Graph g;
            g.stream = st;
            NodeId xn = g.leaf(x1, "x"), gn = g.param(g1, "g"), bn = g.param(b1, "b");
            NodeId d = ref_ops::dropout(g, xn, p, m1, "d1", "d1_mask");
            NodeId y = tempo_ops::layernorm(g, d, gn, bn, 1e-5, "ln1", "ln1_rstd");
            g.tape.backward(y, dy1, kSync);
        }
        {   // GELU
            Graph g;
            g.stream = st;
            NodeId xn = g.leaf(xg, "x");
            NodeId y = tempo_ops::gelu(g, xn, &table, "gelu", "gelu_mask");
            g.tape.backward(y, dyg, kSync);
        }
        {   // hidden dropout 2 -> LayerNorm 2
            Graph g;
            g.stream = st;
            NodeId xn = g.leaf(x2, "x"), gn = g.param(g2, "g"), bn = g.param(b2, "b");
            NodeId d = ref_ops::dropout(g, xn, p, m2, "d2", "d2_mask");
            NodeId y = tempo_ops::layernorm(g, d, gn, bn, 1e-5, "ln2", "ln2_rstd");
            g.tape.backward(y, dy2, kSync);
        }
    };
    for (int i = 0; i < warmup; ++i) step();
    cudaStreamSynchronize(st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto h0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0, st);
    for (int i = 0; i < steps; ++i) step();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    auto h1 = std::chrono::steady_clock::now();
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= steps;
    const double wall_ms = std::chrono::duration<double, std::milli>(h1 - h0).count() / steps;
    // algorithmic bytes moved, this chain: attention fwd reads
    // z and the bits and writes P (8.125 B: the dropout output D is the
    // node's lazy value and nothing here reads it -- a ctx GEMM consumer
    // would rebuild it in its tcgen05 kernel); its fused bwd reads dD, P,
    // bits and writes dZ (12.125); GELU 8.125 + 12.125; each hidden dropout
    // 8.125 fwd + 8.125 bwd; each LN 8 + 12 (+ rows/cols terms)
    const double na = (double)R * S, nh = (double)T * H, ng = (double)T * 4 * H;
    const double bytes = na * (8.125 + 12.125) + ng * (8.125 + 12.125) +
                         2 * nh * (8.125 + 8.125) + 2 * (8 * nh + 4 * T + 8 * H) +
                         2 * (12 * nh + 4 * T + 16 * H);
    std::printf("{\"what\": \"bench.py op chain through the C++ operator API (Graph/Tape, "
                "fresh graphs per step, stream-ordered pooled allocation)\", \"backward\": \"%s\", "
                "\"steps\": %d, "
                "\"ms_per_step\": %.4f, \"wall_ms_per_step\": %.4f, \"bytes_per_step\": %.0f, "
                "\"gbs\": %.1f}\n",
                kSync ? "synchronous" : "async", steps, ms, wall_ms, bytes,
                bytes / (ms * 1e-3) / 1e9);
    return 0;
}
