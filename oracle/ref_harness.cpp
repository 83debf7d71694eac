// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// Thin extern "C" shims over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libtempo_ref.so).  Nothing here re-implements the reference:
// every function builds the reference's own Graph, calls the reference's own
// operator builders (tempo_ops::*, ref_ops::*) and runs the reference's own
// Tape::backward, exactly as its tests do (proj/tests/test_ops_tempo.cpp:35-47,
// proj/tests/acceptance.cpp:306-320).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference arm may load this library, and only as the checker or the timed
// reference arm -- never on the product path.

#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "tempo/encoder.hpp"
#include "tempo/errors.hpp"
#include "tempo/gelu_fit.hpp"
#include "tempo/gelu_table.hpp"
#include "tempo/graph.hpp"
#include "tempo/memory_model.hpp"
#include "tempo/ops_reference.hpp"
#include "tempo/ops_tempo.hpp"

using namespace tempo;

namespace {

thread_local std::string g_err;

// Error codes mirror include/tempo_b200.h's tempo_status_t so the tests can
// check that the CUDA boundary maps the taxonomy the same way.
int code_of(const std::exception& e) {
    if (dynamic_cast<const DimensionError*>(&e)) return 2;
    if (dynamic_cast<const ParamError*>(&e)) return 3;
    if (dynamic_cast<const StateError*>(&e)) return 4;
    if (dynamic_cast<const ConfigError*>(&e)) return 5;
    if (dynamic_cast<const LifecycleError*>(&e)) return 6;
    if (dynamic_cast<const DomainError*>(&e)) return 7;
    if (dynamic_cast<const ParseError*>(&e)) return 8;
    if (dynamic_cast<const FitError*>(&e)) return 9;
    if (dynamic_cast<const InvariantError*>(&e)) return 10;
    return 1;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

Tensor from_f32(const float* p, Shape shape, Dtype dt) {
    std::int64_t n = shape_numel(shape);
    Tensor t = Tensor::zeros(std::move(shape), dt);
    for (std::int64_t i = 0; i < n; ++i) t.set(i, static_cast<double>(p[i]));
    return t;
}

void to_f32(const Tensor& t, float* out) {
    for (std::int64_t i = 0; i < t.numel(); ++i) {
        out[i] = static_cast<float>(t.get(i));
    }
}

void to_f64(const Tensor& t, double* out) {
    for (std::int64_t i = 0; i < t.numel(); ++i) out[i] = t.get(i);
}

Dtype dt_of(int f64) { return f64 ? Dtype::F64 : Dtype::F32; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// fit::fit_table() with default FitOptions (gelu_fit.cpp:331-382), serialized
// in the v1 text form (gelu_table.cpp:204-218).  Returns the needed length.
int ref_fit_table_default(char* buf, std::int64_t cap, std::int64_t* len) {
    return guarded([&] {
        std::string s = fit::fit_table().serialize();
        *len = static_cast<std::int64_t>(s.size());
        if (buf && cap > static_cast<std::int64_t>(s.size())) {
            std::memcpy(buf, s.data(), s.size() + 1);
        }
    });
}

// fit::fit_table(opts) with a chosen tolerance / degree cap (gelu_fit.hpp:32-46).
int ref_fit_table(double tol, int max_degree, char* buf, std::int64_t cap, std::int64_t* len) {
    return guarded([&] {
        fit::FitOptions o;
        o.tolerance = tol;
        o.max_degree = max_degree;
        std::string s = fit::fit_table(o).serialize();
        *len = static_cast<std::int64_t>(s.size());
        if (buf && cap > static_cast<std::int64_t>(s.size())) {
            std::memcpy(buf, s.data(), s.size() + 1);
        }
    });
}

// GeluPolyTable::eval (gelu_table.cpp:172-188) on a parsed v1 table.
int ref_table_eval(const char* table_text, const double* y,
                   const std::uint8_t* m, double* out, std::int64_t n) {
    return guarded([&] {
        GeluPolyTable t = GeluPolyTable::parse_string(table_text);
        for (std::int64_t i = 0; i < n; ++i) out[i] = t.eval(y[i], m[i]);
    });
}

int ref_table_parse(const char* table_text) {
    return guarded([&] { (void)GeluPolyTable::parse_string(table_text); });
}

// tempo_ops::gelu forward + Tape::backward(node, dy) (ops_tempo.cpp:89-96,
// 32-71; tape.cpp:182-237).  Writes y, the 1-byte branch mask, and dx.
int ref_gelu_ip(const char* table_text, const float* x, const float* dy,
                std::int64_t n, int f64, float* y, std::uint8_t* mask,
                float* dx) {
    return guarded([&] {
        GeluPolyTable table = GeluPolyTable::parse_string(table_text);
        Graph g;
        NodeId xn = g.leaf(from_f32(x, {n}, dt_of(f64)), "x");
        NodeId yn = tempo_ops::gelu(g, xn, &table, "y", "y_mask");
        const Tensor& yv = g.value(yn);
        to_f32(yv, y);
        double x_star = table.minimum().x_star;
        for (std::int64_t i = 0; i < n; ++i) {
            // Same classifier the op recorded (ops_tempo.cpp:77-78); the
            // BoolMask itself lives inside the closure.
            mask[i] = static_cast<double>(x[i]) > x_star ? 1 : 0;
        }
        if (dx) {
            GradientMap gm = g.tape.backward(yn, from_f32(dy, {n}, dt_of(f64)));
            to_f32(gm.at(xn), dx);
        }
    });
}

// Baseline GELU forward (ops_reference.cpp:13-17): the pure math both op sets
// share, so the in-place forward is bitwise equal to it.
int ref_gelu_forward(const float* x, std::int64_t n, float* y) {
    return guarded([&] {
        Tensor t = gelu_forward(from_f32(x, {n}, Dtype::F32));
        to_f32(t, y);
    });
}

// tempo_ops::layernorm forward + backward (ops_tempo.cpp:98-156).
// f64 selects the reference's F64 tensors (the dgamma/dbeta oracle).
int ref_layernorm_ip(const float* x, const float* gamma, const float* beta,
                     const float* dy, std::int64_t rows, std::int64_t cols,
                     double eps, int f64, float* y, float* rstd, float* dx,
                     double* dgamma, double* dbeta) {
    return guarded([&] {
        Dtype dt = dt_of(f64);
        Graph g;
        NodeId xn = g.leaf(from_f32(x, {rows, cols}, dt), "x");
        NodeId gn = g.param(from_f32(gamma, {cols}, dt), "gamma");
        NodeId bn = g.param(from_f32(beta, {cols}, dt), "beta");
        NodeId yn = tempo_ops::layernorm(g, xn, gn, bn, eps, "y", "y_rstd");
        to_f32(g.value(yn), y);
        if (rstd) {
            // The rstd stash is node stash #1 (ops_tempo.cpp:117-118).
            const Tensor& rs = g.tape.node(yn).stashes[1].stored();
            to_f32(rs, rstd);
        }
        if (dx) {
            GradientMap gm =
                g.tape.backward(yn, from_f32(dy, {rows, cols}, dt));
            to_f32(gm.at(xn), dx);
            to_f64(gm.at(gn), dgamma);
            to_f64(gm.at(bn), dbeta);
        }
    });
}

// Backward of tempo_ops::layernorm on GIVEN stashes (y, rstd), i.e. the
// closure at ops_tempo.cpp:121-155 run on identical inputs.  Done by
// re-recording a layernorm node whose forward value is replaced: the closure
// only reads stash 0 (y), stash 1 (rstd) and the gamma/beta input values.
int ref_layernorm_ip_bwd(const float* dy, const float* y, const float* rstd,
                         const float* gamma, const float* beta,
                         std::int64_t rows, std::int64_t cols, int f64,
                         float* dx, double* dgamma, double* dbeta) {
    return guarded([&] {
        Dtype dt = dt_of(f64);
        Graph g;
        // Any x works for recording: the stashes are swapped below.
        NodeId xn = g.leaf(from_f32(y, {rows, cols}, dt), "x");
        NodeId gn = g.param(from_f32(gamma, {cols}, dt), "gamma");
        NodeId bn = g.param(from_f32(beta, {cols}, dt), "beta");
        NodeId yn = tempo_ops::layernorm(g, xn, gn, bn, 1e-5, "y", "y_rstd");
        TapeNode& nd = const_cast<TapeNode&>(g.tape.node(yn));
        nd.stashes[0] = LazyStash::materialized(
            "y", StashRole::OpOwnStash, from_f32(y, {rows, cols}, dt), false);
        nd.stashes[1] = LazyStash::materialized(
            "y_rstd", StashRole::Statistic, from_f32(rstd, {rows}, dt), false);
        GradientMap gm = g.tape.backward(yn, from_f32(dy, {rows, cols}, dt));
        to_f32(gm.at(xn), dx);
        to_f64(gm.at(gn), dgamma);
        to_f64(gm.at(bn), dbeta);
    });
}

// tempo_ops::softmax -> tempo_ops::dropout_recompute -> Tape::backward seeded
// at the dropout node with dD (ops_tempo.cpp:158-194).  D_rec is the
// recompute rule "dropout-rescale" (ops_tempo.cpp:17-26) = dropout_apply.
int ref_softmax_dropout(const float* z, const std::uint8_t* keep, double p,
                        const float* dD, std::int64_t rows, std::int64_t cols,
                        float* P, float* D, float* dZ, float* D_rec) {
    return guarded([&] {
        std::int64_t n = rows * cols;
        Graph g;
        NodeId zn = g.leaf(from_f32(z, {rows, cols}, Dtype::F32), "z");
        NodeId pn = tempo_ops::softmax(g, zn, "probs");
        BoolMask mask = BoolMask::from_bytes(
            {rows, cols}, std::vector<std::uint8_t>(keep, keep + n));
        NodeId dn = tempo_ops::dropout_recompute(g, pn, p, mask, "drop",
                                                 "drop_mask");
        to_f32(g.value(pn), P);
        to_f32(g.value(dn), D);
        if (D_rec) to_f32(dropout_apply(g.value(pn), mask, p), D_rec);
        if (dZ) {
            GradientMap gm =
                g.tape.backward(dn, from_f32(dD, {rows, cols}, Dtype::F32));
            to_f32(gm.at(zn), dZ);
        }
    });
}

// softmax_backward_from_output on given (g, y) (ops_reference.cpp:127-145).
int ref_softmax_bwd(const float* g, const float* y, std::int64_t rows,
                    std::int64_t cols, float* dz) {
    return guarded([&] {
        Tensor t = softmax_backward_from_output(
            from_f32(g, {rows, cols}, Dtype::F32),
            from_f32(y, {rows, cols}, Dtype::F32));
        to_f32(t, dz);
    });
}

// ref_ops::dropout forward + backward (ops_reference.cpp:214-225): the hidden
// dropouts of the encoder layer (encoder.cpp:180-184, 200-203).
int ref_dropout(const float* x, const std::uint8_t* keep, double p,
                const float* dy, std::int64_t n, float* y, float* dx) {
    return guarded([&] {
        Graph g;
        NodeId xn = g.leaf(from_f32(x, {n}, Dtype::F32), "x");
        BoolMask mask = BoolMask::from_bytes(
            {n}, std::vector<std::uint8_t>(keep, keep + n));
        NodeId yn = ref_ops::dropout(g, xn, p, mask, "d", "d_mask");
        to_f32(g.value(yn), y);
        if (dx) {
            GradientMap gm = g.tape.backward(yn, from_f32(dy, {n}, Dtype::F32));
            to_f32(gm.at(xn), dx);
        }
    });
}

// BoolMask::bernoulli_keep (tensor.cpp:186-203).
int ref_bernoulli_keep(std::int64_t n, double p, std::uint64_t seed,
                       std::uint8_t* out) {
    return guarded([&] {
        BoolMask m = BoolMask::bernoulli_keep({n}, p, seed);
        for (std::int64_t i = 0; i < n; ++i) out[i] = m.get(i);
    });
}

// encoder::mask_stream_seed (encoder.cpp:39-46).
std::uint64_t ref_mask_stream_seed(std::uint64_t seed, std::uint64_t salt,
                                   int site) {
    return encoder::mask_stream_seed(seed, salt, site);
}

// memory_model (memory_model.cpp:31-137): per-token bytes of one layer.
int ref_memory_model(std::int64_t batch, std::int64_t seq, std::int64_t hidden,
                     std::int64_t heads, std::int64_t* reference_per_token,
                     std::int64_t* optimized_per_token,
                     std::int64_t* savings4) {
    return guarded([&] {
        memory_model::EncoderConfig cfg;
        cfg.batch = batch;
        cfg.seq = seq;
        cfg.hidden = hidden;
        cfg.heads = heads;
        *reference_per_token = memory_model::reference_bytes_per_token(cfg);
        *optimized_per_token = memory_model::optimized_bytes_per_token(cfg);
        int k = 0;
        for (auto opt : memory_model::kAllOptimizations) {
            savings4[k++] = memory_model::saving_bytes_per_token(cfg, opt);
        }
    });
}

// tempo_ops builders' ledger charges for one op on f32 inputs of n elements
// (test_ops_tempo.cpp:181-265): returns the ledger's current bytes.
int ref_ledger_bytes(int op, std::int64_t rows, std::int64_t cols,
                     const char* table_text, std::int64_t* bytes) {
    return guarded([&] {
        Graph g;
        Tensor x = Tensor::randn({rows, cols}, 17, Dtype::F32);
        NodeId xn = g.leaf(x, "x");
        if (op == 0) {
            GeluPolyTable table = GeluPolyTable::parse_string(table_text);
            tempo_ops::gelu(g, xn, &table, "y", "y_mask");
            *bytes = g.ledger.current_bytes();
            return;
        }
        if (op == 1) {
            NodeId gn = g.param(Tensor::full({cols}, 1.0, Dtype::F32), "gamma");
            NodeId bn = g.param(Tensor::zeros({cols}, Dtype::F32), "beta");
            tempo_ops::layernorm(g, xn, gn, bn, 1e-5, "y", "y_rstd");
        } else if (op == 2) {
            tempo_ops::softmax(g, xn, "y");
        } else {
            NodeId sm = tempo_ops::softmax(g, xn, "sm");
            tempo_ops::dropout_recompute(
                g, sm, 0.5, BoolMask::bernoulli_keep({rows, cols}, 0.5, 19),
                "d", "d_mask");
        }
        *bytes = g.ledger.current_bytes();
    });
}

// ---------------------------------------------------------------------------
// The bench's reference arm: one rank-shard of the BERT-large layer's Tempo
// op chain (bench.py Chain, encoder.cpp:155-210 order) run through the
// reference's own builders and Tape::backward.  ref_chain_create builds the
// inputs ONCE, outside the timed region, with the reference's own synthetic
// generators (Tensor::randn, tensor.cpp:71-77; BoolMask::bernoulli_keep,
// tensor.cpp:186-203) and parses the table once; ref_chain_run is the timed
// step: four tapes (softmax -> dropout_recompute; hidden dropout -> LN1;
// GELU; hidden dropout -> LN2), each forward + Tape::backward, plus the
// consumer's recompute of D (recompute rule "dropout-rescale",
// ops_tempo.cpp:17-26).  with_residual: each hidden dropout feeds a
// Graph::add with a residual stream before its LayerNorm, as the layer does
// (encoder.cpp:185, 204) -- the work bench.py's fused chain covers.
// Nothing is copied in or out per step.
struct RefChain {
    GeluPolyTable table;
    double p;
    Tensor z, dD, x1, x2, xg, dyg, dy1, dy2, g1, b1, g2, b2, res1, res2;
    BoolMask ka, k1, k2;
    bool with_residual = false;
};

void* ref_chain_create(const char* table_text, double p, std::int64_t att_rows,
                       std::int64_t seq, std::int64_t tokens, std::int64_t hidden,
                       std::uint64_t seed, int with_residual) {
    RefChain* c = nullptr;
    int rc = guarded([&] {
        c = new RefChain{GeluPolyTable::parse_string(table_text), p};
        Shape sa{att_rows, seq}, sh{tokens, hidden}, sg{tokens, 4 * hidden};
        std::uint64_t s = seed * 64;
        c->z = Tensor::randn(sa, s + 1, Dtype::F32);
        c->dD = Tensor::randn(sa, s + 2, Dtype::F32);
        c->x1 = Tensor::randn(sh, s + 3, Dtype::F32);
        c->x2 = Tensor::randn(sh, s + 4, Dtype::F32);
        c->xg = Tensor::randn(sg, s + 5, Dtype::F32);
        c->dyg = Tensor::randn(sg, s + 6, Dtype::F32);
        c->dy1 = Tensor::randn(sh, s + 7, Dtype::F32);
        c->dy2 = Tensor::randn(sh, s + 8, Dtype::F32);
        Tensor n1 = Tensor::randn({hidden}, s + 9, Dtype::F64);
        Tensor n2 = Tensor::randn({hidden}, s + 10, Dtype::F64);
        c->g1 = Tensor::zeros({hidden}, Dtype::F32);
        c->g2 = Tensor::zeros({hidden}, Dtype::F32);
        c->b1 = Tensor::zeros({hidden}, Dtype::F32);
        c->b2 = Tensor::zeros({hidden}, Dtype::F32);
        for (std::int64_t j = 0; j < hidden; ++j) {
            c->g1.set(j, 1 + 0.2 * n1.get(j));
            c->g2.set(j, 1 - 0.2 * n2.get(j));
            c->b1.set(j, 0.1 * n2.get(j));
            c->b2.set(j, 0.1 * n1.get(j));
        }
        c->with_residual = with_residual != 0;
        if (c->with_residual) {
            c->res1 = Tensor::randn(sh, s + 14, Dtype::F32);
            c->res2 = Tensor::randn(sh, s + 15, Dtype::F32);
        }
        c->ka = BoolMask::bernoulli_keep(sa, p, s + 11);
        c->k1 = BoolMask::bernoulli_keep(sh, p, s + 12);
        c->k2 = BoolMask::bernoulli_keep(sh, p, s + 13);
    });
    if (rc != 0) {
        delete c;
        return nullptr;
    }
    return c;
}

int ref_chain_run(void* handle) {
    return guarded([&] {
        RefChain& c = *static_cast<RefChain*>(handle);
        {   // attention probabilities: softmax -> dropout_recompute, backward
            Graph g;
            NodeId zn = g.leaf(c.z, "z");
            NodeId pn = tempo_ops::softmax(g, zn, "probs");
            NodeId dn = tempo_ops::dropout_recompute(g, pn, c.p, c.ka, "drop", "drop_mask");
            GradientMap gm = g.tape.backward(dn, c.dD);
            Tensor d_rec = dropout_apply(g.value(pn), c.ka, c.p);  // the dV GEMM's recompute
            (void)gm.at(zn);
        }
        for (int k = 0; k < 2; ++k) {  // hidden dropout -> LayerNorm, backward
            Graph g;
            NodeId xn = g.leaf(k ? c.x2 : c.x1, "x");
            NodeId dn = ref_ops::dropout(g, xn, c.p, k ? c.k2 : c.k1, "d", "d_mask");
            if (c.with_residual) {
                NodeId rn = g.leaf(k ? c.res2 : c.res1, "residual");
                dn = g.add(rn, dn, "ln_input");
            }
            NodeId gn = g.param(k ? c.g2 : c.g1, "gamma");
            NodeId bn = g.param(k ? c.b2 : c.b1, "beta");
            NodeId yn = tempo_ops::layernorm(g, dn, gn, bn, 1e-5, "y", "y_rstd");
            GradientMap gm = g.tape.backward(yn, k ? c.dy2 : c.dy1);
            (void)gm.at(xn);
        }
        {   // GELU, backward
            Graph g;
            NodeId xn = g.leaf(c.xg, "x");
            NodeId yn = tempo_ops::gelu(g, xn, &c.table, "y", "y_mask");
            GradientMap gm = g.tape.backward(yn, c.dyg);
            (void)gm.at(xn);
        }
    });
}

void ref_chain_destroy(void* handle) { delete static_cast<RefChain*>(handle); }

// BASELINE configs[0..2] one op pair at a time (bench.py per_config's CPU
// column): kind 0 = GELU-ip fwd + Tape::backward on [rows, cols] (configs[0]),
// 1 = LayerNorm-ip fwd + backward incl. dgamma/dbeta (configs[1]), 2 =
// softmax -> dropout_recompute fwd + backward + the consumer's recompute of D
// (configs[2]); inputs built once by the reference's own generators.
struct RefOp {
    int kind;
    GeluPolyTable table;
    double p;
    Tensor x, dy, g, b;
    BoolMask keep;
};

void* ref_op_create(int kind, const char* table_text, double p, std::int64_t rows,
                    std::int64_t cols, std::uint64_t seed) {
    RefOp* c = nullptr;
    int rc = guarded([&] {
        c = new RefOp{kind, GeluPolyTable::parse_string(table_text), p};
        Shape sh{rows, cols};
        c->x = Tensor::randn(sh, seed * 16 + 1, Dtype::F32);
        c->dy = Tensor::randn(sh, seed * 16 + 2, Dtype::F32);
        if (kind == 1) {
            Tensor n1 = Tensor::randn({cols}, seed * 16 + 3, Dtype::F64);
            c->g = Tensor::zeros({cols}, Dtype::F32);
            c->b = Tensor::zeros({cols}, Dtype::F32);
            for (std::int64_t j = 0; j < cols; ++j) {
                c->g.set(j, 1 + 0.2 * n1.get(j));
                c->b.set(j, 0.1 * n1.get(j));
            }
        }
        if (kind == 2) c->keep = BoolMask::bernoulli_keep(sh, p, seed * 16 + 4);
    });
    if (rc != 0) {
        delete c;
        return nullptr;
    }
    return c;
}

int ref_op_run(void* handle) {
    return guarded([&] {
        RefOp& c = *static_cast<RefOp*>(handle);
        Graph g;
        NodeId xn = g.leaf(c.x, "x");
        if (c.kind == 0) {
            NodeId yn = tempo_ops::gelu(g, xn, &c.table, "y", "y_mask");
            GradientMap gm = g.tape.backward(yn, c.dy);
            (void)gm.at(xn);
        } else if (c.kind == 1) {
            NodeId gn = g.param(c.g, "gamma");
            NodeId bn = g.param(c.b, "beta");
            NodeId yn = tempo_ops::layernorm(g, xn, gn, bn, 1e-5, "y", "y_rstd");
            GradientMap gm = g.tape.backward(yn, c.dy);
            (void)gm.at(xn);
        } else {
            NodeId pn = tempo_ops::softmax(g, xn, "probs");
            NodeId dn = tempo_ops::dropout_recompute(g, pn, c.p, c.keep, "drop", "drop_mask");
            GradientMap gm = g.tape.backward(dn, c.dy);
            Tensor d_rec = dropout_apply(g.value(pn), c.keep, c.p);  // the dV GEMM's recompute
            (void)gm.at(xn);
        }
    });
}

void ref_op_destroy(void* handle) { delete static_cast<RefOp*>(handle); }

}  // extern "C"

