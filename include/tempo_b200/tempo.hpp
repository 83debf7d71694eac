// tempo_b200/tempo.hpp -- the reference's C++ operator API for the Tempo
// in-place path (proj/include/tempo/ops_tempo.hpp:18-66 and the Graph /
// Tape / StashLedger / Tensor / BoolMask / GeluPolyTable types it is built
// on), backed by DEVICE buffers and the sm_100a kernels behind the C-ABI of
// include/tempo_b200.h.  A reference caller switches
//     #include "tempo/ops_tempo.hpp"   ->   #include "tempo_b200/tempo.hpp"
//     namespace tempo                  ->   namespace tempo_b200
// and keeps its builder calls: tempo_ops::gelu / layernorm / softmax /
// dropout_recompute, ref_ops::dropout, Graph::leaf/param/value/input_stash,
// Tape::backward, StashLedger::live_by_tag / current_bytes / peak_bytes.
//
// Differences that follow from the device representation:
//   * Tensor is fp32 on the GPU (the reference's F32 storage); host <->
//     device copies are explicit (from_host / to_host).
//   * BoolMask is bit packed (n/32 uint32 words); the ledger charges its
//     real device bytes (n/8 rounded up to words), and also reports the
//     reference's 1-byte-per-element accounting (reference_bytes()).
//   * Every op runs on the graph's CUDA stream; errors are thrown as the
//     reference's exception classes (proj/include/tempo/errors.hpp:14-61).
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../tempo_b200.h"

// tempo_b200/inplace_elementwise.cuh adds the templated graph builder when
// this header was included first.
#define TEMPO_B200_HAS_GRAPH_API 1

namespace tempo_b200 {

// ---- errors (errors.hpp:14-61) ----------------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct DimensionError : Error { using Error::Error; };
struct ParamError : Error { using Error::Error; };
struct StateError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct LifecycleError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct FitError : Error { using Error::Error; };
struct InvariantError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };

// Throws the exception class matching a tempo_status_t (no-op for TEMPO_OK).
void check(int status);

using Shape = std::vector<std::int64_t>;
std::int64_t shape_numel(const Shape& s);
std::string shape_str(const Shape& s);

// ---- Tensor (tensor.hpp:34-102): shared handle over device fp32 storage ---
// Device buffers are allocated stream-ordered (cudaMallocAsync from the
// device's memory pool) on the thread's current stream and released on the
// same stream; every op builder and backward closure runs under a
// StreamScope of its Graph's stream.  Tensors made outside ops use the
// enclosing scope (default: the legacy default stream).  A stream must
// outlive the tensors allocated on it (they are released on it).
class StreamScope {
public:
    explicit StreamScope(tempo_stream_t s);
    ~StreamScope();
    StreamScope(const StreamScope&) = delete;
    StreamScope& operator=(const StreamScope&) = delete;

private:
    tempo_stream_t prev_;
};
tempo_stream_t current_stream();

class Tensor {
public:
    struct Storage;
    Tensor() = default;
    static Tensor zeros(Shape shape);
    static Tensor empty(Shape shape);
    static Tensor from_host(Shape shape, const std::vector<float>& values);
    std::vector<float> to_host() const;

    bool defined() const { return storage_ != nullptr; }
    const Shape& shape() const;
    std::int64_t numel() const;
    std::size_t byte_size() const { return (std::size_t)numel() * 4; }
    float* data() const;
    const void* ident() const { return storage_.get(); }
    std::weak_ptr<Storage> weak_storage() const { return storage_; }
    static Tensor from_storage(std::shared_ptr<Storage> s);

private:
    std::shared_ptr<Storage> storage_;
};

// ---- BoolMask (tensor.hpp:123-146): bit-packed device mask -----------------
class BoolMask {
public:
    BoolMask() = default;
    // tensor.cpp:186-203 -- the reference's own mt19937_64 stream (host), packed.
    static BoolMask bernoulli_keep(Shape shape, double drop_p, std::uint64_t seed);
    // tensor.cpp:205-220 -- validates every byte is 0 or 1 (ParamError).
    static BoolMask from_bytes(Shape shape, const std::vector<std::uint8_t>& bytes);
    // Uninitialized device words (filled by a Philox-generating kernel).
    static BoolMask empty(Shape shape);
    std::vector<std::uint8_t> to_bytes() const;

    bool defined() const { return words_ != nullptr; }
    const Shape& shape() const;
    std::int64_t numel() const;
    std::size_t byte_size() const;  // device bytes (packed words)
    std::uint32_t* words() const;
    const void* ident() const { return words_.get(); }

private:
    Shape shape_;
    std::shared_ptr<std::uint32_t> words_;
};

// ---- GeluPolyTable (gelu_table.hpp:48-91) ----------------------------------
class GeluPolyTable {
public:
    GeluPolyTable() = default;
    static GeluPolyTable parse_string(const std::string& v1_text);  // ParseError
    static GeluPolyTable load(const std::string& path);
    static GeluPolyTable default_fit();  // fit::fit_table() defaults, shipped as data
    bool empty() const { return !h_; }
    bool verified() const;
    double x_star() const;
    double y_min() const;
    std::string serialize() const;
    double eval(double y, std::uint8_t m) const;  // host, gelu_table.cpp:172-188
    tempo_gelu_table_t handle() const { return h_.get(); }

private:
    std::shared_ptr<struct tempo_gelu_table_s> h_;
};

// ---- StashLedger (ledger.hpp:24-79) ----------------------------------------
enum class StashRole { OpOwnStash, SharedDownstream, Statistic };

struct LedgerEntry {
    std::string tag;
    StashRole role = StashRole::OpOwnStash;
    std::int64_t elems = 0;
    std::int64_t bytes = 0;      // device bytes
    std::int64_t ref_bytes = 0;  // the reference's accounting (1 B per mask element)
    const void* ident = nullptr;
    int refs = 0;
    bool live = false;
};

class StashLedger {
public:
    std::int64_t record(const std::string& tag, StashRole role, const Tensor& t);
    std::int64_t record(const std::string& tag, StashRole role, const BoolMask& m);
    void release(const void* ident);  // LifecycleError on unknown / freed
    bool is_live(const void* ident) const;
    std::int64_t current_bytes() const { return current_; }
    std::int64_t peak_bytes() const { return peak_; }
    std::int64_t reference_bytes() const { return current_ref_; }
    std::map<std::string, std::int64_t> live_by_tag() const;
    const std::vector<LedgerEntry>& entries() const { return entries_; }

private:
    std::int64_t record_raw(const std::string& tag, StashRole role, std::int64_t elems,
                            std::int64_t bytes, std::int64_t ref_bytes, const void* ident);
    std::vector<LedgerEntry> entries_;
    std::unordered_map<const void*, std::size_t> live_index_;
    std::int64_t current_ = 0, peak_ = 0, current_ref_ = 0;
};

// ---- Tape (tape.hpp:33-175) -------------------------------------------------
struct RecomputeRecipe {
    std::string rule;
    std::vector<std::weak_ptr<Tensor::Storage>> sources;
    std::vector<BoolMask> masks;
    std::map<std::string, double> scalars;
    Shape result_shape;
    std::vector<Tensor> lock_sources() const;  // LifecycleError if freed
};
using RecomputeFn = std::function<Tensor(const RecomputeRecipe&)>;
void register_recompute_rule(const std::string& id, RecomputeFn fn);
bool has_recompute_rule(const std::string& id);
Tensor run_recompute_rule(const RecomputeRecipe& recipe);  // ConfigError if unknown

class LazyStash {
public:
    static LazyStash materialized(std::string tag, StashRole role, Tensor t, bool charged = true);
    static LazyStash recomputable(std::string tag, StashRole role, RecomputeRecipe recipe);
    bool is_materialized() const { return value_.has_value(); }
    const std::string& tag() const { return tag_; }
    StashRole role() const { return role_; }
    bool charged() const { return charged_; }
    const Tensor& stored() const;
    const RecomputeRecipe& recipe() const;

private:
    std::string tag_;
    StashRole role_ = StashRole::OpOwnStash;
    bool charged_ = true;
    std::optional<Tensor> value_;
    std::optional<RecomputeRecipe> recipe_;
};

using NodeId = std::int32_t;
class BackwardCtx;
using BackwardFn = std::function<std::vector<Tensor>(BackwardCtx&)>;

struct TapeNode {
    std::string op, tag;
    std::vector<NodeId> inputs;
    std::vector<LazyStash> stashes;
    BackwardFn backward;
    Tensor value;  // undefined while a lazy node's value is not yet needed
    std::vector<const void*> charged;
    std::optional<RecomputeRecipe> output_recipe;
    bool lazy = false;  // value = run_recompute_rule(*output_recipe), built on first read
};

class GradientMap {
public:
    explicit GradientMap(std::vector<Tensor> g) : grads_(std::move(g)) {}
    bool has(NodeId id) const;
    const Tensor& at(NodeId id) const;  // StateError if absent

private:
    std::vector<Tensor> grads_;
};

class Tape {
public:
    explicit Tape(StashLedger* ledger = nullptr, const tempo_stream_t* stream = nullptr)
        : ledger_(ledger), stream_(stream) {}
    NodeId leaf(Tensor value, std::string tag);
    NodeId record(std::string op, std::string tag, std::vector<NodeId> inputs, Tensor value,
                  std::vector<LazyStash> stashes, BackwardFn backward);
    void charge(NodeId id, const std::string& tag, StashRole role, const BoolMask& m);
    void charge(NodeId id, const std::string& tag, StashRole role, const Tensor& t);
    void set_output_recipe(NodeId id, RecomputeRecipe recipe);
    // A node whose forward value is its output recipe, built only when read
    // (Tape::value): a consumer that can fuse the recipe into its own kernel
    // (Graph::matmul with a dropout-rescale left operand: the tcgen05 ctx
    // GEMM) never materialises it.  The recipe's result_shape is the shape.
    NodeId record_lazy(std::string op, std::string tag, std::vector<NodeId> inputs,
                       RecomputeRecipe recipe, std::vector<LazyStash> stashes,
                       BackwardFn backward);
    const TapeNode& node(NodeId id) const;
    const Tensor& value(NodeId id) const;  // materialises a lazy node's value
    bool value_pending(NodeId id) const;   // lazy and not yet materialised
    const Shape& value_shape(NodeId id) const;
    std::size_t size() const { return nodes_.size(); }
    // tape.hpp:139.  Like the reference's (synchronous, CPU) backward it
    // returns with every gradient computed: it synchronizes the graph's
    // stream.  `synchronize = false` returns as soon as the work is queued
    // (results are stream-ordered on the graph's stream; host reads such as
    // Tensor::to_host synchronize anyway) -- valid when every tensor the
    // tape touches was allocated on that stream or outlives the work.
    GradientMap backward(NodeId root, Tensor seed, bool synchronize = true);

private:
    std::vector<TapeNode> nodes_;
    StashLedger* ledger_ = nullptr;
    const tempo_stream_t* stream_ = nullptr;  // the owning Graph's stream
    bool backward_done_ = false;
    void check_node_id(NodeId id) const;
    friend class BackwardCtx;
};

class BackwardCtx {
public:
    const Tensor& grad_out() const { return grad_out_; }
    const Tensor& stash(std::size_t i);  // runs a recompute recipe on first use
    // The stash itself, unmaterialised: a consumer that can fuse the
    // recompute into its own kernel (Graph::matmul's dV with a dropout-rescale
    // recipe) reads the recipe instead of calling stash(i).
    const LazyStash& lazy_stash(std::size_t i) const;
    const Tensor& input_value(std::size_t i) const;

private:
    BackwardCtx(Tape* t, NodeId id, const Tensor& g);
    void release_temps();
    Tape* tape_;
    NodeId id_;
    const Tensor& grad_out_;
    std::vector<Tensor> cache_;
    std::vector<const void*> temp_idents_;
    friend class Tape;
};

// ---- Graph (graph.hpp:20-54) -----------------------------------------------
struct Graph {
    StashLedger ledger;
    Tape tape{&ledger, &stream};
    tempo_stream_t stream = nullptr;  // cudaStream_t every op (and its backward) runs on

    NodeId leaf(Tensor value, std::string tag) { return tape.leaf(std::move(value), std::move(tag)); }
    NodeId param(Tensor value, std::string tag) { return leaf(std::move(value), std::move(tag)); }
    const Tensor& value(NodeId id) const { return tape.value(id); }
    // Stash helper honoring the producer's output recipe (graph.cpp:23-30).
    LazyStash input_stash(NodeId in, StashRole role) const;

    // Generic nodes of graph.hpp:35-44 that tempo_ops::sdpa composes.  The
    // GEMMs are plain library GEMMs (cuBLAS, fp32 pedantic: no TF32), batched
    // over equal leading dims; they stash both inputs (through input_stash,
    // so a dropout_recompute producer is rebuilt on demand in the backward).
    // [.., m, k] x [.., k, n]
    NodeId matmul(NodeId a, NodeId b, std::string tag = "");
    // [.., m, k] x [.., n, k]^T
    NodeId matmul_nt(NodeId a, NodeId b, std::string tag = "");
    // c * a, no stash (graph.cpp:73-80)
    NodeId scale(NodeId a, double c, std::string tag = "");
    // a + b, no stash (graph.cpp:82-89)
    NodeId add(NodeId a, NodeId b, std::string tag = "");
};

// ---- Tempo operators (ops_tempo.hpp:33-63) ---------------------------------
namespace tempo_ops {
inline constexpr double kLayerNormGammaMin = 1e-12;
NodeId gelu(Graph& g, NodeId x, const GeluPolyTable* table, std::string tag,
            std::string mask_tag);
NodeId layernorm(Graph& g, NodeId x, NodeId gamma, NodeId beta, double epsilon,
                 std::string tag, std::string rstd_tag);
NodeId softmax(Graph& g, NodeId z, std::string tag);
NodeId dropout_recompute(Graph& g, NodeId x, double p, BoolMask mask, std::string tag,
                         std::string mask_tag);
// Fused device form of softmax -> dropout_recompute (one forward kernel).
// probs_out == nullptr: ONE node z -> D whose backward is the fused
// attention-probs kernel (tempo_attn_probs_bwd); with probs_out, two nodes
// (softmax_ip, then dropout_recompute) like the reference, *probs_out = the
// softmax node.  A Philox mask is generated when `mask` is undefined
// (seed/offset), else it is read.
NodeId softmax_dropout(Graph& g, NodeId z, double p, BoolMask mask, std::uint64_t seed,
                       std::uint64_t offset, const std::string& probs_tag,
                       const std::string& drop_tag, const std::string& mask_tag,
                       NodeId* probs_out);
// The reference layer's hidden dropout -> residual add -> layernorm
// (encoder.cpp:180-191, 198-210: ref_ops::dropout(proj) -> Graph::add ->
// tempo_ops::layernorm) as ONE node: y = LN(residual + dropout(proj)), stash
// = y + rstd + the mask bits (neither the dropout output nor the sum is
// stored); its backward returns {d_proj, d_residual, dgamma, dbeta} in one
// pass (tempo_dropout_add_ln_fwd/bwd).  A Philox mask is generated when
// `mask` is undefined (seed/offset: the bits ref_ops::dropout would read from
// tempo_dropout_fwd's Philox stream), else it is read.  Inputs of the node:
// {proj, residual, gamma, beta}.
NodeId dropout_add_layernorm(Graph& g, NodeId proj, NodeId residual, double p, BoolMask mask,
                             std::uint64_t seed, std::uint64_t offset, NodeId gamma,
                             NodeId beta, double epsilon, std::string tag, std::string rstd_tag,
                             std::string mask_tag);
void ensure_recompute_rules();
// ops_tempo.cpp:196-210: q k^T -> scale 1/sqrt(d) -> softmax-ip ->
// dropout_recompute -> x v, on [B, A, S, d] inputs (DimensionError otherwise).
NodeId sdpa(Graph& g, NodeId q, NodeId k, NodeId v, double p, BoolMask mask,
            const std::string& prefix = "");
}  // namespace tempo_ops

namespace ref_ops {
// ops_reference.cpp:214-225 (hidden dropouts): mask-only stash.
NodeId dropout(Graph& g, NodeId x, double p, BoolMask mask, std::string tag,
               std::string mask_tag);
}  // namespace ref_ops

}  // namespace tempo_b200
