// tempo_host.cpp -- the reference's C++ operator API on device buffers
// (include/tempo_b200/tempo.hpp).  Types and control flow follow the
// reference (tensor.cpp, ledger.cpp, tape.cpp, graph.cpp, ops_tempo.cpp,
// ops_reference.cpp); every numeric op is a call through the C-ABI
// (include/tempo_b200.h) into the sm_100a kernels -- there is no host math;
// the GEMMs of Graph::matmul/matmul_nt (sdpa) are plain cuBLAS calls.
#include <cublas_v2.h>

#include "../../include/tempo_b200/tempo.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <fstream>
#include <atomic>
#include <map>
#include <mutex>
#include <sstream>

namespace tempo_b200 {

// ---- errors -------------------------------------------------------------------
void check(int status) {
    if (status == TEMPO_OK) return;
    std::string msg = tempo_last_error();
    switch (status) {
        case TEMPO_ERR_DIMENSION: throw DimensionError(msg);
        case TEMPO_ERR_PARAM: throw ParamError(msg);
        case TEMPO_ERR_STATE: throw StateError(msg);
        case TEMPO_ERR_CONFIG: throw ConfigError(msg);
        case TEMPO_ERR_LIFECYCLE: throw LifecycleError(msg);
        case TEMPO_ERR_DOMAIN: throw DomainError(msg);
        case TEMPO_ERR_PARSE: throw ParseError(msg);
        case TEMPO_ERR_FIT: throw FitError(msg);
        case TEMPO_ERR_INVARIANT: throw InvariantError(msg);
        case TEMPO_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

static void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

std::int64_t shape_numel(const Shape& s) {
    std::int64_t n = 1;
    for (std::int64_t d : s) {
        if (d < 0) throw DimensionError("negative dimension in " + shape_str(s));
        n *= d;
    }
    return n;
}

std::string shape_str(const Shape& s) {
    std::string o = "[";
    for (std::size_t i = 0; i < s.size(); ++i) o += (i ? ", " : "") + std::to_string(s[i]);
    return o + "]";
}

static void require_same_shape(const Shape& a, const Shape& b, const char* what) {
    if (a != b)
        throw DimensionError(std::string(what) + " shapes " + shape_str(a) + " and " +
                             shape_str(b) + " differ");
}

// ---- device memory: stream-ordered, pooled ---------------------------------------
// Every device buffer of this API comes from the device's default memory pool
// through cudaMallocAsync on the stream of the op that creates it (the
// thread's current StreamScope) and goes back with cudaFreeAsync on the same
// stream: no device-wide synchronization per tensor (cudaFree would), and the
// pool keeps freed blocks for reuse (release threshold = unlimited).
namespace {
thread_local tempo_stream_t t_stream = nullptr;

void pool_init() {
    static std::mutex mu;
    static std::map<int, bool> done;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lock(mu);
    if (done[dev]) return;
    cudaMemPool_t pool;
    cuda_check(cudaDeviceGetDefaultMemPool(&pool, dev), "cudaDeviceGetDefaultMemPool");
    std::uint64_t keep = ~0ull;
    cuda_check(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep),
               "cudaMemPoolSetAttribute");
    done[dev] = true;
}

void* dev_alloc(std::size_t bytes, tempo_stream_t st) {
    pool_init();
    void* p = nullptr;
    cuda_check(cudaMallocAsync(&p, bytes, static_cast<cudaStream_t>(st)), "cudaMallocAsync");
    return p;
}
void dev_free(void* p, tempo_stream_t st) {
    if (p) cudaFreeAsync(p, static_cast<cudaStream_t>(st));
}
}  // namespace

StreamScope::StreamScope(tempo_stream_t s) : prev_(t_stream) { t_stream = s; }
StreamScope::~StreamScope() { t_stream = prev_; }
tempo_stream_t current_stream() { return t_stream; }

// ---- Tensor ---------------------------------------------------------------------
struct Tensor::Storage {
    Shape shape;
    float* ptr = nullptr;
    tempo_stream_t stream = nullptr;  // allocation (and release) stream
    // The LayerNorm |gamma| >= 1e-12 refusal (ops_tempo.cpp:100-106) passed
    // for these values: Tensors are immutable values (tensor.hpp:6-9), so the
    // synchronous check (a D2H copy) runs once per gamma storage, not once
    // per layernorm call.
    std::atomic<bool> gamma_ok{false};
    ~Storage() { dev_free(ptr, stream); }
};

Tensor Tensor::empty(Shape shape) {
    auto s = std::make_shared<Storage>();
    std::int64_t n = shape_numel(shape);
    s->shape = std::move(shape);
    s->stream = t_stream;
    if (n > 0) s->ptr = static_cast<float*>(dev_alloc((size_t)n * sizeof(float), t_stream));
    Tensor t;
    t.storage_ = std::move(s);
    return t;
}

Tensor Tensor::zeros(Shape shape) {
    Tensor t = empty(std::move(shape));
    if (t.numel() > 0)
        cuda_check(cudaMemsetAsync(t.data(), 0, t.byte_size(), static_cast<cudaStream_t>(t_stream)),
                   "cudaMemsetAsync");
    return t;
}

Tensor Tensor::from_host(Shape shape, const std::vector<float>& values) {
    if ((std::int64_t)values.size() != shape_numel(shape))
        throw DimensionError("value count " + std::to_string(values.size()) +
                             " does not fill shape " + shape_str(shape));
    Tensor t = empty(std::move(shape));
    if (t.numel() > 0)
        cuda_check(cudaMemcpy(t.data(), values.data(), t.byte_size(), cudaMemcpyHostToDevice),
                   "cudaMemcpy");
    return t;
}

std::vector<float> Tensor::to_host() const {
    std::vector<float> out((size_t)numel());
    // the producer may have run on any stream: finish the device work first
    if (numel() > 0) cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    if (numel() > 0)
        cuda_check(cudaMemcpy(out.data(), data(), byte_size(), cudaMemcpyDeviceToHost),
                   "cudaMemcpy");
    return out;
}

const Shape& Tensor::shape() const {
    if (!storage_) throw StateError("shape() on undefined tensor");
    return storage_->shape;
}
std::int64_t Tensor::numel() const { return storage_ ? shape_numel(storage_->shape) : 0; }
float* Tensor::data() const {
    if (!storage_) throw StateError("data() on undefined tensor");
    return storage_->ptr;
}
Tensor Tensor::from_storage(std::shared_ptr<Storage> s) {
    Tensor t;
    t.storage_ = std::move(s);
    return t;
}

// ---- BoolMask ---------------------------------------------------------------------
static std::int64_t words_of(std::int64_t n) { return (n + 31) / 32; }

BoolMask BoolMask::empty(Shape shape) {
    BoolMask m;
    std::int64_t n = shape_numel(shape);
    m.shape_ = std::move(shape);
    std::size_t bytes = (std::size_t)std::max<std::int64_t>(1, words_of(n)) * 4;
    tempo_stream_t st = t_stream;
    auto* p = static_cast<std::uint32_t*>(dev_alloc(bytes, st));
    m.words_ = std::shared_ptr<std::uint32_t>(p, [st](std::uint32_t* q) { dev_free(q, st); });
    return m;
}

BoolMask BoolMask::bernoulli_keep(Shape shape, double drop_p, std::uint64_t seed) {
    std::int64_t n = shape_numel(shape);
    if (n >= (std::int64_t(1) << 22)) {
        // large masks: the same std::mt19937_64 stream generated on the
        // device by jump-ahead (tempo_bernoulli_keep_bits), bit for bit
        if (!(drop_p >= 0.0) || drop_p >= 1.0)  // tensor.cpp:188-191
            throw ParamError("drop probability must lie in [0, 1), got " + std::to_string(drop_p));
        BoolMask m = empty(std::move(shape));
        const size_t ws_bytes = tempo_bernoulli_keep_bits_workspace_size(0, n);
        void* ws = dev_alloc(ws_bytes, t_stream);
        const int rc = tempo_bernoulli_keep_bits(n, drop_p, seed, 0, m.words(), ws, ws_bytes,
                                                 t_stream);
        dev_free(ws, t_stream);
        check(rc);
        return m;
    }
    std::vector<std::uint32_t> host((size_t)words_of(n));
    check(tempo_bernoulli_keep_bits_host(n, drop_p, seed, host.data()));
    BoolMask m = empty(std::move(shape));
    if (!host.empty())
        cuda_check(cudaMemcpy(m.words(), host.data(), host.size() * 4, cudaMemcpyHostToDevice),
                   "cudaMemcpy");
    return m;
}

BoolMask BoolMask::from_bytes(Shape shape, const std::vector<std::uint8_t>& bytes) {
    std::int64_t n = shape_numel(shape);
    if ((std::int64_t)bytes.size() != n)  // tensor.cpp:207-210
        throw DimensionError("byte count " + std::to_string(bytes.size()) +
                             " does not fill shape " + shape_str(shape));
    std::vector<std::uint32_t> host((size_t)words_of(n), 0u);
    for (std::int64_t i = 0; i < n; ++i) {
        if (bytes[i] > 1)  // tensor.cpp:211-215
            throw ParamError("mask byte out of {0,1}: " + std::to_string(int(bytes[i])));
        if (bytes[i]) host[i / 32] |= 1u << (i % 32);
    }
    BoolMask m = empty(std::move(shape));
    if (!host.empty())
        cuda_check(cudaMemcpy(m.words(), host.data(), host.size() * 4, cudaMemcpyHostToDevice),
                   "cudaMemcpy");
    return m;
}

std::vector<std::uint8_t> BoolMask::to_bytes() const {
    std::int64_t n = numel();
    std::vector<std::uint32_t> host((size_t)words_of(n));
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    if (!host.empty())
        cuda_check(cudaMemcpy(host.data(), words(), host.size() * 4, cudaMemcpyDeviceToHost),
                   "cudaMemcpy");
    std::vector<std::uint8_t> out((size_t)n);
    for (std::int64_t i = 0; i < n; ++i) out[i] = (host[i / 32] >> (i % 32)) & 1u;
    return out;
}

const Shape& BoolMask::shape() const {
    if (!words_) throw StateError("shape() on undefined mask");
    return shape_;
}
std::int64_t BoolMask::numel() const { return words_ ? shape_numel(shape_) : 0; }
std::size_t BoolMask::byte_size() const { return (std::size_t)words_of(numel()) * 4; }
std::uint32_t* BoolMask::words() const {
    if (!words_) throw StateError("words() on undefined mask");
    return words_.get();
}

// ---- GeluPolyTable ------------------------------------------------------------------
GeluPolyTable GeluPolyTable::parse_string(const std::string& v1_text) {
    tempo_gelu_table_t h = nullptr;
    check(tempo_gelu_table_create(v1_text.c_str(), &h));
    GeluPolyTable t;
    t.h_ = std::shared_ptr<tempo_gelu_table_s>(h, [](tempo_gelu_table_t p) {
        tempo_gelu_table_destroy(p);
    });
    return t;
}

GeluPolyTable GeluPolyTable::load(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ParamError("cannot open table file '" + path + "'");  // gelu_table.cpp:304-306
    std::stringstream ss;
    ss << in.rdbuf();
    return parse_string(ss.str());
}

GeluPolyTable GeluPolyTable::default_fit() { return parse_string(tempo_gelu_default_table_v1()); }

bool GeluPolyTable::verified() const {
    if (!h_) return false;
    int v = 0;
    check(tempo_gelu_table_info(h_.get(), nullptr, nullptr, nullptr, nullptr, &v, nullptr,
                                nullptr));
    return v != 0;
}
double GeluPolyTable::x_star() const {
    double v = 0;
    check(tempo_gelu_table_info(h_.get(), &v, nullptr, nullptr, nullptr, nullptr, nullptr,
                                nullptr));
    return v;
}
double GeluPolyTable::y_min() const {
    double v = 0;
    check(tempo_gelu_table_info(h_.get(), nullptr, &v, nullptr, nullptr, nullptr, nullptr,
                                nullptr));
    return v;
}
std::string GeluPolyTable::serialize() const {
    size_t n = 0;
    check(tempo_gelu_table_serialize(h_.get(), nullptr, 0, &n));
    std::string s(n + 1, '\0');
    check(tempo_gelu_table_serialize(h_.get(), s.data(), n + 1, &n));
    s.resize(n);
    return s;
}
double GeluPolyTable::eval(double y, std::uint8_t m) const {
    if (!h_) throw ConfigError("eval on an empty table");
    double out = 0;
    check(tempo_gelu_table_eval_host(h_.get(), &y, &m, &out, 1));
    return out;
}

// ---- StashLedger (ledger.cpp:31-95) ------------------------------------------------
std::int64_t StashLedger::record(const std::string& tag, StashRole role, const Tensor& t) {
    if (!t.defined()) throw ParamError("record of undefined tensor: " + tag);
    return record_raw(tag, role, t.numel(), (std::int64_t)t.byte_size(),
                      (std::int64_t)t.byte_size(), t.ident());
}

std::int64_t StashLedger::record(const std::string& tag, StashRole role, const BoolMask& m) {
    if (!m.defined()) throw ParamError("record of undefined mask: " + tag);
    return record_raw(tag, role, m.numel(), (std::int64_t)m.byte_size(), m.numel(), m.ident());
}

std::int64_t StashLedger::record_raw(const std::string& tag, StashRole role, std::int64_t elems,
                                     std::int64_t bytes, std::int64_t ref_bytes,
                                     const void* ident) {
    auto it = live_index_.find(ident);
    if (it != live_index_.end()) {  // dedup by storage identity
        entries_[it->second].refs++;
        return 0;
    }
    LedgerEntry e;
    e.tag = tag;
    e.role = role;
    e.elems = elems;
    e.bytes = bytes;
    e.ref_bytes = ref_bytes;
    e.ident = ident;
    e.refs = 1;
    e.live = true;
    live_index_[ident] = entries_.size();
    entries_.push_back(e);
    current_ += bytes;
    current_ref_ += ref_bytes;
    if (current_ > peak_) peak_ = current_;
    return bytes;
}

void StashLedger::release(const void* ident) {
    auto it = live_index_.find(ident);
    if (it == live_index_.end())
        throw LifecycleError("release of an identity that is not live in the ledger");
    LedgerEntry& e = entries_[it->second];
    if (--e.refs > 0) return;
    e.live = false;
    current_ -= e.bytes;
    current_ref_ -= e.ref_bytes;
    live_index_.erase(it);
}

bool StashLedger::is_live(const void* ident) const { return live_index_.count(ident) != 0; }

std::map<std::string, std::int64_t> StashLedger::live_by_tag() const {
    std::map<std::string, std::int64_t> out;
    for (const LedgerEntry& e : entries_)
        if (e.live) out[e.tag] += e.bytes;
    return out;
}

// ---- recompute rules (tape.cpp:12-56) ---------------------------------------------
static std::unordered_map<std::string, RecomputeFn>& registry() {
    static std::unordered_map<std::string, RecomputeFn> r;
    return r;
}
void register_recompute_rule(const std::string& id, RecomputeFn fn) { registry()[id] = std::move(fn); }
bool has_recompute_rule(const std::string& id) { return registry().count(id) != 0; }
Tensor run_recompute_rule(const RecomputeRecipe& recipe) {
    auto it = registry().find(recipe.rule);
    if (it == registry().end()) throw ConfigError("unknown recompute rule '" + recipe.rule + "'");
    Tensor t = it->second(recipe);
    if (t.shape() != recipe.result_shape)
        throw InvariantError("recompute rule '" + recipe.rule + "' produced shape " +
                             shape_str(t.shape()) + ", expected " +
                             shape_str(recipe.result_shape));
    return t;
}
std::vector<Tensor> RecomputeRecipe::lock_sources() const {
    std::vector<Tensor> out;
    for (const auto& w : sources) {
        auto s = w.lock();
        if (!s)
            throw LifecycleError("recompute source for rule '" + rule +
                                 "' was freed before backward");
        out.push_back(Tensor::from_storage(std::move(s)));
    }
    return out;
}

LazyStash LazyStash::materialized(std::string tag, StashRole role, Tensor t, bool charged) {
    if (!t.defined()) throw ParamError("materialized stash '" + tag + "' needs a tensor");
    LazyStash s;
    s.tag_ = std::move(tag);
    s.role_ = role;
    s.charged_ = charged;
    s.value_ = std::move(t);
    return s;
}
LazyStash LazyStash::recomputable(std::string tag, StashRole role, RecomputeRecipe recipe) {
    LazyStash s;
    s.tag_ = std::move(tag);
    s.role_ = role;
    s.recipe_ = std::move(recipe);
    return s;
}
const Tensor& LazyStash::stored() const {
    if (!value_) throw StateError("stash '" + tag_ + "' is recomputable, not stored");
    return *value_;
}
const RecomputeRecipe& LazyStash::recipe() const {
    if (!recipe_) throw StateError("stash '" + tag_ + "' is materialized, has no recipe");
    return *recipe_;
}

// ---- Tape (tape.cpp:95-288) -----------------------------------------------------------
bool GradientMap::has(NodeId id) const {
    return id >= 0 && id < (NodeId)grads_.size() && grads_[id].defined();
}
const Tensor& GradientMap::at(NodeId id) const {
    if (!has(id)) throw StateError("no gradient recorded for node " + std::to_string(id));
    return grads_[id];
}

void Tape::check_node_id(NodeId id) const {
    if (id < 0 || id >= (NodeId)nodes_.size())
        throw ParamError("node id " + std::to_string(id) + " out of range");
}

NodeId Tape::leaf(Tensor value, std::string tag) {
    return record("leaf", std::move(tag), {}, std::move(value), {}, nullptr);
}

NodeId Tape::record(std::string op, std::string tag, std::vector<NodeId> inputs, Tensor value,
                    std::vector<LazyStash> stashes, BackwardFn backward) {
    if (backward_done_) throw StateError("record on a tape whose backward already ran");
    if (!value.defined()) throw ParamError("record of op '" + op + "' without a value");
    for (NodeId in : inputs) check_node_id(in);
    TapeNode node;
    node.op = std::move(op);
    node.tag = std::move(tag);
    node.inputs = std::move(inputs);
    node.value = std::move(value);
    node.backward = std::move(backward);
    node.stashes = std::move(stashes);
    if (ledger_) {
        for (const LazyStash& s : node.stashes) {
            if (s.is_materialized() && s.charged()) {
                ledger_->record(s.tag(), s.role(), s.stored());
                node.charged.push_back(s.stored().ident());
            }
        }
    }
    nodes_.push_back(std::move(node));
    return (NodeId)(nodes_.size() - 1);
}

void Tape::charge(NodeId id, const std::string& tag, StashRole role, const BoolMask& m) {
    check_node_id(id);
    if (!ledger_) return;
    ledger_->record(tag, role, m);
    nodes_[id].charged.push_back(m.ident());
}
void Tape::charge(NodeId id, const std::string& tag, StashRole role, const Tensor& t) {
    check_node_id(id);
    if (!ledger_) return;
    ledger_->record(tag, role, t);
    nodes_[id].charged.push_back(t.ident());
}
void Tape::set_output_recipe(NodeId id, RecomputeRecipe recipe) {
    check_node_id(id);
    nodes_[id].output_recipe = std::move(recipe);
}
const TapeNode& Tape::node(NodeId id) const {
    check_node_id(id);
    return nodes_[id];
}
NodeId Tape::record_lazy(std::string op, std::string tag, std::vector<NodeId> inputs,
                         RecomputeRecipe recipe, std::vector<LazyStash> stashes,
                         BackwardFn backward) {
    if (backward_done_) throw StateError("record on a tape whose backward already ran");
    for (NodeId in : inputs) check_node_id(in);
    TapeNode node;
    node.op = std::move(op);
    node.tag = std::move(tag);
    node.inputs = std::move(inputs);
    node.backward = std::move(backward);
    node.stashes = std::move(stashes);
    node.output_recipe = std::move(recipe);
    node.lazy = true;
    if (ledger_) {
        for (const LazyStash& s : node.stashes) {
            if (s.is_materialized() && s.charged()) {
                ledger_->record(s.tag(), s.role(), s.stored());
                node.charged.push_back(s.stored().ident());
            }
        }
    }
    nodes_.push_back(std::move(node));
    return (NodeId)(nodes_.size() - 1);
}

const Tensor& Tape::value(NodeId id) const {
    const TapeNode& nd = node(id);
    if (nd.lazy && !nd.value.defined()) {  // first read: run the recipe on the tape's stream
        StreamScope scope(stream_ ? *stream_ : current_stream());
        const_cast<TapeNode&>(nd).value = run_recompute_rule(*nd.output_recipe);
    }
    return nd.value;
}
bool Tape::value_pending(NodeId id) const {
    const TapeNode& nd = node(id);
    return nd.lazy && !nd.value.defined();
}
const Shape& Tape::value_shape(NodeId id) const {
    const TapeNode& nd = node(id);
    return value_pending(id) ? nd.output_recipe->result_shape : nd.value.shape();
}

GradientMap Tape::backward(NodeId root, Tensor seed, bool synchronize) {
    check_node_id(root);
    if (backward_done_) throw StateError("backward already ran on this tape");
    if (!seed.defined()) throw ParamError("backward needs a seed gradient");
    if (seed.shape() != value_shape(root))
        throw DimensionError("seed shape " + shape_str(seed.shape()) +
                             " does not match root value shape " +
                             shape_str(value_shape(root)));
    backward_done_ = true;
    const tempo_stream_t st = stream_ ? *stream_ : nullptr;
    StreamScope scope(st);
    std::vector<Tensor> grads(nodes_.size());
    grads[root] = std::move(seed);
    for (NodeId i = root; i >= 0; --i) {
        if (!grads[i].defined()) continue;
        TapeNode& nd = nodes_[i];
        if (nd.inputs.empty() && !nd.backward) continue;  // leaf
        if (!nd.backward) throw ConfigError("no backward rule recorded for op '" + nd.op + "'");
        BackwardCtx ctx(this, i, grads[i]);
        std::vector<Tensor> gin = nd.backward(ctx);
        if (gin.size() != nd.inputs.size())
            throw InvariantError("op '" + nd.op + "' returned " + std::to_string(gin.size()) +
                                 " gradients for " + std::to_string(nd.inputs.size()) +
                                 " inputs");
        for (std::size_t j = 0; j < gin.size(); ++j) {
            if (!gin[j].defined()) continue;
            NodeId in = nd.inputs[j];
            if (gin[j].shape() != value_shape(in))
                throw InvariantError("op '" + nd.op + "' gradient " + std::to_string(j) +
                                     " has shape " + shape_str(gin[j].shape()));
            if (grads[in].defined()) {  // fan-out accumulation (tape.cpp:225-226)
                Tensor sum = Tensor::empty(gin[j].shape());
                check(tempo_tensor_add(grads[in].data(), gin[j].data(), sum.data(), sum.numel(),
                                       st));
                grads[in] = sum;
            } else {
                grads[in] = gin[j];
            }
        }
        ctx.release_temps();
        if (ledger_)
            for (const void* ident : nd.charged) ledger_->release(ident);
        nd.charged.clear();
        if (i != root) grads[i] = Tensor();
    }
    if (synchronize)
        cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(st)), "backward");
    else
        cuda_check(cudaGetLastError(), "backward");
    return GradientMap(std::move(grads));
}

BackwardCtx::BackwardCtx(Tape* t, NodeId id, const Tensor& g) : tape_(t), id_(id), grad_out_(g) {
    cache_.resize(tape_->nodes_[id_].stashes.size());
}

const Tensor& BackwardCtx::stash(std::size_t i) {  // tape.cpp:244-264
    const TapeNode& nd = tape_->nodes_[id_];
    if (i >= nd.stashes.size())
        throw ParamError("stash index " + std::to_string(i) + " out of range for op '" + nd.op +
                         "'");
    if (cache_[i].defined()) return cache_[i];
    const LazyStash& s = nd.stashes[i];
    if (s.is_materialized()) {
        cache_[i] = s.stored();
    } else {
        Tensor t = run_recompute_rule(s.recipe());
        if (tape_->ledger_) {
            tape_->ledger_->record(s.tag() + "#recomputed", StashRole::OpOwnStash, t);
            temp_idents_.push_back(t.ident());
        }
        cache_[i] = std::move(t);
    }
    return cache_[i];
}

const LazyStash& BackwardCtx::lazy_stash(std::size_t i) const {
    const TapeNode& nd = tape_->nodes_[id_];
    if (i >= nd.stashes.size())
        throw ParamError("stash index " + std::to_string(i) + " out of range for op '" + nd.op +
                         "'");
    return nd.stashes[i];
}

const Tensor& BackwardCtx::input_value(std::size_t i) const {
    const TapeNode& nd = tape_->nodes_[id_];
    if (i >= nd.inputs.size())
        throw ParamError("input index " + std::to_string(i) + " out of range for op '" + nd.op +
                         "'");
    return tape_->value(nd.inputs[i]);
}

void BackwardCtx::release_temps() {
    if (tape_->ledger_)
        for (const void* ident : temp_idents_) tape_->ledger_->release(ident);
    temp_idents_.clear();
    cache_.clear();
}

LazyStash Graph::input_stash(NodeId in, StashRole role) const {
    const TapeNode& producer = tape.node(in);
    if (producer.output_recipe)
        return LazyStash::recomputable(producer.tag, role, *producer.output_recipe);
    return LazyStash::materialized(producer.tag, role, producer.value);
}

// ---- generic nodes (graph.cpp:32-89) ---------------------------------------------
namespace {
std::string fallback_tag(std::string tag, const char* op, std::size_t id) {
    if (!tag.empty()) return tag;
    return std::string(op) + "_" + std::to_string(id);
}

// One cuBLAS handle per (thread, device): cublasSetStream + the GEMM on a
// handle shared across threads would race (another thread's SetStream could
// land between them and put the GEMM on the wrong stream).  Thread-local
// handles need no lock; they are released at thread exit.
struct BlasHandles {
    std::map<int, cublasHandle_t> h;
    ~BlasHandles() {
        for (auto& kv : h)
            if (kv.second) cublasDestroy(kv.second);
    }
};
cublasHandle_t blas(tempo_stream_t st) {
    thread_local BlasHandles handles;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    cublasHandle_t& h = handles.h[dev];
    if (!h) {
        if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) throw StateError("cublasCreate failed");
        cublasSetMathMode(h, CUBLAS_PEDANTIC_MATH);  // true fp32, never TF32
    }
    cublasSetStream(h, static_cast<cudaStream_t>(st));
    return h;
}

// Row-major batched C[b] = op_a(A[b]) * op_b(B[b]) (m x n, inner k) as the
// column-major product C^T = op_b(B)^T op_a(A)^T.
void gemm(tempo_stream_t st, bool ta, bool tb, std::int64_t batch, std::int64_t m,
          std::int64_t n, std::int64_t k, const float* A, const float* B, float* C) {
    if (batch == 0 || m == 0 || n == 0) return;
    if (k == 0) {
        cuda_check(cudaMemsetAsync(C, 0, (size_t)(batch * m * n) * 4,
                                   static_cast<cudaStream_t>(st)), "cudaMemsetAsync");
        return;
    }
    const float one = 1.0f, zero = 0.0f;
    const int lda = (int)(ta ? m : k), ldb = (int)(tb ? k : n);
    cublasStatus_t r = cublasSgemmStridedBatched(
        blas(st), tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N, (int)n, (int)m,
        (int)k, &one, B, ldb, (long long)(k * n), A, lda, (long long)(m * k), &zero, C, (int)n,
        (long long)(m * n), (int)batch);
    if (r != CUBLAS_STATUS_SUCCESS) throw StateError("cublasSgemmStridedBatched failed");
}

struct MatDims {
    std::int64_t batch, r, c;
};
MatDims mat_dims(const Shape& s, const char* what) {
    if (s.size() < 2) throw DimensionError(std::string(what) + " needs rank >= 2, got " + shape_str(s));
    std::int64_t b = 1;
    for (size_t i = 0; i + 2 < s.size(); ++i) b *= s[i];
    return {b, s[s.size() - 2], s.back()};
}
void same_batch(const Shape& a, const Shape& b, const char* what) {
    if (a.size() != b.size() || !std::equal(a.begin(), a.end() - 2, b.begin()))
        throw DimensionError(std::string(what) + " needs equal leading dims, got " +
                             shape_str(a) + " and " + shape_str(b));
}
Shape with_last2(const Shape& s, std::int64_t r, std::int64_t c) {
    Shape o = s;
    o[o.size() - 2] = r;
    o.back() = c;
    return o;
}
// c = a b (nn), a b^T (nt), a^T b (tn) on device tensors
Tensor mm(tempo_stream_t st, const Tensor& a, const Tensor& b, bool ta, bool tb) {
    same_batch(a.shape(), b.shape(), "matmul");
    MatDims da = mat_dims(a.shape(), "matmul"), db = mat_dims(b.shape(), "matmul");
    const std::int64_t m = ta ? da.c : da.r, k = ta ? da.r : da.c;
    const std::int64_t kb = tb ? db.c : db.r, n = tb ? db.r : db.c;
    if (k != kb)
        throw DimensionError("matmul inner dims differ: " + shape_str(a.shape()) + " and " +
                             shape_str(b.shape()));
    Tensor c = Tensor::empty(with_last2(a.shape(), m, n));
    gemm(st, ta, tb, da.batch, m, n, k, a.data(), b.data(), c.data());
    return c;
}
}  // namespace

// dV = D^T g for D = the output of dropout_recompute, without D: the
// consumer-side recompute fused into the tcgen05 GEMM (tempo_attn_dropout_dv,
// SURVEY 8f rank 2).  Returns an undefined Tensor when the shapes are outside
// the kernel's envelope; the caller then materialises D through the recipe.
Tensor fused_dropout_dv(tempo_stream_t st, const RecomputeRecipe& recipe, const Tensor& g) {
    if (recipe.rule != "dropout-rescale" || recipe.masks.size() != 1) return Tensor();
    std::vector<Tensor> src = recipe.lock_sources();
    if (src.size() != 1) return Tensor();
    const Tensor& P = src[0];
    const Shape& ps = P.shape();
    const Shape& gs = g.shape();
    if (ps.size() < 2 || gs.size() != ps.size() ||
        !std::equal(ps.begin(), ps.end() - 1, gs.begin()))
        return Tensor();
    const MatDims dp = mat_dims(ps, "matmul"), dg = mat_dims(gs, "matmul");
    Tensor dv = Tensor::empty(with_last2(gs, dp.c, dg.c));
    const int rc = tempo_attn_dropout_dv(P.data(), recipe.masks[0].words(), recipe.scalars.at("p"),
                                         g.data(), dv.data(), dp.batch, dp.r, dp.c, dg.c, st);
    if (rc == TEMPO_ERR_UNSUPPORTED || rc == TEMPO_ERR_ALIGNMENT) return Tensor();
    check(rc);
    return dv;
}

// ctx = D V for D = the (unmaterialised) output of a dropout-rescale recipe:
// the forward consumer of the recompute, fused into the tcgen05 GEMM
// (tempo_attn_dropout_ctx).  Undefined Tensor outside the kernel's envelope.
Tensor fused_dropout_ctx(tempo_stream_t st, const RecomputeRecipe& recipe, const Tensor& v) {
    if (recipe.rule != "dropout-rescale" || recipe.masks.size() != 1) return Tensor();
    std::vector<Tensor> src = recipe.lock_sources();
    if (src.size() != 1) return Tensor();
    const Tensor& P = src[0];
    const Shape& ps = P.shape();
    const Shape& vs = v.shape();
    if (ps.size() < 2 || vs.size() != ps.size() ||
        !std::equal(ps.begin(), ps.end() - 2, vs.begin()))
        return Tensor();
    const MatDims dp = mat_dims(ps, "matmul"), dv = mat_dims(vs, "matmul");
    if (dv.r != dp.c) return Tensor();
    Tensor ctx = Tensor::empty(with_last2(ps, dp.r, dv.c));
    const int rc = tempo_attn_dropout_ctx(P.data(), recipe.masks[0].words(), recipe.scalars.at("p"),
                                          v.data(), ctx.data(), dp.batch, dp.r, dp.c, dv.c, st);
    if (rc == TEMPO_ERR_UNSUPPORTED || rc == TEMPO_ERR_ALIGNMENT) return Tensor();
    check(rc);
    return ctx;
}

NodeId Graph::matmul(NodeId a, NodeId b, std::string tag) {  // graph.cpp:32-51
    StreamScope scope_(stream);
    const Tensor& vb = tape.value(b);
    // a dropout_recompute left operand not yet materialised: D never is
    Tensor out;
    if (tape.value_pending(a)) {
        if (tape.value_shape(a).size() != vb.shape().size())
            throw DimensionError("graph matmul needs equal-rank operands, got " +
                                 shape_str(tape.value_shape(a)) + " and " + shape_str(vb.shape()));
        same_batch(tape.value_shape(a), vb.shape(), "matmul");
        out = fused_dropout_ctx(stream, *tape.node(a).output_recipe, vb);
    }
    if (!out.defined()) {
        const Tensor& va = tape.value(a);
        if (va.shape().size() != vb.shape().size())
            throw DimensionError("graph matmul needs equal-rank operands, got " +
                                 shape_str(va.shape()) + " and " + shape_str(vb.shape()));
        out = mm(stream, va, vb, false, false);
    }
    tag = fallback_tag(std::move(tag), "matmul", tape.size());
    tempo_stream_t st = stream;
    return tape.record("matmul", tag, {a, b}, out,
                       {input_stash(a, StashRole::SharedDownstream),
                        input_stash(b, StashRole::SharedDownstream)},
                       [st](BackwardCtx& ctx) -> std::vector<Tensor> {
                           const Tensor& g = ctx.grad_out();
                           Tensor da = mm(st, g, ctx.stash(1), false, true);
                           // a dropout_recompute left operand: its consumer
                           // rebuilds D inside the dV GEMM (no #recomputed D)
                           const LazyStash& s0 = ctx.lazy_stash(0);
                           Tensor db;
                           if (!s0.is_materialized()) db = fused_dropout_dv(st, s0.recipe(), g);
                           if (!db.defined()) db = mm(st, ctx.stash(0), g, true, false);
                           return {da, db};
                       });
}

NodeId Graph::matmul_nt(NodeId a, NodeId b, std::string tag) {  // graph.cpp:53-71
    StreamScope scope_(stream);
    const Tensor& va = tape.value(a);
    const Tensor& vb = tape.value(b);
    if (va.shape().size() != vb.shape().size())
        throw DimensionError("graph matmul_nt needs equal-rank operands, got " +
                             shape_str(va.shape()) + " and " + shape_str(vb.shape()));
    Tensor out = mm(stream, va, vb, false, true);
    tag = fallback_tag(std::move(tag), "matmul_nt", tape.size());
    tempo_stream_t st = stream;
    return tape.record("matmul_nt", tag, {a, b}, out,
                       {input_stash(a, StashRole::SharedDownstream),
                        input_stash(b, StashRole::SharedDownstream)},
                       [st](BackwardCtx& ctx) -> std::vector<Tensor> {
                           // c = a b^T: da = g b, db = g^T a
                           const Tensor& g = ctx.grad_out();
                           Tensor da = mm(st, g, ctx.stash(1), false, false);
                           Tensor db = mm(st, g, ctx.stash(0), true, false);
                           return {da, db};
                       });
}

NodeId Graph::scale(NodeId a, double c, std::string tag) {  // graph.cpp:73-80
    StreamScope scope_(stream);
    const Tensor& va = tape.value(a);
    Tensor out = Tensor::empty(va.shape());
    check(tempo_tensor_scale(va.data(), c, out.data(), va.numel(), stream));
    tag = fallback_tag(std::move(tag), "scale", tape.size());
    tempo_stream_t st = stream;
    return tape.record("scale", tag, {a}, out, {},
                       [c, st](BackwardCtx& ctx) -> std::vector<Tensor> {
                           const Tensor& g = ctx.grad_out();
                           Tensor d = Tensor::empty(g.shape());
                           check(tempo_tensor_scale(g.data(), c, d.data(), g.numel(), st));
                           return {d};
                       });
}

NodeId Graph::add(NodeId a, NodeId b, std::string tag) {  // graph.cpp:82-89
    StreamScope scope_(stream);
    const Tensor& va = tape.value(a);
    const Tensor& vb = tape.value(b);
    require_same_shape(va.shape(), vb.shape(), "add");
    Tensor out = Tensor::empty(va.shape());
    check(tempo_tensor_add(va.data(), vb.data(), out.data(), va.numel(), stream));
    tag = fallback_tag(std::move(tag), "add", tape.size());
    return tape.record("add", tag, {a, b}, out, {},
                       [](BackwardCtx& ctx) -> std::vector<Tensor> {
                           return {ctx.grad_out(), ctx.grad_out()};
                       });
}

// ---- operators (ops_tempo.cpp, ops_reference.cpp) ---------------------------------
namespace tempo_ops {

void ensure_recompute_rules() {  // ops_tempo.cpp:15-30
    static const bool done = [] {
        register_recompute_rule("dropout-rescale", [](const RecomputeRecipe& recipe) {
            std::vector<Tensor> src = recipe.lock_sources();
            if (src.size() != 1 || recipe.masks.size() != 1)
                throw ConfigError("dropout-rescale recipe needs one source, one mask");
            const double p = recipe.scalars.at("p");
            Tensor d = Tensor::empty(src[0].shape());
            check(tempo_dropout_fwd(src[0].data(), p, TEMPO_MASK_SUPPLIED,
                                    recipe.masks[0].words(), 0, 0, d.data(), d.numel(),
                                    current_stream()));
            return d;
        });
        return true;
    }();
    (void)done;
}

static std::int64_t last_dim(const Shape& s) {
    if (s.empty()) throw DimensionError("expected rank >= 1");
    return s.back();
}

NodeId gelu(Graph& g, NodeId x, const GeluPolyTable* table, std::string tag,
            std::string mask_tag) {  // ops_tempo.cpp:89-96, 32-71
    StreamScope scope_(g.stream);
    if (table == nullptr || table->empty()) throw ConfigError("in-place gelu needs a fitted table");
    const Tensor& vx = g.value(x);
    Tensor y = Tensor::empty(vx.shape());
    BoolMask mask = BoolMask::empty(vx.shape());
    check(tempo_gelu_ip_fwd(vx.data(), y.data(), mask.words(), vx.numel(), table->handle(),
                            g.stream));
    GeluPolyTable tb = *table;  // shared handle
    tempo_stream_t st = g.stream;
    NodeId id = g.tape.record(
        "gelu_ip", tag, {x}, y, {LazyStash::materialized(tag, StashRole::OpOwnStash, y)},
        [tb, mask, st](BackwardCtx& ctx) -> std::vector<Tensor> {
            const Tensor& gy = ctx.grad_out();
            const Tensor& yv = ctx.stash(0);
            require_same_shape(gy.shape(), yv.shape(), "gelu backward");
            Tensor dx = Tensor::empty(yv.shape());
            check(tempo_gelu_ip_bwd(gy.data(), yv.data(), mask.words(), tb.handle(), dx.data(),
                                    yv.numel(), st));
            return {dx};
        });
    g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
    return id;
}

NodeId layernorm(Graph& g, NodeId x, NodeId gamma, NodeId beta, double epsilon, std::string tag,
                 std::string rstd_tag) {  // ops_tempo.cpp:98-156
    StreamScope scope_(g.stream);
    const Tensor& vx = g.value(x);
    const Tensor& vg = g.value(gamma);
    const Tensor& vb = g.value(beta);
    const std::int64_t m = last_dim(vx.shape());
    if (vg.shape() != Shape{m} || vb.shape() != Shape{m})
        throw DimensionError("layernorm affine params " + shape_str(vg.shape()) + ", " +
                             shape_str(vb.shape()) + " do not match " + shape_str(vx.shape()));
    {  // |gamma| < 1e-12 -> ParamError; checked once per (immutable) gamma storage
        std::shared_ptr<Tensor::Storage> gs = vg.weak_storage().lock();
        if (!gs || !gs->gamma_ok.load(std::memory_order_acquire)) {
            check(tempo_ln_check_gamma(vg.data(), m, g.stream));
            if (gs) gs->gamma_ok.store(true, std::memory_order_release);
        }
    }
    const std::int64_t rows = m ? vx.numel() / m : 0;
    Shape rshape(vx.shape().begin(), vx.shape().end() - 1);
    Tensor y = Tensor::empty(vx.shape());
    Tensor rstd = Tensor::empty(rshape);
    check(tempo_ln_ip_fwd(vx.data(), vg.data(), vb.data(), epsilon, y.data(), rstd.data(), rows, m,
                          nullptr, g.stream));
    std::vector<LazyStash> stashes;
    stashes.push_back(LazyStash::materialized(tag, StashRole::OpOwnStash, y));
    stashes.push_back(LazyStash::materialized(rstd_tag, StashRole::Statistic, rstd));
    tempo_stream_t st = g.stream;
    return g.tape.record(
        "layernorm_ip", tag, {x, gamma, beta}, y, std::move(stashes),
        [st, rows, m](BackwardCtx& ctx) -> std::vector<Tensor> {
            const Tensor& gy = ctx.grad_out();
            const Tensor& yv = ctx.stash(0);
            const Tensor& rs = ctx.stash(1);
            const Tensor& gv = ctx.input_value(1);
            const Tensor& bv = ctx.input_value(2);
            Tensor dx = Tensor::empty(yv.shape());
            Tensor dg = Tensor::empty({m}), db = Tensor::empty({m});
            size_t ws_bytes = tempo_ln_ip_bwd_workspace_size(rows, m);
            void* ws = ws_bytes ? dev_alloc(ws_bytes, st) : nullptr;
            int rc = tempo_ln_ip_bwd(gy.data(), yv.data(), rs.data(), gv.data(), bv.data(),
                                     dx.data(), dg.data(), db.data(), ws, ws_bytes, rows, m, st);
            dev_free(ws, st);
            check(rc);
            return {dx, dg, db};
        });
}

NodeId dropout_add_layernorm(Graph& g, NodeId proj, NodeId residual, double p, BoolMask mask,
                             std::uint64_t seed, std::uint64_t offset, NodeId gamma,
                             NodeId beta, double epsilon, std::string tag, std::string rstd_tag,
                             std::string mask_tag) {  // encoder.cpp:180-191, 198-210
    StreamScope scope_(g.stream);
    const Tensor& vp = g.value(proj);
    const Tensor& vr = g.value(residual);
    const Tensor& vg = g.value(gamma);
    const Tensor& vb = g.value(beta);
    require_same_shape(vp.shape(), vr.shape(), "add");
    const std::int64_t m = last_dim(vp.shape());
    if (vg.shape() != Shape{m} || vb.shape() != Shape{m})
        throw DimensionError("layernorm affine params " + shape_str(vg.shape()) + ", " +
                             shape_str(vb.shape()) + " do not match " + shape_str(vp.shape()));
    {  // as tempo_ops::layernorm: checked once per (immutable) gamma storage
        std::shared_ptr<Tensor::Storage> gs = vg.weak_storage().lock();
        if (!gs || !gs->gamma_ok.load(std::memory_order_acquire)) {
            check(tempo_ln_check_gamma(vg.data(), m, g.stream));
            if (gs) gs->gamma_ok.store(true, std::memory_order_release);
        }
    }
    const bool generate = !mask.defined();
    if (generate) mask = BoolMask::empty(vp.shape());
    require_same_shape(vp.shape(), mask.shape(), "mask_scale");
    const std::int64_t rows = m ? vp.numel() / m : 0;
    Shape rshape(vp.shape().begin(), vp.shape().end() - 1);
    Tensor y = Tensor::empty(vp.shape());
    Tensor rstd = Tensor::empty(rshape);
    check(tempo_dropout_add_ln_fwd(vp.data(), vr.data(), p,
                                   generate ? TEMPO_MASK_PHILOX : TEMPO_MASK_SUPPLIED,
                                   mask.words(), seed, offset, vg.data(), vb.data(), epsilon,
                                   y.data(), rstd.data(), rows, m, nullptr, g.stream));
    std::vector<LazyStash> stashes;
    stashes.push_back(LazyStash::materialized(tag, StashRole::OpOwnStash, y));
    stashes.push_back(LazyStash::materialized(rstd_tag, StashRole::Statistic, rstd));
    tempo_stream_t st = g.stream;
    NodeId id = g.tape.record(
        "dropout_add_layernorm", tag, {proj, residual, gamma, beta}, y, std::move(stashes),
        [st, rows, m, mask, p](BackwardCtx& ctx) -> std::vector<Tensor> {
            const Tensor& gy = ctx.grad_out();
            const Tensor& yv = ctx.stash(0);
            const Tensor& rs = ctx.stash(1);
            const Tensor& gv = ctx.input_value(2);
            const Tensor& bv = ctx.input_value(3);
            Tensor d_res = Tensor::empty(yv.shape()), d_proj = Tensor::empty(yv.shape());
            Tensor dg = Tensor::empty({m}), db = Tensor::empty({m});
            size_t ws_bytes = tempo_ln_ip_bwd_workspace_size(rows, m);
            void* ws = ws_bytes ? dev_alloc(ws_bytes, st) : nullptr;
            int rc = tempo_dropout_add_ln_bwd(gy.data(), yv.data(), rs.data(), gv.data(),
                                              bv.data(), mask.words(), p, d_res.data(),
                                              d_proj.data(), dg.data(), db.data(), ws, ws_bytes,
                                              rows, m, nullptr, st);
            dev_free(ws, st);
            check(rc);
            return {d_proj, d_res, dg, db};
        });
    g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
    return id;
}

NodeId softmax(Graph& g, NodeId z, std::string tag) {  // ops_tempo.cpp:158-166
    StreamScope scope_(g.stream);
    const Tensor& vz = g.value(z);
    const std::int64_t c = last_dim(vz.shape());
    const std::int64_t rows = c ? vz.numel() / c : 0;
    Tensor y = Tensor::empty(vz.shape());
    check(tempo_softmax_ip_fwd(vz.data(), y.data(), rows, c, g.stream));
    tempo_stream_t st = g.stream;
    return g.tape.record("softmax_ip", tag, {z}, y,
                         {LazyStash::materialized(tag, StashRole::OpOwnStash, y)},
                         [st, rows, c](BackwardCtx& ctx) -> std::vector<Tensor> {
                             const Tensor& yv = ctx.stash(0);
                             Tensor dz = Tensor::empty(yv.shape());
                             check(tempo_softmax_ip_bwd(ctx.grad_out().data(), yv.data(),
                                                        dz.data(), rows, c, st));
                             return {dz};
                         });
}

// The dropout_recompute node (ops_tempo.cpp:168-194) with a LAZY value: its
// output D = mask ? x / (1-p) : 0 is the node's recipe ("dropout-rescale"
// over x and the mask) and is built only when someone reads it; the
// attention context GEMM (Graph::matmul) consumes the recipe directly, so in
// tempo_ops::sdpa D is materialised in neither pass.  Reading g.value(d)
// gives the same bits as the eager dropout (the recipe IS that kernel).
static NodeId record_dropout_recompute(Graph& g, NodeId x, double p, const BoolMask& mask,
                                       std::string tag, const std::string& mask_tag) {
    const Tensor& vx = g.value(x);
    RecomputeRecipe recipe;
    recipe.rule = "dropout-rescale";
    recipe.sources = {vx.weak_storage()};
    recipe.masks = {mask};
    recipe.scalars["p"] = p;
    recipe.result_shape = vx.shape();
    tempo_stream_t st = g.stream;
    NodeId id = g.tape.record_lazy("dropout_recompute", std::move(tag), {x}, std::move(recipe), {},
                                   [mask, p, st](BackwardCtx& ctx) -> std::vector<Tensor> {
                                       const Tensor& gy = ctx.grad_out();
                                       Tensor dx = Tensor::empty(gy.shape());
                                       check(tempo_dropout_bwd(gy.data(), mask.words(), p, dx.data(),
                                                               gy.numel(), st));
                                       return {dx};
                                   });
    g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
    return id;
}

NodeId dropout_recompute(Graph& g, NodeId x, double p, BoolMask mask, std::string tag,
                         std::string mask_tag) {  // ops_tempo.cpp:168-194
    StreamScope scope_(g.stream);
    ensure_recompute_rules();
    const Tensor& vx = g.value(x);
    if (!g.ledger.is_live(vx.ident()))
        throw ConfigError("dropout_recompute requires its input to be retained upstream");
    require_same_shape(vx.shape(), mask.shape(), "mask_scale");
    if (!(p >= 0.0 && p < 1.0)) throw ParamError("dropout p must be in [0, 1)");
    return record_dropout_recompute(g, x, p, mask, std::move(tag), mask_tag);
}

NodeId softmax_dropout(Graph& g, NodeId z, double p, BoolMask mask, std::uint64_t seed,
                       std::uint64_t offset, const std::string& probs_tag,
                       const std::string& drop_tag, const std::string& mask_tag,
                       NodeId* probs_out) {
    StreamScope scope_(g.stream);
    ensure_recompute_rules();
    const Tensor& vz = g.value(z);
    const std::int64_t c = last_dim(vz.shape());
    const std::int64_t rows = c ? vz.numel() / c : 0;
    const bool generate = !mask.defined();
    if (generate) mask = BoolMask::empty(vz.shape());
    require_same_shape(vz.shape(), mask.shape(), "mask_scale");
    // P and the mask bits only: D is the lazy value of the dropout node
    Tensor P = Tensor::empty(vz.shape());
    check(tempo_softmax_dropout_fwd(vz.data(), p,
                                    generate ? TEMPO_MASK_PHILOX : TEMPO_MASK_SUPPLIED,
                                    mask.words(), seed, offset, P.data(), nullptr, rows, c,
                                    g.stream));
    tempo_stream_t st = g.stream;
    if (!probs_out) {
        // One node z -> D whose backward is the fused attention-probs backward
        // (dropout bwd + output-only softmax bwd in one pass, stash = P + bits);
        // consumers of D get it recomputed from P and the mask (dropout-rescale).
        RecomputeRecipe recipe;
        recipe.rule = "dropout-rescale";
        recipe.sources = {P.weak_storage()};
        recipe.masks = {mask};
        recipe.scalars["p"] = p;
        recipe.result_shape = P.shape();
        NodeId id = g.tape.record_lazy(
            "softmax_dropout", drop_tag, {z}, std::move(recipe),
            {LazyStash::materialized(probs_tag, StashRole::OpOwnStash, P)},
            [st, rows, c, mask, p](BackwardCtx& ctx) -> std::vector<Tensor> {
                const Tensor& pv = ctx.stash(0);
                Tensor dz = Tensor::empty(pv.shape());
                check(tempo_attn_probs_bwd(ctx.grad_out().data(), pv.data(), mask.words(), p,
                                           dz.data(), nullptr, rows, c, st));
                return {dz};
            });
        g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
        return id;
    }
    NodeId pn = g.tape.record("softmax_ip", probs_tag, {z}, P,
                              {LazyStash::materialized(probs_tag, StashRole::OpOwnStash, P)},
                              [st, rows, c](BackwardCtx& ctx) -> std::vector<Tensor> {
                                  const Tensor& yv = ctx.stash(0);
                                  Tensor dz = Tensor::empty(yv.shape());
                                  check(tempo_softmax_ip_bwd(ctx.grad_out().data(), yv.data(),
                                                             dz.data(), rows, c, st));
                                  return {dz};
                              });
    if (probs_out) *probs_out = pn;
    return record_dropout_recompute(g, pn, p, mask, drop_tag, mask_tag);
}

NodeId sdpa(Graph& g, NodeId q, NodeId k, NodeId v, double p, BoolMask mask,
            const std::string& prefix) {  // ops_tempo.cpp:196-210
    StreamScope scope_(g.stream);
    const Shape& qs = g.value(q).shape();
    if (qs.size() != 4) throw DimensionError("sdpa expects [B,A,S,d] inputs, got " + shape_str(qs));
    const std::int64_t d = qs.back();
    NodeId raw = g.matmul_nt(q, k, prefix + "scores_raw");
    NodeId scores = g.scale(raw, 1.0 / std::sqrt(double(d)), prefix + "scores");
    NodeId probs = softmax(g, scores, prefix + "probs");
    NodeId drop = dropout_recompute(g, probs, p, std::move(mask), prefix + "drop_out",
                                    prefix + "drop_mask");
    return g.matmul(drop, v, prefix + "context_heads");
}

}  // namespace tempo_ops

namespace ref_ops {
NodeId dropout(Graph& g, NodeId x, double p, BoolMask mask, std::string tag,
               std::string mask_tag) {  // ops_reference.cpp:214-225
    StreamScope scope_(g.stream);
    const Tensor& vx = g.value(x);
    require_same_shape(vx.shape(), mask.shape(), "mask_scale");
    Tensor y = Tensor::empty(vx.shape());
    check(tempo_dropout_fwd(vx.data(), p, TEMPO_MASK_SUPPLIED, mask.words(), 0, 0, y.data(),
                            vx.numel(), g.stream));
    tempo_stream_t st = g.stream;
    NodeId id = g.tape.record("dropout_ref", std::move(tag), {x}, y, {},
                              [mask, p, st](BackwardCtx& ctx) -> std::vector<Tensor> {
                                  const Tensor& gy = ctx.grad_out();
                                  Tensor dx = Tensor::empty(gy.shape());
                                  check(tempo_dropout_bwd(gy.data(), mask.words(), p, dx.data(),
                                                          gy.numel(), st));
                                  return {dx};
                              });
    g.tape.charge(id, mask_tag, StashRole::OpOwnStash, mask);
    return id;
}
}  // namespace ref_ops

}  // namespace tempo_b200
