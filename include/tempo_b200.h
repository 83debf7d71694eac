/*
 * tempo_b200.h -- the C-ABI drop-in boundary of the Tempo in-place
 * activation operators (arXiv 2210.10246) on NVIDIA B200 (sm_100a).
 *
 * Every entry point replaces one reference interface; the citation next to it
 * names the reference file:line (under /root/reference/proj) whose behaviour
 * it reproduces.  INTEGRATION.md shows the binding a maintainer adds on the
 * reference side (its C++ tempo_ops builders calling these from their
 * forward bodies and BackwardFn closures).
 *
 * Conventions
 *   - Tensor pointers are DEVICE pointers, caller-allocated, fp32, row-major,
 *     contiguous.  Nothing here allocates device memory or retains a pointer
 *     past the call (the LayerNorm backward's scratch is a caller workspace).
 *   - Masks are bit-packed uint32 words: bit (i % 32) of word (i / 32) is
 *     element i of the flattened tensor -- the reference's BoolMask byte
 *     order (proj/src/tensor.cpp:199-201) at 1 bit instead of 1 byte.
 *     bit 1 = kept (dropout, tensor.cpp:200) / right-of-minimum (GELU,
 *     ops_tempo.cpp:78).
 *   - Work is enqueued on `stream` (cudaStream_t; NULL = legacy default
 *     stream) and is asynchronous; argument errors are reported before
 *     anything is enqueued.
 *   - Return value: TEMPO_OK or a tempo_status_t mirroring the reference's
 *     exception taxonomy (proj/include/tempo/errors.hpp:14-61);
 *     tempo_last_error() holds the message (thread-local).
 *   - Reentrant; no global mutable state beyond a per-device launch-config
 *     cache.  A table handle is immutable after creation and shareable.
 */
#ifndef TEMPO_B200_H
#define TEMPO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* tempo_stream_t; /* a cudaStream_t */

/* errors.hpp:14-61, one code per exception class, plus device-side failures */
typedef enum {
    TEMPO_OK = 0,
    TEMPO_ERR_UNKNOWN = 1,    /* tempo::Error                                  */
    TEMPO_ERR_DIMENSION = 2,  /* DimensionError: shapes / sizes                 */
    TEMPO_ERR_PARAM = 3,      /* ParamError: p not in [0,1), eps <= 0, |gamma|<1e-12 */
    TEMPO_ERR_STATE = 4,      /* StateError                                     */
    TEMPO_ERR_CONFIG = 5,     /* ConfigError: missing / unverified table        */
    TEMPO_ERR_LIFECYCLE = 6,  /* LifecycleError                                 */
    TEMPO_ERR_DOMAIN = 7,     /* DomainError                                    */
    TEMPO_ERR_PARSE = 8,      /* ParseError: malformed v1 table text            */
    TEMPO_ERR_FIT = 9,        /* FitError                                       */
    TEMPO_ERR_INVARIANT = 10, /* InvariantError                                 */
    TEMPO_ERR_ALIGNMENT = 11, /* pointer not aligned as the call requires       */
    TEMPO_ERR_CUDA = 20,      /* a CUDA runtime error (message has the name)    */
    TEMPO_ERR_UNSUPPORTED = 21
} tempo_status_t;

const char* tempo_last_error(void);
const char* tempo_version(void);

/* ---------------------------------------------------------------------- */
/* GELU derivative-from-output table  (gelu_table.hpp:27-91)               */
/* ---------------------------------------------------------------------- */
typedef struct tempo_gelu_table_s* tempo_gelu_table_t;

/* Parse + validate the v1 text form (GeluPolyTable::parse,
 * gelu_table.cpp:227-301, tiling invariants :106-148).  Host only; the device
 * copy travels as a kernel parameter, so no GPU is touched.  ParseError codes
 * exactly where the reference throws. */
int tempo_gelu_table_create(const char* v1_text, tempo_gelu_table_t* out);
int tempo_gelu_table_destroy(tempo_gelu_table_t table);
/* GeluPolyTable::minimum(), verified(), verified_max_error(), tolerance(),
 * and the segment count/max degree (gelu_table.hpp:55-63). */
int tempo_gelu_table_info(tempo_gelu_table_t table, double* x_star, double* y_min,
                          double* tolerance, double* verified_max_error, int* verified,
                          int* n_segments, int* max_degree);
/* Re-serialize (GeluPolyTable::serialize, gelu_table.cpp:204-218);
 * returns the needed length (without NUL) in *len. */
int tempo_gelu_table_serialize(tempo_gelu_table_t table, char* buf, size_t cap, size_t* len);
/* The table every default-configured reference process fits
 * (fit::fit_table() with default FitOptions, gelu_fit.cpp:331-382),
 * shipped as data so no fit runs at startup.  Static string. */
const char* tempo_gelu_default_table_v1(void);
/* Host-side GeluPolyTable::eval(y, m) (gelu_table.cpp:172-188), double. */
int tempo_gelu_table_eval_host(tempo_gelu_table_t table, const double* y, const uint8_t* m,
                               double* out, int64_t n);

/* ---------------------------------------------------------------------- */
/* In-Place GELU  (tempo_ops::gelu, ops_tempo.cpp:89-96 -> 32-87)          */
/* ---------------------------------------------------------------------- */
/* Forward: y = x*Phi(x) (math.hpp:26-28) and the branch mask
 * m_i = x_i > table.x_star (ops_tempo.cpp:77-78).  mask has ceil(n/32) words.
 * Refuses a NULL/empty table (ConfigError, ops_tempo.cpp:91-94). */
int tempo_gelu_ip_fwd(const float* x, float* y, uint32_t* mask, int64_t n,
                      tempo_gelu_table_t table, tempo_stream_t stream);
/* Reference-exact mode of the forward: y = float(x*0.5*erfc(-x/sqrt2))
 * evaluated in fp64 for EVERY element (math.hpp:17-28, one rounding) instead
 * of the fp32 fast path -- the survey's <= 2-ulp contract with room (it
 * differs from the reference only where CUDA's and glibc's double erfc
 * straddle a float rounding boundary), at several times the FP64 cost (the
 * default forward is <= 6 ulp, 14x inside the 1e-5 relative contract).  Same
 * mask bits, same stash, same backward. */
int tempo_gelu_ip_fwd_exact(const float* x, float* y, uint32_t* mask, int64_t n,
                            tempo_gelu_table_t table, tempo_stream_t stream);
/* Backward closure (ops_tempo.cpp:59-68 + gelu_spec :79-85):
 * dx = dy * table.eval(y, m).  Refuses an unverified table with ConfigError
 * (ops_tempo.cpp:80-83).  dx may alias dy (in place). */
int tempo_gelu_ip_bwd(const float* dy, const float* y, const uint32_t* mask,
                      tempo_gelu_table_t table, float* dx, int64_t n, tempo_stream_t stream);

/* ---------------------------------------------------------------------- */
/* In-Place LayerNorm  (tempo_ops::layernorm, ops_tempo.cpp:98-156)        */
/* ---------------------------------------------------------------------- */
/* Forward over rows of `cols`: two-pass moments (kernels.cpp:153-179), y =
 * gamma*(x-mean)*rstd+beta (ops_reference.cpp:47-65), stashes y and
 * rstd = 1/sqrt(var+eps) per row (ops_tempo.cpp:110-118).  eps <= 0 ->
 * ParamError (ops_reference.cpp:50-52).  The |gamma_j| < 1e-12 refusal
 * (ops_tempo.cpp:100-106) needs gamma's values: pass dev_status (an int32 in
 * device memory, may be NULL) and the kernel writes TEMPO_ERR_PARAM there
 * when any |gamma_j| < 1e-12, or call tempo_ln_check_gamma() up front. */
int tempo_ln_ip_fwd(const float* x, const float* gamma, const float* beta, double eps,
                    float* y, float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                    tempo_stream_t stream);
/* Synchronous refusal check of ops_tempo.cpp:100-106 (copies gamma to host). */
int tempo_ln_check_gamma(const float* gamma, int64_t cols, tempo_stream_t stream);
/* Scratch bytes tempo_ln_ip_bwd needs (two-stage dgamma/dbeta reduction). */
size_t tempo_ln_ip_bwd_workspace_size(int64_t rows, int64_t cols);
/* Backward closure (ops_tempo.cpp:121-155): xhat = (y-beta)/gamma,
 * s1 = sum g*gamma, s2 = sum g*gamma*xhat, dx = (g*gamma - s1/M -
 * xhat*s2/M)*rstd; dgamma_j = sum_i g*xhat, dbeta_j = sum_i g over ALL rows,
 * reduced in a fixed order (bitwise reproducible run to run). */
int tempo_ln_ip_bwd(const float* dy, const float* y, const float* rstd, const float* gamma,
                    const float* beta, float* dx, float* dgamma, float* dbeta, void* workspace,
                    size_t workspace_bytes, int64_t rows, int64_t cols, tempo_stream_t stream);

/* The two stages separately (SURVEY 8b's split form of the backward
 * closure, ops_tempo.cpp:121-155, whose dgamma/dbeta accumulation :150-151
 * becomes stage 2), for callers that combine partials themselves: stage 1
 * writes dx and leaves the per-CTA
 * fp64 partial rows in `workspace` ([*nparts][2*cols]: dgamma partials, then
 * dbeta partials; *nparts is set); tempo_ln_param_reduce sums nparts such
 * rows (any producer: stage 1 here, or partial rows gathered from several
 * ranks) in a fixed order into dgamma/dbeta -- tempo_ln_ip_bwd is exactly
 * stage 1 then stage 2 on the same workspace. */
int tempo_ln_ip_bwd_partials(const float* dy, const float* y, const float* rstd,
                             const float* gamma, const float* beta, float* dx, void* workspace,
                             size_t workspace_bytes, int64_t rows, int64_t cols, int64_t* nparts,
                             tempo_stream_t stream);
int tempo_ln_param_reduce(const double* partials, int64_t nparts, int64_t cols, float* dgamma,
                          float* dbeta, tempo_stream_t stream);

/* Multi-GPU: the path's one collective -- the sum of every
 * rank's LayerNorm dgamma/dbeta -- fused into the backward's stage 2 over
 * peer memory instead of a separate all-reduce (replaces the reference's
 * serial accumulation in the backward closure, ops_tempo.cpp:150-151, summed
 * over row shards).  Each rank owns an inbox and a flag buffer (sizes below,
 * zero-initialised once) that every rank can address: same process (tests),
 * P2P peers, or CUDA IPC mappings (tempo_ipc_*).  `inbox` / `flags` are
 * DEVICE arrays of `world` pointers (rank p's buffers as mapped here); epoch
 * is 1, 2, 3, ... per exchange (the same on all ranks).  The result is the
 * fixed-order (rank 0, 1, ...) sum of the ranks' fixed-order partial sums:
 * bitwise identical on every rank.  A peer that never arrives within
 * timeout_ms (0 = the library default, 30 s) sets *status to
 * TEMPO_ERR_STATE and the affected dgamma/dbeta entries to NaN (never a
 * partial sum) instead of hanging the GPU.  *status is sticky: while it is
 * nonzero every exchange on this rank writes NaN without waiting; rebuild
 * the group (fresh zeroed buffers, epoch 1) to recover. */
typedef struct {
    int32_t rank;
    int32_t world;
    double* const* inbox;
    uint32_t* const* flags;
    uint32_t epoch;
    int32_t* status;
    uint32_t timeout_ms;
} tempo_ln_peer_t;
size_t tempo_ln_peer_inbox_bytes(int32_t world, int64_t cols);
size_t tempo_ln_peer_flag_bytes(int32_t world, int64_t cols);
/* tempo_ln_ip_bwd with the cross-rank dgamma/dbeta sum fused in. */
int tempo_ln_ip_bwd_peer(const float* dy, const float* y, const float* rstd, const float* gamma,
                         const float* beta, float* dx, float* dgamma, float* dbeta,
                         void* workspace, size_t workspace_bytes, int64_t rows, int64_t cols,
                         const tempo_ln_peer_t* peer, tempo_stream_t stream);
/* Stage 2 alone on caller-provided fp64 partial rows [nparts][2*cols]
 * (dgamma partials, then dbeta partials): local fixed-order sum + exchange. */
int tempo_ln_param_reduce_peer(const double* partials, int64_t nparts, int64_t cols,
                               const tempo_ln_peer_t* peer, float* dgamma, float* dbeta,
                               tempo_stream_t stream);
/* Exchange buffers: a dedicated, zero-filled cudaMalloc allocation (an IPC
 * handle always maps the START of an allocation, so sub-allocations of a
 * caching allocator cannot be shared this way). */
/* NCCL fallback of the same sum for callers without P2P / IPC peers
 * (SURVEY 8b tempo_allreduce_ln_params): every rank's bucket of LayerNorm
 * dgamma/dbeta (e.g. [dg2 | db2 | dg1 | db1], 2*cols floats per LN, as
 * written by tempo_ln_ip_bwd) is summed in place over the ranks of
 * `nccl_comm` (an ncclComm_t) on `stream` -- the reference's single-process
 * dgamma/dbeta (ops_tempo.cpp:150-151) summed over row shards.  NCCL is
 * loaded at first use (dlopen "libnccl.so.2"); TEMPO_ERR_UNSUPPORTED if it
 * is absent.  The comm helpers build a communicator from a 128-byte
 * ncclUniqueId that the caller distributes (any out-of-band channel). */
int tempo_allreduce_ln_params(void* nccl_comm, float* bucket, int64_t count,
                              tempo_stream_t stream);
int tempo_nccl_unique_id(void* id128);
int tempo_nccl_comm_init(int32_t world, int32_t rank, const void* id128, void** comm);
int tempo_nccl_comm_destroy(void* comm);

int tempo_peer_alloc(size_t bytes, void** dev_ptr);
int tempo_peer_free(void* dev_ptr);
/* CUDA IPC plumbing for the inbox/flag buffers of other processes:
 * handle = 64 opaque bytes (cudaIpcMemHandle_t) of a tempo_peer_alloc
 * pointer. */
int tempo_ipc_get_handle(const void* dev_ptr, void* handle64);
int tempo_ipc_open_handle(const void* handle64, void** dev_ptr);
int tempo_ipc_close(void* dev_ptr);

/* ---------------------------------------------------------------------- */
/* Output-only softmax + Sub-Layer Dropout Recomputation                   */
/* (tempo_ops::softmax ops_tempo.cpp:158-166, dropout_recompute :168-194)   */
/* ---------------------------------------------------------------------- */
typedef enum {
    TEMPO_MASK_SUPPLIED = 0, /* mask is an input (e.g. the reference's
                                BoolMask::bernoulli_keep stream, packed)     */
    TEMPO_MASK_PHILOX = 1    /* mask is generated in-kernel (Philox4x32-10,
                                counter = global element index + offset) and
                                written: keep <=> u >= p, u = r * 2^-32       */
} tempo_mask_mode_t;

/* softmax_forward (ops_reference.cpp:104-125) alone. */
int tempo_softmax_ip_fwd(const float* z, float* P, int64_t rows, int64_t cols,
                         tempo_stream_t stream);
/* softmax_backward_from_output (ops_reference.cpp:127-145): dZ = P*(dP - sum dP*P). */
int tempo_softmax_ip_bwd(const float* dP, const float* P, float* dZ, int64_t rows, int64_t cols,
                         tempo_stream_t stream);
/* Fused forward: P = softmax(z) and D = dropout_apply(P, mask, p)
 * (ops_reference.cpp:147-153) in one pass; the stash is P + mask bits only.
 * `mask` is read (SUPPLIED) or written (PHILOX, with seed and
 * `offset` = global index of element 0, so row shards reproduce the
 * unsharded mask).  p not in [0,1) -> ParamError.  D may be NULL. */
int tempo_softmax_dropout_fwd(const float* z, double p, tempo_mask_mode_t mode, uint32_t* mask,
                              uint64_t seed, uint64_t offset, float* P, float* D, int64_t rows,
                              int64_t cols, tempo_stream_t stream);
/* Fused attention-probs backward: dropout_backward (ops_tempo.cpp:188-190),
 * softmax_backward_from_output on the stashed P, and optionally the
 * "dropout-rescale" recompute of D (ops_tempo.cpp:17-26, run by the
 * consumer at tape.cpp:255-260) written to D_out (NULL = skip) -- bitwise
 * equal to the forward D. */
int tempo_attn_probs_bwd(const float* dD, const float* P, const uint32_t* mask, double p,
                         float* dZ, float* D_out, int64_t rows, int64_t cols,
                         tempo_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Dropout with bit masks (dropout_apply / dropout_backward,               */
/* ops_reference.cpp:147-161; ref_ops::dropout :214-225)                   */
/* ---------------------------------------------------------------------- */
/* y = mask ? x*(1/(1-p)) : 0.  SUPPLIED reads mask, PHILOX writes it.
 * Also the recompute rule "dropout-rescale" (ops_tempo.cpp:17-26). */
int tempo_dropout_fwd(const float* x, double p, tempo_mask_mode_t mode, uint32_t* mask,
                      uint64_t seed, uint64_t offset, float* y, int64_t n, tempo_stream_t stream);
/* The recompute rule "dropout-rescale" (ops_tempo.cpp:17-26, run from the
 * consumer's BackwardCtx::stash, tape.cpp:244-264): D = mask ? P*(1/(1-p)) :
 * 0, bitwise the forward's D (the same kernel as tempo_dropout_fwd with a
 * SUPPLIED mask; the mask is only read). */
int tempo_dropout_recompute(const float* P, const uint32_t* mask, double p, float* D, int64_t n,
                            tempo_stream_t stream);
/* dx = mask ? dy*(1/(1-p)) : 0.  dx may alias dy. */
int tempo_dropout_bwd(const float* dy, const uint32_t* mask, double p, float* dx, int64_t n,
                      tempo_stream_t stream);

/* The dropout recompute fused into its consumer: the
 * attention-context GEMM's input gradient dV = D^T @ dO, per (batch, head),
 * where D' = keep ? P : 0 is rebuilt tile by tile by the GEMM's producer
 * warps from the stashed P and mask and written straight into tensor memory
 * as the MMA's A operand (1/(1-p) applied to the result) --
 * the consumer's BackwardCtx::stash of the "dropout-rescale" recipe
 * (graph.cpp:46-50, tape.cpp:244-264, ops_tempo.cpp:17-26) without D ever
 * reaching HBM.  P: [heads][s_q][s_k] (the softmax output, row = query),
 * mask: its bit-packed keep bits (global element order), dO: [heads][s_q][d],
 * dV: [heads][s_k][d]; fp32 in and out, computed on the tcgen05 tensor
 * cores in 3xTF32 (error within 2e-6 of |ref| + sum |D||dO| at any s_q:
 * the accumulation is drained into fp32 beyond s_q = 1024).  Pair with
 * tempo_attn_probs_bwd(..., D_out = NULL).  Needs s_q % 32 == 0,
 * s_k % 256 == 0, d in {32, 64, 128} (else TEMPO_ERR_UNSUPPORTED) and
 * 16-byte aligned P, dO, dV. */
int tempo_attn_dropout_dv(const float* P, const uint32_t* mask, double p, const float* dO,
                          float* dV, int64_t heads, int64_t s_q, int64_t s_k, int64_t d,
                          tempo_stream_t stream);
/* The FORWARD consumer of the recomputed map: ctx = D @ V per (batch, head),
 * D = keep ? P/(1-p) : 0 rebuilt inside a tcgen05 (3xTF32) GEMM from P and
 * the mask -- tempo_ops::sdpa's matmul(dropout_recompute(probs), v)
 * (ops_tempo.cpp:196-210) without D in HBM: pair with
 * tempo_softmax_dropout_fwd(..., D = NULL), so the forward writes P and the
 * bits only.  P: [heads][s_q][s_k], V: [heads][s_k][d], ctx: [heads][s_q][d],
 * fp32, error within 2e-6 of |ref| + sum |D||V| at any s_k.  Needs s_k % 32 == 0,
 * d in {32, 64} (else TEMPO_ERR_UNSUPPORTED), 16-byte aligned
 * P, V, ctx. */
int tempo_attn_dropout_ctx(const float* P, const uint32_t* mask, double p, const float* V,
                           float* ctx, int64_t heads, int64_t s_q, int64_t s_k, int64_t d,
                           tempo_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Hidden dropout -> residual add -> In-Place LayerNorm, fused             */
/* (the reference layer's ref_ops::dropout -> Graph::add ->                */
/*  tempo_ops::layernorm chain, encoder.cpp:180-191 and 198-210)            */
/* ---------------------------------------------------------------------- */
/* Forward: r = residual + (keep ? float(double(proj) / (1-p)) : 0), then the
 * in-place LayerNorm of r (y, rstd as tempo_ln_ip_fwd) -- bit-identical to
 * tempo_dropout_fwd, an fp32 add and tempo_ln_ip_fwd on the same inputs,
 * without storing the dropout output or r.  SUPPLIED reads `mask`, PHILOX
 * writes it (the same bits tempo_dropout_fwd generates for these global
 * element offsets).  cols % 32 == 0 (else TEMPO_ERR_UNSUPPORTED: use the
 * separate ops).  HBM: 12.125 B/element. */
int tempo_dropout_add_ln_fwd(const float* proj, const float* residual, double p,
                             tempo_mask_mode_t mode, uint32_t* mask, uint64_t seed,
                             uint64_t offset, const float* gamma, const float* beta, double eps,
                             float* y, float* rstd, int64_t rows, int64_t cols,
                             int32_t* dev_status, tempo_stream_t stream);
/* Backward: d_residual = the LayerNorm input gradient (tempo_ln_ip_bwd's dx;
 * the add passes it through to the residual branch) and d_proj = keep ?
 * float(double(d_residual) / (1-p)) : 0 (dropout_backward), in one pass;
 * dgamma/dbeta as tempo_ln_ip_bwd (same workspace query), summed over the
 * ranks of `peer` when it is non-NULL (as tempo_ln_ip_bwd_peer).  cols % 4
 * == 0.  HBM: 16.125 B/element. */
int tempo_dropout_add_ln_bwd(const float* dy, const float* y, const float* rstd,
                             const float* gamma, const float* beta, const uint32_t* mask,
                             double p, float* d_residual, float* d_proj, float* dgamma,
                             float* dbeta, void* workspace, size_t workspace_bytes, int64_t rows,
                             int64_t cols, const tempo_ln_peer_t* peer, tempo_stream_t stream);

/* out = float(double(a) * c): tempo::scale (kernels.cpp:209-213), used by
 * Graph::scale (the 1/sqrt(d) of tempo_ops::sdpa).  out may alias a. */
int tempo_tensor_scale(const float* a, double c, float* out, int64_t n, tempo_stream_t stream);

/* out = a + b elementwise: the gradient accumulation at fan-out of
 * Tape::backward (tape.cpp:225-226 via tempo::add, kernels.cpp:183-186).
 * out may alias a or b. */
int tempo_tensor_add(const float* a, const float* b, float* out, int64_t n,
                     tempo_stream_t stream);

/* ---------------------------------------------------------------------- */
/* Masks                                                                   */
/* ---------------------------------------------------------------------- */
/* BoolMask byte form <-> packed bits, on device.  pack refuses bytes > 1
 * like BoolMask::from_bytes (tensor.cpp:205-220) by writing TEMPO_ERR_PARAM
 * to dev_status (may be NULL). */
int tempo_mask_pack(const uint8_t* bytes, uint32_t* bits, int64_t n, int32_t* dev_status,
                    tempo_stream_t stream);
int tempo_mask_unpack(const uint32_t* bits, uint8_t* bytes, int64_t n, tempo_stream_t stream);
/* The reference's own mask stream, on the HOST, packed:
 * BoolMask::bernoulli_keep(shape, p, seed) (tensor.cpp:186-203 --
 * std::mt19937_64 + uniform_real_distribution<double>, keep <=> u >= p).
 * bits has ceil(n/32) words. */
int tempo_bernoulli_keep_bits_host(int64_t n, double p, uint64_t seed, uint32_t* bits);
/* The same stream generated ON THE DEVICE, bit for bit: the keep bits of
 * elements [offset, offset + n) of BoolMask::bernoulli_keep(shape, p, seed)
 * (for any shape with at least offset + n elements) into ceil(n/32) words at
 * `bits` (device).  The std::mt19937_64 stream is cut into 2^19-output
 * chunks whose states are reached by GF(2) jump-ahead (x^J mod the
 * characteristic polynomial); row shards pass their global offset.
 * offset % 32 != 0 or p not in [0,1) -> TEMPO_ERR_PARAM.  The workspace
 * (device, size from the query) holds the chunk states; the jump polynomials
 * are computed once per process (~1 s) and uploaded once per device. */
size_t tempo_bernoulli_keep_bits_workspace_size(uint64_t offset, int64_t n);
int tempo_bernoulli_keep_bits(int64_t n, double p, uint64_t seed, uint64_t offset,
                              uint32_t* bits, void* workspace, size_t workspace_bytes,
                              tempo_stream_t stream);
/* softmax -> dropout_recompute forward (as tempo_softmax_dropout_fwd) whose
 * mask is the reference's OWN stream: elements [offset, offset + rows*cols)
 * of BoolMask::bernoulli_keep(shape, p, seed), generated on the device INSIDE
 * the softmax kernel (warp-specialised: generator warps run the jumped chunk
 * recurrence, consumer warps the softmax rows) and written to `mask` (the
 * stash), bit-identical to tempo_bernoulli_keep_bits followed by the
 * supplied-mask forward -- which is what runs when the shape does not fit
 * the fused kernel (cols not in {128, 256, 512, 1024}, offset % 2^19 != 0 or
 * rows*cols % 8192 != 0).  Workspace: tempo_bernoulli_keep_bits_workspace_size(
 * offset, rows*cols).  offset % 32 != 0 -> TEMPO_ERR_PARAM. */
int tempo_softmax_dropout_fwd_refmask(const float* z, double p, uint64_t seed, uint64_t offset,
                                      uint32_t* mask, float* P, float* D, int64_t rows,
                                      int64_t cols, void* workspace, size_t workspace_bytes,
                                      tempo_stream_t stream);
/* Host reference of the jump construction (test helper): `count` outputs of
 * std::mt19937_64(seed) after discard(steps), via x^steps mod P.  0 = ok. */
int tempo_mt_outputs_after_host(uint64_t seed, uint64_t steps, int64_t count, uint64_t* out);
/* encoder::mask_stream_seed (encoder.cpp:39-46). */
uint64_t tempo_mask_stream_seed(uint64_t mask_seed, uint64_t salt, int site);

/* ---------------------------------------------------------------------- */
/* Stash accounting (memory_model.cpp:31-137; ledger semantics)            */
/* ---------------------------------------------------------------------- */
/* Bytes one BERT layer retains between forward and backward, per token.
 * mask_bits = 0: the reference's 1-byte masks (66H+13AS baseline,
 * 46H+5AS+8 Tempo); mask_bits = 1: this library's bit-packed masks.
 * tempo_variant = 0: baseline inventory, 1: all four Tempo optimizations. */
int64_t tempo_layer_stash_bytes_per_token(int64_t seq, int64_t hidden, int64_t heads,
                                          int tempo_variant, int mask_bits);

#ifdef __cplusplus
}
#endif

#endif /* TEMPO_B200_H */
