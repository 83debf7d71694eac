// tempo_internal.h -- host/device shared definitions of the Tempo B200 library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#ifndef TM_PDL
#define TM_PDL 1
#endif

#include "../../include/tempo_b200.h"

namespace tb {

// ---- GELU table, device form -------------------------------------------
// Host-precomputed from the parsed v1 table (gelu_table.cpp) so that every
// double comparison of GeluPolyTable::eval becomes an fp32 comparison with
// the same outcome for every float input (hard part 2):
//   y < y_min      <=>  y_f < ymin_up      (ymin_up = smallest float >= y_min)
//   lo <= y        <=>  y_f >= lo_up       (lo_up   = smallest float >= lo)
//   x > x_star     <=>  x_f >= xstar_gt    (xstar_gt = smallest float > x_star)
constexpr int kMaxSeg = 32;   // total over both branches
constexpr int kMaxCoef = 64;  // gelu_table.cpp:123 allows up to 64

struct GeluDevTable {
    float xstar_gt;
    float ymin_up;
    float ymin_hi, ymin_lo;  // y_min as a float-float pair
    int nseg[2];             // branch 0 segments are [0, nseg0), branch 1 follow
    int ncoef;               // max coefficient count over all segments
    int stride;              // odd smem stride >= ncoef (bank-conflict free)
    float lo_up[kMaxSeg];
    float s[kMaxSeg];  // t = clamp(u * s + b, -1, 1); constant segments: s = b = 0
    float b[kMaxSeg];
    int sqrt_shift[kMaxSeg];
    float coef[kMaxSeg][kMaxCoef];  // Chebyshev coefficients, zero padded
    // Specialized kernel only: the same polynomials in the power basis of
    // v = u - u0 (u0 the segment's midpoint, t = s * v), i.e. coefficients
    // a_k * s^k of the power basis a_k in t (host fp64 conversion), used with
    // Horner's rule when `horner` is set (the conversion's error bound is
    // small enough, see capi.cpp).  No (s, b) and no clamp: the segment
    // search keeps v inside the segment, y < y_min is clamped on y.
    int horner;
    float monov[kMaxSeg][16];
    float u0[kMaxSeg];
};

// Kernel launchers (defined in the .cu files; return cudaGetLastError()).
// reference-exact forward: the fp64 formula for every element
cudaError_t launch_gelu_fwd_exact(const float* x, float* y, uint32_t* mask, int64_t n,
                                  float xstar_gt, cudaStream_t st);
cudaError_t launch_gelu_fwd(const float* x, float* y, uint32_t* mask, int64_t n, float xstar_gt,
                            cudaStream_t st);
cudaError_t launch_gelu_bwd(const float* dy, const float* y, const uint32_t* mask,
                            const GeluDevTable& t, float* dx, int64_t n, cudaStream_t st);

cudaError_t launch_ln_fwd(const float* x, const float* gamma, const float* beta, double eps,
                          float* y, float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                          cudaStream_t st);
size_t ln_bwd_workspace(int64_t rows, int64_t cols);
// The cross-rank exchange fused into stage 2 (layernorm_kernels.cu): every
// rank's inbox / flag buffers, mapped into this process (P2P / IPC).
struct LnPeer {
    int rank, world;
    double* const* inbox;     // device array [world]: rank p's inbox
    uint32_t* const* flags;   // device array [world]: rank p's flags
    uint32_t epoch;           // 1, 2, 3, ... per exchange
    int32_t* status;          // device int: TEMPO_ERR_STATE if a peer never arrived (sticky)
    uint32_t timeout_ms;      // bound on the wait for peers; 0 = library default (30 s)
};
size_t ln_peer_inbox_bytes(int world, int64_t cols);
size_t ln_peer_flag_bytes(int world, int64_t cols);
cudaError_t launch_ln_param_reduce_peer(const double* partials, int64_t nparts, int64_t cols,
                                        const LnPeer& peer, float* dgamma, float* dbeta,
                                        cudaStream_t st);
// nparts_out != nullptr: stage 1 only -- the fp64 partial rows stay in ws
// ([nparts][2*cols]: dgamma partials, then dbeta) and their count is returned
cudaError_t launch_ln_bwd(const float* dy, const float* y, const float* rstd, const float* gamma,
                          const float* beta, float* dx, float* dgamma, float* dbeta, void* ws,
                          int64_t rows, int64_t cols, cudaStream_t st,
                          const LnPeer* peer = nullptr, const uint32_t* mask = nullptr,
                          double scale = 1.0, float* dproj = nullptr,
                          int64_t* nparts_out = nullptr);
// stage 2 alone: dgamma/dbeta = the fixed-order sum of nparts partial rows
cudaError_t launch_ln_param_reduce(const double* partials, int64_t nparts, int64_t cols,
                                   float* dgamma, float* dbeta, cudaStream_t st);
// hidden dropout -> residual add -> LayerNorm forward, fused (cols % 32 == 0)
cudaError_t launch_dal_fwd(const float* proj, const float* res, double scale, uint64_t thresh,
                           int philox, uint32_t* mask, uint64_t seed, uint64_t offset,
                           const float* gamma, const float* beta, double eps, float* y,
                           float* rstd, int64_t rows, int64_t cols, int32_t* dev_status,
                           cudaStream_t st);

cudaError_t launch_softmax_fwd(const float* z, float* P, int64_t rows, int64_t cols,
                               cudaStream_t st);
cudaError_t launch_softmax_bwd(const float* dP, const float* P, float* dZ, int64_t rows,
                               int64_t cols, cudaStream_t st);
cudaError_t launch_softmax_dropout_fwd(const float* z, double scale, uint64_t thresh, int philox,
                                       uint32_t* mask, uint64_t seed, uint64_t offset, float* P,
                                       float* D, int64_t rows, int64_t cols, cudaStream_t st);
cudaError_t launch_attn_probs_bwd(const float* dD, const float* P, const uint32_t* mask,
                                  double scale, float* dZ, float* D, int64_t rows, int64_t cols,
                                  cudaStream_t st);

// dV = D^T dO with D rebuilt from P and the mask in the GEMM's operand
// staging (dv_gemm_kernels.cu; tcgen05, 3xTF32)
bool dv_gemm_supported(int64_t s_q, int64_t s_k, int64_t d);
// the forward consumer: ctx = dropout(P) @ V, D rebuilt inside the tcgen05 GEMM
bool ctx_gemm_supported(int64_t s_q, int64_t s_k, int64_t d);
cudaError_t launch_ctx_recompute_gemm(const float* P, const uint32_t* mask, double scale,
                                      const float* V, float* ctx, int64_t heads, int64_t s_q,
                                      int64_t s_k, int64_t d, cudaStream_t st);
cudaError_t launch_dv_recompute_gemm(const float* P, const uint32_t* mask, double scale,
                                     const float* dO, float* dV, int64_t heads, int64_t s_q,
                                     int64_t s_k, int64_t d, cudaStream_t st);

cudaError_t launch_dropout_fwd(const float* x, double scale, uint64_t thresh, int philox,
                               uint32_t* mask, uint64_t seed, uint64_t offset, float* y, int64_t n,
                               cudaStream_t st);
cudaError_t launch_dropout_bwd(const float* dy, const uint32_t* mask, double scale, float* dx,
                               int64_t n, cudaStream_t st);
cudaError_t launch_mask_pack(const uint8_t* bytes, uint32_t* bits, int64_t n, int32_t* status,
                             cudaStream_t st);
cudaError_t launch_mask_unpack(const uint32_t* bits, uint8_t* bytes, int64_t n, cudaStream_t st);
cudaError_t launch_scale(const float* a, double c, float* out, int64_t n, cudaStream_t st);
cudaError_t launch_add(const float* a, const float* b, float* out, int64_t n, cudaStream_t st);

// Launch `kernel` as a programmatic dependent of the previous work on the
// stream (PDL, cudaLaunchAttributeProgrammaticStreamSerialization): its
// launch overlaps the predecessor's tail; the kernel itself must call
// grid_dep_wait() before reading the predecessor's outputs.
template <typename... Args>
cudaError_t launch_pdl(const void* kernel, int grid, int block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* argv[] = {(void*)&args...};
    return cudaLaunchKernelExC(&cfg, kernel, argv);
}

// The reference's mask stream (std::mt19937_64, tensor.cpp:186-203) on the
// device: keep bits of elements [e_begin, e_begin + n), e_begin % 32 == 0.
size_t mt_keep_workspace(uint64_t e_begin, int64_t n);
// The chunk start states (kMtN words each) of the chunks covering elements
// [e_begin, e_begin + n) of the stream, computed into the workspace
// (mt_keep_workspace bytes); *states = chunk e_begin / kMtChunk's state.
cudaError_t launch_mt_chunk_states(uint64_t seed, uint64_t e_begin, int64_t n, void* ws,
                                   size_t ws_bytes, const uint64_t** states, cudaStream_t st);
// Softmax + dropout forward with the reference's mask stream generated inside
// the kernel (softmax_kernels.cu); falls back to launch_mt_keep_bits + the
// supplied-mask forward when the shape does not fit the fused kernel.
cudaError_t launch_softmax_dropout_fwd_mt(const float* z, double p, uint64_t seed,
                                          uint64_t e_begin, uint32_t* mask, float* P, float* D,
                                          int64_t rows, int64_t cols, void* ws, size_t ws_bytes,
                                          cudaStream_t st);
cudaError_t launch_mt_keep_bits(uint64_t seed, double p, uint64_t e_begin, int64_t n,
                                uint32_t* mask, void* ws, size_t ws_bytes, cudaStream_t st);

// Type-checked launch: launch(kernel, grid, block, smem, stream)(args...) is
// `kernel<<<grid, block, smem, stream>>>(args...)`, with programmatic stream
// serialization when TM_PDL=1 (default).  Every kernel of this library
// starts with grid_dep_wait() (before any global access), which makes PDL
// safe after any predecessor.  Measured on the bench chain: with every kernel
// triggering its dependents at its start it LOST 7-10 % (2.05 -> 2.20 ms:
// the dependents' early CTAs take the slots of the later waves of the
// multi-wave row kernels); with the trigger only in the single-wave
// persistent kernels (grid_dep_launch_persistent) and implicit at exit
// elsewhere it WINS 1.4 % (2.048 -> 2.021 ms/step: launch gaps hidden).
template <typename... KArgs>
struct Launch {
    void (*kernel)(KArgs...);
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute attr[2];
    unsigned nattr = 1;
    // thread-block clusters of k CTAs along x (grid.x % k == 0)
    Launch& cluster(unsigned k) {
        attr[nattr].id = cudaLaunchAttributeClusterDimension;
        attr[nattr].val.clusterDim.x = k;
        attr[nattr].val.clusterDim.y = 1;
        attr[nattr].val.clusterDim.z = 1;
        ++nattr;
        return *this;
    }
    template <typename... A>
    cudaError_t operator()(A&&... a) {
        cfg.attrs = attr;
        cfg.numAttrs = nattr;
        return cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(a)...);
    }
};
template <typename... KArgs>
Launch<KArgs...> launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                        cudaStream_t st) {
    Launch<KArgs...> L;
    L.kernel = kernel;
    L.cfg = cudaLaunchConfig_t{};
    L.cfg.gridDim = grid;
    L.cfg.blockDim = block;
    L.cfg.dynamicSmemBytes = smem;
    L.cfg.stream = st;
    L.attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    L.attr[0].val.programmaticStreamSerializationAllowed = TM_PDL;
    return L;
}

// Persistent-grid sizing: SM count x resident CTAs per SM (cached per device).
// cap_per_sm > 0 limits the CTAs per SM (fewer, longer-lived CTAs); waves > 1
// launches that many resident-capacity waves (CTAs that finish early are
// replaced by fresh ones: load balance for loops without prefetch).
int grid_for(const void* kernel, int block, size_t smem, int64_t work_items, int cap_per_sm = 0,
             int waves = 1);

}  // namespace tb
