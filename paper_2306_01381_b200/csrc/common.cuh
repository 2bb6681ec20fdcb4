// common.cuh — shared helpers for the sm_100a boundary-message kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "qgnn_b200.h"
#include "status.hpp"

namespace qgnn_b200 {

// Device error word bits (latched by kernels, read by qgnn_ctx_check).
enum : int {
  kErrNonFinite = 1,   // quantize: non-finite input       -> QGNN_EINVAL   (quant.hpp:64)
  kErrDecode = 2,      // chunk width/count/index mismatch -> QGNN_EDECODE  (codec.hpp:82-95)
  kErrBadWidth = 4,    // bit width not in {2,4,8}         -> QGNN_EINVAL   (quant.hpp:61)
  kErrLabel = 8,       // label out of range               -> QGNN_EINVAL   (model.hpp:185)
  kErrProtocol = 16,   // chunk envelope (source, target, plan version) differs from the
                       // receiver's expectation           -> QGNN_EPROTOCOL (engine.hpp:530-541)
  kErrMissing = 32,    // peer-store flag wait timed out: a payload never arrived
                       //                                  -> QGNN_EPROTOCOL (engine.hpp:530)
};

#define QGNN_CUDA(call)                                                                  \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::qgnn_b200::Status(QGNN_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Launch check: catches configuration errors synchronously.
inline void check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw Status(QGNN_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---- arithmetic policy ------------------------------------------------------
// F64 reproduces the reference's x86-64 arithmetic (mul rounded, then add
// rounded, no contraction); F32 is the production path and contracts.
template <typename T>
struct Arith;
template <>
struct Arith<double> {
  __device__ __forceinline__ static double madd(double a, double x, double acc) {
    return __dadd_rn(acc, __dmul_rn(a, x));
  }
  __device__ __forceinline__ static double mul(double a, double x) { return __dmul_rn(a, x); }
};
template <>
struct Arith<float> {
  __device__ __forceinline__ static float madd(float a, float x, float acc) {
    return fmaf(a, x, acc);
  }
  __device__ __forceinline__ static float mul(float a, float x) { return a * x; }
};

// ReLU-backward mask of the 4 columns [c, c + 4) of row r as bits 0..3: the
// activation row itself (ldm > 0 floats per row: h > 0) or 1[h > 0] bit words
// written by the forward GEMM epilogue (ldm < 0: -ldm 32-bit words per row, the
// pointer reinterpreted) -- 32 B instead of 1 KB per 256-wide row.
__device__ __forceinline__ uint32_t relu_bits4(const float* __restrict__ m, int64_t ldm, int64_t r,
                                               int64_t c) {
  if (ldm < 0)
    return (__ldg(reinterpret_cast<const uint32_t*>(m) + r * (-ldm) + (c >> 5)) >> (c & 31)) &
           0xfu;
  const float4 h = __ldg(reinterpret_cast<const float4*>(m + r * ldm + c));
  return (h.x > 0.f ? 1u : 0u) | (h.y > 0.f ? 2u : 0u) | (h.z > 0.f ? 4u : 0u) |
         (h.w > 0.f ? 8u : 0u);
}
__device__ __forceinline__ float4 apply_bits4(float4 v, uint32_t b) {
  return make_float4((b & 1u) ? v.x : 0.f, (b & 2u) ? v.y : 0.f, (b & 4u) ? v.z : 0.f,
                     (b & 8u) ? v.w : 0.f);
}

struct Ctx;  // defined in ctx.cu

// fp32 GPU-layout decode + scatter-add, ReLU-backward mask by h (codec.cu)
void dequant_add_masked_f32(qgnn_ctx* ctx, const uint8_t* in, int64_t n, int dim,
                            const uint8_t* bits, const uint64_t* offsets, const int32_t* dst_rows,
                            float* out, int64_t ld, const float* mask, int64_t ldm,
                            const uint32_t* expect, cudaStream_t s);
// fp32 input gradient out = A W^T for rows [row_begin, row_begin + n_rows) with the
// ReLU-backward mask by h folded into the epilogue (dense.cu); mbits (optional): the
// same mask as 1[h > 0] bit words written by dense_forward_bits_f32 (row pitch ldmb)
void input_grad_masked_f32(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int64_t din,
                           int64_t dout, int64_t row_begin, int64_t n_rows, float* out,
                           int64_t ldo, const float* mask, int64_t ldm, cudaStream_t s,
                           const uint32_t* mbits = nullptr, int64_t ldmb = 0);
// qgnn_dense_forward (fp32, ReLU) that also writes 1[out > 0] as 32-column bit words of
// each row (row pitch ldb words) when it runs on the tcgen05 path; false: no bits
bool dense_forward_bits_f32(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W,
                            int64_t din, int64_t dout, int64_t row_begin, int64_t n_rows,
                            float* out, int64_t ldo, uint32_t* bits, int64_t ldb, cudaStream_t s);
// backward scatter-add in one launch: destination rows with their incoming
// messages in ascending source order, decoded + summed per row (codec.cu)
// words (optional): chunk word of every entry (encode_chunk_words over msg), so an
// entry costs one load instead of message -> offset / width
void dequant_rows_add_f32(qgnn_ctx* ctx, const uint8_t* in, int64_t n_rows, const int32_t* rows,
                          const int32_t* ptr, const int32_t* msg, const int32_t* words, int dim,
                          const uint8_t* bits,
                          const uint64_t* offsets, float* out, int64_t ld, const float* mask,
                          int64_t ldm, const uint32_t* expect, cudaStream_t s);
// Adam with the bias corrections in device memory (captured epoch graphs, dense.cu)
void adam_step_devbc(int dtype, void* p, void* m, void* v, const void* g, int64_t n, double lr,
                     double beta1, double beta2, double eps, const double* bc, cudaStream_t s);
// fp32 loss phase for the engine: CE over train rows + val/test hit counts (dense.cu)
void loss_f32(qgnn_ctx* ctx, const float* logits, int64_t ld, int classes, const int32_t* labels,
              const int32_t* rows, int64_t n_train, int64_t n_val, int64_t n_test,
              double inv_denom, float* grad, int64_t ldg, double* loss_acc,
              unsigned long long* correct, cudaStream_t s);
}  // namespace qgnn_b200

struct qgnn_ctx {
  int device = 0;
  int* d_err = nullptr;          // device error word
  void* scratch = nullptr;       // split-K workspace
  size_t scratch_bytes = 0;
  void* gemm_b = nullptr;        // pre-split weight operand of the tcgen05 GEMM
  size_t gemm_b_bytes = 0;
  // outgrown workspaces, freed with the context: a cudaFree while kernels run would
  // synchronize the whole device (and deadlock peer-store ranks sharing one GPU)
  std::vector<void*> retired;
  int num_sms = 148;
  // Reuse of the pre-split weight operand across consecutive GEMMs with the same
  // weights (the P partitions of one layer).  Opt-in: an owner that knows when its
  // weights change (the engine: Adam step, set_weights) sets b_reuse and bumps
  // wgen on every change; plain C-ABI callers always re-split.
  bool b_reuse = false;
  uint64_t wgen = 0;
  int last_gemm_launches = 0;  // kernels the last tc_gemm_rows call launched (1 or 2)
  struct {
    const void* W = nullptr;
    const void* buf = nullptr;
    int wcols = 0, N = 0, K = 0, transpose = -1;
    uint64_t gen = ~uint64_t{0};
  } bprep;
};

namespace qgnn_b200 {
// Grows ctx->scratch to at least `bytes` (synchronous; call outside capture).
void* ctx_scratch(qgnn_ctx* ctx, size_t bytes);
void* ctx_gemm_b(qgnn_ctx* ctx, size_t bytes);
// tcgen05 GEMMs (gemm_tc.cu)
// bits_out: with relu, 1[out > 0] of every output row as 32-column words (row pitch
// ldbo words); bits_in: ReLU-backward mask given as such words instead of `mask`
void tc_gemm_rows(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int wcols, int N,
                  int K, int transpose_w, int64_t n_rows, int relu, float* out, int64_t ldo,
                  cudaStream_t s, const float* mask = nullptr, int64_t ldm = 0,
                  uint32_t* bits_out = nullptr, int64_t ldbo = 0,
                  const uint32_t* bits_in = nullptr, int64_t ldbi = 0);
float* tc_gemm_wgrad_partials(qgnn_ctx* ctx, const float* A, int64_t lda, const float* B,
                              int64_t ldb, int M, int N, int64_t n_rows, int* splits_out,
                              cudaStream_t s);
bool use_tc_gemm();
// Hub rows of one SpMM call site, split into 256-edge segments (device arrays).
struct HubPlan {
  int64_t hub_deg = 0;        // rows with more neighbours than this are hubs
  int64_t n_hubs = 0, n_segs = 0;
  const int32_t* hubs = nullptr;     // [n_hubs] rows
  const int32_t* seg_ptr = nullptr;  // [n_hubs + 1] segment range per hub
  const int64_t* seg = nullptr;      // [n_segs][4] = a_begin, a_end, b_begin, b_end
  float* part = nullptr;             // [n_segs][ldp] partial rows (workspace)
  int64_t ldp = 0;
  const int32_t* order = nullptr;    // [n_order] non-hub rows of the range, degree-descending
  int64_t n_order = 0;
  // in-kernel hub reduction: the last segment of a hub to finish reduces it
  const int32_t* seg_hub = nullptr;  // [n_segs] hub index of each segment
  int32_t* cnt = nullptr;            // [n_hubs] arrivals; zero between launches
  double avg_deg = 0;                // mean (a + b) degree of the range's rows
};
// Per-row activation chain with LayerNorm / dropout (chain.cu; model.hpp:62-153)
struct ChainArgs {
  int ln = 0;                 // layer_norm
  int relu = 0;               // Activation::kRelu
  double keep = 1.0;          // 1 - dropout (1: no dropout on this layer)
  uint64_t keep_thr = 0;      // ceil(keep * 2^53): draw >> 11 below it keeps the element
  const uint64_t* drop_key = nullptr;  // [dev] RngStream key of fork({0x4, epoch, l, device})
  const int32_t* ref_row = nullptr;    // GPU row -> reference owned-row index
};

template <typename T>
void chain_forward(const T* z, T* act, int64_t ld, T* h, int64_t ldh, T* inv_std, int dout,
                   int64_t r0, int64_t n, const ChainArgs& c, cudaStream_t s);
template <typename T>
void chain_backward(const T* dh, int64_t lddh, const T* act, int64_t ld, const T* h, int64_t ldh,
                    const T* inv_std, T* dz, int64_t lddz, int dout, int64_t r0, int64_t n,
                    const ChainArgs& c, cudaStream_t s);

// Forward halo rows read straight from the exchange arena:
// remote slot s is message s of the receive list, its chunk at arena + off[s]
// with width bits[s]; the marginal SpMM dequantizes the 8 columns a lane needs
// in registers (code * S + Z, the value K3 would have stored) instead of
// reading a materialised fp32 halo row.  Headers are checked like K3 (width,
// count -> kErrDecode; envelope env[s] -> kErrProtocol).
struct PackedHalo {
  const uint8_t* arena = nullptr;
  const uint64_t* off = nullptr;
  const uint8_t* bits = nullptr;
  const uint32_t* env = nullptr;
  int dim = 0;
  int* err = nullptr;
  // direct: the b-range column entries are chunk words (offset / 16 in bits 0..29,
  // width code 0 / 2 / 4 / 8 -> 0..3 in bits 30..31; encode_chunk_words) instead of
  // slot indices, so a gather reaches its chunk in one dependent round trip; the
  // headers are validated once per message by check_chunk_headers instead
  bool direct = false;
};
// chunk words of the packed-halo gathers: out[e] = word of message idx[e] (engine.cu)
void encode_chunk_words(const int32_t* idx, int64_t n, const uint64_t* off, const uint8_t* bits,
                        int32_t* out, cudaStream_t s);
// header checks of n received chunks (width, count, envelope) -> DecodeError /
// ProtocolError in the error word, once per message (codec.hpp:82-95, engine.hpp:530-541)
void check_chunk_headers(const uint8_t* arena, const uint64_t* off, const uint8_t* bits,
                         const uint32_t* env, int64_t n, int dim, int* err, cudaStream_t s);
// fp32 row-range SpMM with segmented hub rows (spmm.cu)
// returns the number of kernels launched.  pk != nullptr: the b range (remote
// CSR) gathers from the packed arena instead of y (spmm_packed_ok must hold).
int spmm_f32(qgnn_ctx* ctx, int dim, const float* x, int64_t ldx, const float* y, int64_t ldy,
              const float* sa, const int64_t* pa, const int32_t* ca, const float* aa,
              const int64_t* pb, const int32_t* cb, const float* ab, int64_t row_begin,
              int64_t n_rows, float* out, int64_t ldo, const HubPlan* hp, cudaStream_t s,
              const float* mask = nullptr, int64_t ldm = 0, const PackedHalo* pk = nullptr);
// whether spmm_f32 runs this range through a kernel with a packed-halo variant
// (the grouped <= 128-wide and the 256-wide row kernels, 32-byte aligned rows)
bool spmm_packed_ok(int dim, const HubPlan* hp, const float* x, int64_t ldx);
}  // namespace qgnn_b200
