// ctx.cu — context, error word, thread-local error messages, RNG entry points.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>

#include "common.cuh"
#include "rng.cuh"

namespace qgnn_b200 {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

int status_from_exception() {
  try {
    throw;
  } catch (const Status& s) {
    g_last_error = s.what();
    return s.code;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return QGNN_EINVAL;
  } catch (const std::bad_alloc& e) {
    g_last_error = "out of host memory";
    return QGNN_ERESOURCE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return QGNN_EINVAL;
  } catch (...) {
    g_last_error = "unknown error";
    return QGNN_EINVAL;
  }
}

void* ctx_scratch(qgnn_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->scratch_bytes) return ctx->scratch;
  if (ctx->scratch) ctx->retired.push_back(ctx->scratch);
  ctx->scratch = nullptr;
  ctx->scratch_bytes = 0;
  QGNN_CUDA(cudaMalloc(&ctx->scratch, bytes));
  ctx->scratch_bytes = bytes;
  return ctx->scratch;
}

void* ctx_gemm_b(qgnn_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->gemm_b_bytes) return ctx->gemm_b;
  if (ctx->gemm_b) ctx->retired.push_back(ctx->gemm_b);
  ctx->gemm_b = nullptr;
  ctx->gemm_b_bytes = 0;
  QGNN_CUDA(cudaMalloc(&ctx->gemm_b, bytes));
  ctx->gemm_b_bytes = bytes;
  return ctx->gemm_b;
}

// tcgen05 GEMM unless QGNN_GEMM=simt (debug / A-B comparison switch)
bool use_tc_gemm() {
  static const bool tc = [] {
    const char* e = std::getenv("QGNN_GEMM");
    return !(e && std::string(e) == "simt");
  }();
  return tc;
}

// Maps a latched device error word onto the reference's exception taxonomy.
int status_from_error_word(int w, std::string& msg) {
  if (w & kErrNonFinite) {
    msg = "quantize: non-finite input";
    return QGNN_EINVAL;
  }
  if (w & kErrBadWidth) {
    msg = "quantize: bit width must be 2, 4, or 8";
    return QGNN_EINVAL;
  }
  if (w & kErrLabel) {
    msg = "loss: label out of range";
    return QGNN_EINVAL;
  }
  if (w & kErrMissing) {  // a missing payload also explains any decode error after it
    msg = "exchange: missing payload (peer-store flags not received in time)";
    return QGNN_EPROTOCOL;
  }
  if (w & kErrDecode) {
    msg = "message set: chunk disagrees with index";
    return QGNN_EDECODE;
  }
  if (w & kErrProtocol) {
    msg = "exchange: misrouted payload or plan version skew";
    return QGNN_EPROTOCOL;
  }
  return QGNN_OK;
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" {

const char* qgnn_last_error(void) { return g_last_error.c_str(); }
const char* qgnn_version(void) { return "qgnn_b200 0.1 (sm_100a)"; }

uint64_t qgnn_rng_seed_key(uint64_t seed) { return rng_seed_key(seed); }
uint64_t qgnn_rng_fork(uint64_t key, uint64_t coord) { return rng_fork(key, coord); }
uint64_t qgnn_rng_u64(uint64_t key, uint64_t counter) { return rng_u64(key, counter); }

int qgnn_ctx_create(int device, qgnn_ctx** out) {
  QGNN_API_BEGIN
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  QGNN_REQUIRE(e == cudaSuccess && count > 0, QGNN_ECUDA,
               "no CUDA device: the B200 path has no CPU fallback");
  QGNN_REQUIRE(device >= 0 && device < count, QGNN_EINVAL, "bad device ordinal");
  QGNN_CUDA(cudaSetDevice(device));
  auto* c = new qgnn_ctx;
  c->device = device;
  QGNN_CUDA(cudaMalloc(&c->d_err, sizeof(int)));
  QGNN_CUDA(cudaMemset(c->d_err, 0, sizeof(int)));
  QGNN_CUDA(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
  *out = c;
  QGNN_API_END
}

int qgnn_ctx_destroy(qgnn_ctx* ctx) {
  QGNN_API_BEGIN
  if (!ctx) return QGNN_OK;
  cudaSetDevice(ctx->device);
  if (ctx->d_err) cudaFree(ctx->d_err);
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->gemm_b) cudaFree(ctx->gemm_b);
  for (void* p : ctx->retired) cudaFree(p);
  delete ctx;
  QGNN_API_END
}

int qgnn_ctx_check(qgnn_ctx* ctx, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "null context");
  int w = 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  QGNN_CUDA(cudaMemcpyAsync(&w, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
  QGNN_CUDA(cudaStreamSynchronize(s));
  if (w) {
    QGNN_CUDA(cudaMemsetAsync(ctx->d_err, 0, sizeof(int), s));
    QGNN_CUDA(cudaStreamSynchronize(s));
    std::string msg;
    const int st = status_from_error_word(w, msg);
    throw Status(st, msg);
  }
  QGNN_API_END
}

}  // extern "C"
