// chain.cu — the per-row activation chain of a layer when LayerNorm and/or
// dropout are on (model.hpp:62-153; TrainSettings::layer_norm / dropout,
// engine.hpp:42-43, 574-578, 600):
//
//   forward   z = h_agg W  ->  y = LN(z) (if layer_norm)  ->  a = act(y)
//             ->  h = a * mask (hidden layers, if dropout)
//   backward  tmp = dh * mask  ->  tmp = 0 where act_in <= 0 (ReLU)
//             ->  dz = LN'(tmp) (if layer_norm)
//
// act_in (y with LN, else z) and inv_std are kept from the forward pass.  The
// dropout mask is a pure function of the reference's coordinates: row r (the
// reference's owned-row index) of device d at layer l and epoch e draws
// RngStream(seed).fork({0x4, e, l, d}).fork(r), element j its (j+1)-th double
// (engine.hpp:600, model.hpp:114-119); keep iff u < 1 - dropout, i.e.
// (draw >> 11) < ceil((1 - dropout) 2^53) exactly.  Backward needs no draws:
// h > 0 <=> (act_in > 0 and the element was kept), so tmp = h > 0 ? dh / keep : 0.
//
// f64: one thread per row in the reference's exact order (sequential sums,
// no contraction) -- bit-identical to model.hpp.  f32: one warp per row,
// warp-shuffle sums.
#include <cuda_runtime.h>

#include "common.cuh"
#include "rng.cuh"

namespace qgnn_b200 {

// ---- f64: the reference's exact sequence -------------------------------------------------
// z and act may be the same buffer (LN in place; act_in = z without LN)
__global__ void k_chain_fwd_f64(const double* z, double* act,
                                int64_t ld, double* __restrict__ h, int64_t ldh,
                                double* __restrict__ inv_std, int dout, int64_t r0, int64_t n,
                                ChainArgs c) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = r0 + i;
  const double* zr = z + r * ld;
  double* ar = act + r * ld;
  double* hr = h + r * ldh;
  if (c.ln) {  // detail::layer_norm_row (model.hpp:62-73)
    double mean = 0.0;
    for (int j = 0; j < dout; ++j) mean = __dadd_rn(mean, zr[j]);
    mean = __ddiv_rn(mean, double(dout));
    double var = 0.0;
    for (int j = 0; j < dout; ++j) {
      const double d = __dsub_rn(zr[j], mean);
      var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, double(dout));
    const double is = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, 1e-6)));
    inv_std[r] = is;
    for (int j = 0; j < dout; ++j) ar[j] = __dmul_rn(__dsub_rn(zr[j], mean), is);
  } else if (ar != zr) {
    for (int j = 0; j < dout; ++j) ar[j] = zr[j];
  }
  const bool drop = c.keep < 1.0;
  const uint64_t key = drop ? rng_fork(*c.drop_key, uint64_t(c.ref_row[r])) : 0;
  const double scale = 1.0 / c.keep;
  for (int j = 0; j < dout; ++j) {
    double o = ar[j];
    if (c.relu) o = 0.0 < o ? o : 0.0;  // std::max(0.0, src)
    if (drop) {
      const double m = (rng_u64(key, uint64_t(j) + 1) >> 11) < c.keep_thr ? scale : 0.0;
      o = __dmul_rn(o, m);
    }
    hr[j] = o;
  }
}

__global__ void k_chain_bwd_f64(const double* __restrict__ dh, int64_t lddh,
                                const double* __restrict__ act, int64_t ld,
                                const double* __restrict__ h, int64_t ldh,
                                const double* __restrict__ inv_std, double* __restrict__ dz,
                                int64_t lddz, int dout, int64_t r0, int64_t n, ChainArgs c) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t r = r0 + i;
  const double* g = dh + r * lddh;
  const double* y = act + r * ld;
  const double* hr = h + r * ldh;
  double* o = dz + r * lddz;
  const bool drop = c.keep < 1.0;
  const double scale = 1.0 / c.keep;
  // layer_backward_rows (model.hpp:128-153): tmp = dh * mask, ReLU zeroes act_in <= 0
  for (int j = 0; j < dout; ++j) {
    double t = g[j];
    if (drop) t = __dmul_rn(t, hr[j] != 0.0 || (!c.relu && y[j] != 0.0) ? scale : 0.0);
    if (c.relu && !(y[j] > 0.0)) t = 0.0;
    o[j] = t;
  }
  if (!c.ln) return;
  double mdy = 0.0, mdyy = 0.0;  // detail::layer_norm_row_backward (model.hpp:76-86)
  for (int j = 0; j < dout; ++j) {
    mdy = __dadd_rn(mdy, o[j]);
    mdyy = __dadd_rn(mdyy, __dmul_rn(o[j], y[j]));
  }
  mdy = __ddiv_rn(mdy, double(dout));
  mdyy = __ddiv_rn(mdyy, double(dout));
  const double is = inv_std[r];
  for (int j = 0; j < dout; ++j)
    o[j] = __dmul_rn(is, __dsub_rn(__dsub_rn(o[j], mdy), __dmul_rn(y[j], mdyy)));
}

// ---- f32: warp per row ------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(256) k_chain_fwd_f32(const float* z, float* act, int64_t ld,
                                                       float* __restrict__ h, int64_t ldh,
                                                       float* __restrict__ inv_std, int dout,
                                                       int64_t r0, int64_t n, ChainArgs c) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t r = r0 + i;
  const float* zr = z + r * ld;
  float* ar = act + r * ld;
  float* hr = h + r * ldh;
  float mean = 0.f, is = 1.f;
  if (c.ln) {
    float s = 0.f;
    for (int j = lane; j < dout; j += 32) s += zr[j];
    mean = warp_sum(s) / float(dout);
    float v = 0.f;
    for (int j = lane; j < dout; j += 32) {
      const float d = zr[j] - mean;
      v = fmaf(d, d, v);
    }
    is = rsqrtf(warp_sum(v) / float(dout) + 1e-6f);
    if (lane == 0) inv_std[r] = is;
  }
  const bool drop = c.keep < 1.0;
  const uint64_t key = drop ? rng_fork(*c.drop_key, uint64_t(c.ref_row[r])) : 0;
  const float scale = float(1.0 / c.keep);
  for (int j = lane; j < dout; j += 32) {
    const float y = c.ln ? (zr[j] - mean) * is : zr[j];
    if (c.ln || ar != zr) ar[j] = y;
    float o = c.relu ? (0.f < y ? y : 0.f) : y;
    if (drop) o *= (rng_u64(key, uint64_t(j) + 1) >> 11) < c.keep_thr ? scale : 0.f;
    hr[j] = o;
  }
}

__global__ void __launch_bounds__(256) k_chain_bwd_f32(const float* __restrict__ dh, int64_t lddh,
                                                       const float* __restrict__ act, int64_t ld,
                                                       const float* __restrict__ h, int64_t ldh,
                                                       const float* __restrict__ inv_std,
                                                       float* __restrict__ dz, int64_t lddz,
                                                       int dout, int64_t r0, int64_t n,
                                                       ChainArgs c) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int64_t r = r0 + i;
  const float* g = dh + r * lddh;
  const float* y = act + r * ld;
  const float* hr = h + r * ldh;
  float* o = dz + r * lddz;
  const bool drop = c.keep < 1.0;
  const float scale = float(1.0 / c.keep);
  float sdy = 0.f, sdyy = 0.f;
  for (int j = lane; j < dout; j += 32) {
    float t = g[j];
    if (drop) t *= hr[j] != 0.f || (!c.relu && y[j] != 0.f) ? scale : 0.f;
    if (c.relu && !(y[j] > 0.f)) t = 0.f;
    o[j] = t;
    sdy += t;
    sdyy = fmaf(t, y[j], sdyy);
  }
  if (!c.ln) return;
  const float mdy = warp_sum(sdy) / float(dout), mdyy = warp_sum(sdyy) / float(dout);
  const float is = inv_std[r];
  for (int j = lane; j < dout; j += 32) o[j] = is * (o[j] - mdy - y[j] * mdyy);
}

template <typename T>
void chain_forward(const T* z, T* act, int64_t ld, T* h, int64_t ldh, T* inv_std, int dout,
                   int64_t r0, int64_t n, const ChainArgs& c, cudaStream_t s) {
  if (n <= 0) return;
  if constexpr (sizeof(T) == 8)
    k_chain_fwd_f64<<<unsigned(ceil_div(n, 128)), 128, 0, s>>>(z, act, ld, h, ldh, inv_std, dout,
                                                                r0, n, c);
  else
    k_chain_fwd_f32<<<unsigned(ceil_div(n * 32, 256)), 256, 0, s>>>(z, act, ld, h, ldh, inv_std,
                                                                     dout, r0, n, c);
  check_launch("chain_forward");
}

template <typename T>
void chain_backward(const T* dh, int64_t lddh, const T* act, int64_t ld, const T* h, int64_t ldh,
                    const T* inv_std, T* dz, int64_t lddz, int dout, int64_t r0, int64_t n,
                    const ChainArgs& c, cudaStream_t s) {
  if (n <= 0) return;
  if constexpr (sizeof(T) == 8)
    k_chain_bwd_f64<<<unsigned(ceil_div(n, 128)), 128, 0, s>>>(dh, lddh, act, ld, h, ldh, inv_std,
                                                                dz, lddz, dout, r0, n, c);
  else
    k_chain_bwd_f32<<<unsigned(ceil_div(n * 32, 256)), 256, 0, s>>>(dh, lddh, act, ld, h, ldh,
                                                                     inv_std, dz, lddz, dout, r0,
                                                                     n, c);
  check_launch("chain_backward");
}

template void chain_forward<float>(const float*, float*, int64_t, float*, int64_t, float*, int,
                                   int64_t, int64_t, const ChainArgs&, cudaStream_t);
template void chain_forward<double>(const double*, double*, int64_t, double*, int64_t, double*,
                                    int, int64_t, int64_t, const ChainArgs&, cudaStream_t);
template void chain_backward<float>(const float*, int64_t, const float*, int64_t, const float*,
                                    int64_t, const float*, float*, int64_t, int, int64_t, int64_t,
                                    const ChainArgs&, cudaStream_t);
template void chain_backward<double>(const double*, int64_t, const double*, int64_t,
                                     const double*, int64_t, const double*, double*, int64_t, int,
                                     int64_t, int64_t, const ChainArgs&, cudaStream_t);

}  // namespace qgnn_b200
