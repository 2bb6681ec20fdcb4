// dense.cu — K5 dense transform and the per-epoch elementwise kernels.
//
// F32 (production): a shared-memory tiled SIMT GEMM (128x64x16 tiles, 8x4
// outputs per thread) with fused ReLU epilogue, a transposed-B variant for
// input gradients and a deterministic split-K weight-gradient GEMM whose
// partial tiles are reduced in fixed order.
// F64 (parity): one thread per output element summing in the reference's
// loop order with explicit round-to-nearest mul/add (model.hpp:90-170,
// matrix.hpp:51-65), so results are bit-identical to the CPU reference.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"

namespace qgnn_b200 {

// --------------------------------------------------------------- SIMT F32 ---
constexpr int BM = 128, BN = 64, BK = 16;

// C[M x N] = Aop[M x K] * Bop[K x N]
//  TA = false: Aop(i, k) = A[row(i) * lda + k]        row(i) = rows ? rows[i] : rb + i
//  TA = true : Aop(i, k) = A[row(k) * lda + i]        (weight grad: K runs over rows)
//  TB = false: Bop(k, j) = B[rowb(k) * ldb + j]       rowb(k) = TA ? row(k) : k
//  TB = true : Bop(k, j) = B[j * ldb + k]             (input grad: W^T)
// split-K over gridDim.z writes partial tiles to C + z * M * N (ldc = N).
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) k_sgemm(int M, int N, int K, const float* __restrict__ A,
                                               int64_t lda, const float* __restrict__ B,
                                               int64_t ldb, const int32_t* __restrict__ rows,
                                               int64_t rb, float* __restrict__ C, int64_t ldc,
                                               const int32_t* __restrict__ out_rows,
                                               int64_t out_rb, int relu, int k_per_split) {
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15;  // N direction: 4 columns each
  const int ty = tid >> 4;  // M direction: 8 rows each
  const int m0 = blockIdx.x * BM;
  const int n0 = blockIdx.y * BN;
  const int kz0 = blockIdx.z * k_per_split;
  const int kz1 = min(K, kz0 + k_per_split);

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k0 = kz0; k0 < kz1; k0 += BK) {
    // ---- A tile -> As[k][i]
    if (!TA) {
      // 128 rows x 16 k: thread loads 8 elements, k fastest
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int idx = tid + t * 256;
        const int i = idx >> 4, k = idx & 15;
        const int gm = m0 + i, gk = k0 + k;
        float v = 0.f;
        if (gm < M && gk < kz1) {
          const int64_t r = rows ? rows[gm] : rb + gm;
          v = __ldg(A + r * lda + gk);
        }
        As[k][i] = v;
      }
    } else {
      // 16 k(rows) x 128 i: i fastest
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int idx = tid + t * 256;
        const int k = idx >> 7, i = idx & 127;
        const int gm = m0 + i, gk = k0 + k;
        float v = 0.f;
        if (gm < M && gk < kz1) {
          const int64_t r = rows ? rows[gk] : rb + gk;
          v = __ldg(A + r * lda + gm);
        }
        As[k][i] = v;
      }
    }
    // ---- B tile -> Bs[k][j]
    if (!TB) {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int idx = tid + t * 256;
        const int k = idx >> 6, j = idx & 63;
        const int gk = k0 + k, gn = n0 + j;
        float v = 0.f;
        if (gk < kz1 && gn < N) {
          const int64_t r = TA ? (rows ? rows[gk] : rb + gk) : gk;
          v = __ldg(B + r * ldb + gn);
        }
        Bs[k][j] = v;
      }
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int idx = tid + t * 256;
        const int j = idx >> 4, k = idx & 15;
        const int gk = k0 + k, gn = n0 + j;
        float v = 0.f;
        if (gk < kz1 && gn < N) v = __ldg(B + static_cast<int64_t>(gn) * ldb + gk);
        Bs[k][j] = v;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[k][ty * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[k][ty * 8 + 4]);
      const float4 bv = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[4] = {bv.x, bv.y, bv.z, bv.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* Cz = C + static_cast<int64_t>(blockIdx.z) * (TA ? static_cast<int64_t>(M) * N : 0);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int gm = m0 + ty * 8 + i;
    if (gm >= M) continue;
    const int64_t orow = TA ? gm : (out_rows ? out_rows[gm] : out_rb + gm);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float v = acc[i][j];
      if (relu) v = v > 0.f ? v : 0.f;
      Cz[orow * ldc + gn] = v;
    }
  }
}

// out[i] (+)= sum_z part[z][i], fixed z order
__global__ void k_splitk_reduce(const float* __restrict__ part, int splits, int64_t mn,
                                float* __restrict__ out, int accumulate) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= mn) return;
  // the adds stay in z order (bit-identical); unrolling keeps 8 loads in flight
  float s = 0.f;
  int z = 0;
  for (; z + 8 <= splits; z += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcs(part + static_cast<int64_t>(z + j) * mn + i);
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; z < splits; ++z) s += __ldcs(part + static_cast<int64_t>(z) * mn + i);
  out[i] = accumulate ? out[i] + s : s;
}

// --------------------------------------------------------------- exact F64 ---
// model.hpp:95-113: z_j = sum_i (skip h_i == 0) h_i * w_ij, then act
__global__ void k_dfwd_exact(const double* __restrict__ A, int64_t lda, const double* __restrict__ W,
                             int din, int dout, const int32_t* __restrict__ rows, int64_t rb,
                             int64_t n, int relu, double* __restrict__ out, int64_t ldo) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * dout) return;
  const int64_t k = t / dout;
  const int j = static_cast<int>(t % dout);
  const int64_t r = rows ? rows[k] : rb + k;
  double z = 0.0;
  for (int i = 0; i < din; ++i) {
    const double h = A[r * lda + i];
    if (h == 0.0) continue;
    z = __dadd_rn(z, __dmul_rn(h, W[static_cast<int64_t>(i) * dout + j]));
  }
  out[r * ldo + j] = relu ? (0.0 < z ? z : 0.0) : z;
}

// model.hpp:156-170: dh_i = sum_j dz_j * w_ij
__global__ void k_dgrad_exact(const double* __restrict__ A, int64_t lda, const double* __restrict__ W,
                              int din, int dout, const int32_t* __restrict__ rows, int64_t rb,
                              int64_t n, double* __restrict__ out, int64_t ldo) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * din) return;
  const int64_t k = t / din;
  const int i = static_cast<int>(t % din);
  const int64_t r = rows ? rows[k] : rb + k;
  double acc = 0.0;
  for (int j = 0; j < dout; ++j)
    acc = __dadd_rn(acc, __dmul_rn(A[r * lda + j], W[static_cast<int64_t>(i) * dout + j]));
  out[r * ldo + i] = acc;
}

// matrix.hpp:51-65 then add_inplace (engine.hpp:701): out_ij (+)= sum_k (skip a_ki == 0) a_ki b_kj
__global__ void k_wgrad_exact(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                              int64_t ldb, int m, int nn, const int32_t* __restrict__ rows,
                              int64_t rb, int64_t n_rows, int accumulate, double* __restrict__ out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(m) * nn) return;
  const int i = static_cast<int>(t / nn), j = static_cast<int>(t % nn);
  double s = 0.0;
  for (int64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows ? rows[k] : rb + k;
    const double a = A[r * lda + i];
    if (a == 0.0) continue;
    s = __dadd_rn(s, __dmul_rn(a, B[r * ldb + j]));
  }
  out[t] = accumulate ? __dadd_rn(out[t], s) : s;
}

// ------------------------------------------------------------ elementwise ---
template <typename T>
__global__ void k_relu_backward(const T* __restrict__ act, int64_t lda, const T* __restrict__ dh,
                                int64_t ldh, int dim, int64_t rb, int64_t n, T* __restrict__ dz,
                                int64_t ldz) {
  // 2D grid: blockIdx.y walks rows, x covers the row (no 64-bit div/mod per element)
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dim) return;
  for (int64_t k = blockIdx.y; k < n; k += gridDim.y) {
    const int64_t r = rb + k;
    const T a = act[r * lda + j];
    dz[r * ldz + j] = a <= T(0) ? T(0) : dh[r * ldh + j];
  }
}

// float4 variant (dim, leading dims and bases multiples of 4 floats)
__global__ void k_relu_backward4(const float4* __restrict__ act, int64_t lda4,
                                 const float4* __restrict__ dh, int64_t ldh4, int dim4, int64_t rb,
                                 int64_t n, float4* __restrict__ dz, int64_t ldz4) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t total = n * dim4;
  for (int64_t i = t; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = i / dim4;
    const int j = int(i - k * dim4);
    const int64_t r = rb + k;
    const float4 a = act[r * lda4 + j];
    const float4 g = dh[r * ldh4 + j];
    dz[r * ldz4 + j] = make_float4(a.x <= 0.f ? 0.f : g.x, a.y <= 0.f ? 0.f : g.y,
                                   a.z <= 0.f ? 0.f : g.z, a.w <= 0.f ? 0.f : g.w);
  }
}

// One warp per listed row: softmax CE (model.hpp:175-200); loss term per row to `terms`.
template <typename T>
__global__ void k_ce_rows(const T* __restrict__ logits, int64_t ld, int classes,
                          const int32_t* __restrict__ labels, const int32_t* __restrict__ rows,
                          int64_t n, double inv_denom, T* __restrict__ grad, int64_t ldg,
                          double* __restrict__ terms, int* __restrict__ err) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (k >= n) return;
  const int64_t r = rows[k];
  const T* row = logits + r * ld;
  const int y = labels[r];
  if (y < 0 || y >= classes) {
    if (lane == 0) atomicOr(err, kErrLabel);
    return;
  }
  double hi = -INFINITY;
  for (int c = lane; c < classes; c += 32) hi = fmax(hi, static_cast<double>(row[c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  double sum = 0.0;
  for (int c = lane; c < classes; c += 32) sum += exp(static_cast<double>(row[c]) - hi);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double lse = hi + log(sum);
  if (lane == 0) terms[k] = (lse - static_cast<double>(row[y])) * inv_denom;
  T* g = grad + r * ldg;
  for (int c = lane; c < classes; c += 32)
    g[c] = static_cast<T>((exp(static_cast<double>(row[c]) - lse) - (c == y ? 1.0 : 0.0)) *
                          inv_denom);
}

// Fixed-order tree sum of n terms into *acc (single block => deterministic).
__global__ void k_sum_fixed(const double* __restrict__ terms, int64_t n, double* __restrict__ acc) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += terms[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc += sh[0];
}

// count_correct (model.hpp:216-227): first argmax
template <typename T>
__global__ void k_count_correct(const T* __restrict__ logits, int64_t ld, int classes,
                                const int32_t* __restrict__ labels,
                                const int32_t* __restrict__ rows, int64_t n,
                                unsigned long long* __restrict__ acc) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned hit = 0;
  if (k < n) {
    const int64_t r = rows[k];
    const T* row = logits + r * ld;
    int best = 0;
    for (int c = 1; c < classes; ++c)
      if (row[c] > row[best]) best = c;
    hit = best == labels[r];
  }
  const unsigned total = __reduce_add_sync(0xffffffffu, hit);
  if ((threadIdx.x & 31) == 0 && total) atomicAdd(acc, static_cast<unsigned long long>(total));
}

// Production fp32 loss phase in one launch per partition (model.hpp:172-227):
// rows = [train | val | test] of the partition; warp per row.  Train rows:
// softmax cross-entropy in fp32 (max, sum of expf, logf), the loss term in
// fp64 and the gradient (softmax - onehot) / n_train_global written to grad;
// val / test rows: first-argmax hit counts.  Each block adds its 32 row terms
// in row order into block_part[blockIdx.x] (a fixed-order tree over blocks
// follows), so the loss is deterministic.
__global__ void __launch_bounds__(256) k_loss_f32(
    const float* __restrict__ logits, int64_t ld, int classes, const int32_t* __restrict__ labels,
    const int32_t* __restrict__ rows, int64_t n_train, int64_t n_val, int64_t n_test,
    double inv_denom, float* __restrict__ grad, int64_t ldg, double* __restrict__ block_part,
    unsigned long long* __restrict__ correct, int* __restrict__ err) {
  // 8 lanes per row, 32 rows per block (4 per warp): four independent
  // index -> label -> logits chains per warp keep the loads in flight
  __shared__ double rterm[32];
  __shared__ unsigned rhit[32][2];
  const int lane = threadIdx.x & 31, sub = lane & 7, slot = threadIdx.x >> 3;
  const unsigned gm = 0xffu << (lane & 24);  // the row's 8 lanes (groups branch independently)
  const int64_t k = int64_t(blockIdx.x) * 32 + slot;
  const int64_t n_all = n_train + n_val + n_test;
  double term = 0.0;
  unsigned hit_v = 0, hit_t = 0;
  const bool live = k < n_all;
  const int64_t r = live ? rows[k] : 0;
  const int y = live ? labels[r] : 0;
  const float* row = logits + r * ld;
  if (live && (y < 0 || y >= classes)) {
    if (sub == 0) atomicOr(err, kErrLabel);
  } else if (live && k < n_train) {
    float hi = -INFINITY;
    for (int c = sub; c < classes; c += 8) hi = fmaxf(hi, row[c]);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) hi = fmaxf(hi, __shfl_xor_sync(gm, hi, o));
    float sum = 0.f;
    for (int c = sub; c < classes; c += 8) sum += expf(row[c] - hi);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) sum += __shfl_xor_sync(gm, sum, o);
    const float lse = hi + logf(sum);
    term = (static_cast<double>(lse) - static_cast<double>(row[y])) * inv_denom;
    const float sc = static_cast<float>(inv_denom);
    float* g = grad + r * ldg;
    for (int c = sub; c < classes; c += 8) g[c] = (expf(row[c] - lse) - (c == y ? 1.f : 0.f)) * sc;
  } else if (live) {
    // first argmax (model.hpp:216-227): larger value wins, ties -> lower index
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int c = sub; c < classes; c += 8)
      if (row[c] > best) best = row[c], bi = c;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(gm, best, o);
      const int oi = __shfl_xor_sync(gm, bi, o);
      if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi;
    }
    const unsigned hit = bi == y;
    if (k < n_train + n_val) hit_v = hit; else hit_t = hit;
  }
  if (sub == 0) {
    rterm[slot] = term;
    rhit[slot][0] = hit_v;
    rhit[slot][1] = hit_t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    unsigned hv = 0, ht = 0;
    for (int w = 0; w < 32; ++w) t += rterm[w], hv += rhit[w][0], ht += rhit[w][1];
    block_part[blockIdx.x] = t;
    if (hv) atomicAdd(correct, static_cast<unsigned long long>(hv));
    if (ht) atomicAdd(correct + 1, static_cast<unsigned long long>(ht));
  }
}

void loss_f32(qgnn_ctx* ctx, const float* logits, int64_t ld, int classes, const int32_t* labels,
              const int32_t* rows, int64_t n_train, int64_t n_val, int64_t n_test,
              double inv_denom, float* grad, int64_t ldg, double* loss_acc,
              unsigned long long* correct, cudaStream_t s) {
  const int64_t n_all = n_train + n_val + n_test;
  if (!n_all) return;
  const int64_t blocks = ceil_div(n_all, 32);
  double* part = static_cast<double*>(ctx_scratch(ctx, sizeof(double) * blocks));
  k_loss_f32<<<unsigned(blocks), 256, 0, s>>>(logits, ld, classes, labels, rows, n_train, n_val,
                                              n_test, inv_denom, grad, ldg, part, correct,
                                              ctx->d_err);
  k_sum_fixed<<<1, 1024, 0, s>>>(part, blocks, loss_acc);
  check_launch("loss_f32");
}

// optim.hpp:47-62
template <typename T>
__global__ void k_adam(T* __restrict__ p, T* __restrict__ m, T* __restrict__ v,
                       const T* __restrict__ g, int64_t n, T lr, T b1, T b2, T eps, T bc1,
                       T bc2) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T gi = g[i];
  if constexpr (sizeof(T) == 8) {
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), gi));
    const double vi =
        __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mhat = __ddiv_rn(mi, bc1);
    const double vhat = __ddiv_rn(vi, bc2);
    p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  } else {
    const T mi = b1 * m[i] + (T(1) - b1) * gi;
    const T vi = b2 * v[i] + (T(1) - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

// Same step with the bias corrections read from device memory (bc[0], bc[1]), so a
// captured epoch graph picks up each epoch's values (engine).
template <typename T>
__global__ void k_adam_devbc(T* __restrict__ p, T* __restrict__ m, T* __restrict__ v,
                             const T* __restrict__ g, int64_t n, T lr, T b1, T b2, T eps,
                             const double* __restrict__ bc) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const T bc1 = static_cast<T>(bc[0]), bc2 = static_cast<T>(bc[1]);
  const T gi = g[i];
  if constexpr (sizeof(T) == 8) {
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), gi));
    const double vi =
        __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mhat = __ddiv_rn(mi, bc1);
    const double vhat = __ddiv_rn(vi, bc2);
    p[i] = __dsub_rn(p[i], __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  } else {
    const T mi = b1 * m[i] + (T(1) - b1) * gi;
    const T vi = b2 * v[i] + (T(1) - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / bc1) / (sqrtf(vi / bc2) + eps);
  }
}

inline dim3 grid1(int64_t n, int t) { return dim3(static_cast<unsigned>(ceil_div(n, t))); }

// TMA needs a 16-byte aligned base and row pitch
inline bool tma_ok(const void* base, int64_t ld, int64_t row_begin) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(static_cast<const float*>(base) + row_begin * ld);
  return (a & 15) == 0 && (ld * 4) % 16 == 0;
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" {

int qgnn_dense_forward(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* W,
                       int64_t din, int64_t dout, const int32_t* rows, int64_t row_begin,
                       int64_t n_rows, int relu, void* out, int64_t ld_out, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "dense_forward: null context");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == QGNN_F64) {
    k_dfwd_exact<<<grid1(n_rows * dout, 256), 256, 0, s>>>(
        static_cast<const double*>(A), lda, static_cast<const double*>(W), int(din), int(dout),
        rows, row_begin, n_rows, relu, static_cast<double*>(out), ld_out);
  } else if (!rows && use_tc_gemm() && din <= 4096 && tma_ok(A, lda, row_begin)) {
    tc_gemm_rows(ctx, static_cast<const float*>(A) + row_begin * lda, lda,
                 static_cast<const float*>(W), int(dout), int(dout), int(din), 1, n_rows, relu,
                 static_cast<float*>(out) + row_begin * ld_out, ld_out, s);
  } else {
    dim3 g(static_cast<unsigned>(ceil_div(n_rows, BM)), static_cast<unsigned>(ceil_div(dout, BN)), 1);
    k_sgemm<false, false><<<g, 256, 0, s>>>(int(n_rows), int(dout), int(din),
                                            static_cast<const float*>(A), lda,
                                            static_cast<const float*>(W), dout, rows, row_begin,
                                            static_cast<float*>(out), ld_out, rows, row_begin,
                                            relu, int(round_up(din, BK)));
  }
  check_launch("dense_forward");
  QGNN_API_END
}

int qgnn_dense_input_grad(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* W,
                          int64_t din, int64_t dout, const int32_t* rows, int64_t row_begin,
                          int64_t n_rows, void* out, int64_t ld_out, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "dense_input_grad: null context");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == QGNN_F64) {
    k_dgrad_exact<<<grid1(n_rows * din, 256), 256, 0, s>>>(
        static_cast<const double*>(A), lda, static_cast<const double*>(W), int(din), int(dout),
        rows, row_begin, n_rows, static_cast<double*>(out), ld_out);
  } else if (!rows && use_tc_gemm() && dout <= 4096 && tma_ok(A, lda, row_begin)) {
    tc_gemm_rows(ctx, static_cast<const float*>(A) + row_begin * lda, lda,
                 static_cast<const float*>(W), int(dout), int(din), int(dout), 0, n_rows, 0,
                 static_cast<float*>(out) + row_begin * ld_out, ld_out, s);
  } else {
    dim3 g(static_cast<unsigned>(ceil_div(n_rows, BM)), static_cast<unsigned>(ceil_div(din, BN)), 1);
    k_sgemm<false, true><<<g, 256, 0, s>>>(int(n_rows), int(din), int(dout),
                                           static_cast<const float*>(A), lda,
                                           static_cast<const float*>(W), dout, rows, row_begin,
                                           static_cast<float*>(out), ld_out, rows, row_begin, 0,
                                           int(round_up(dout, BK)));
  }
  check_launch("dense_input_grad");
  QGNN_API_END
}

int qgnn_dense_weight_grad(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* B,
                           int64_t ldb, int64_t m, int64_t n, const int32_t* rows,
                           int64_t row_begin, int64_t n_rows, int accumulate, void* out,
                           void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "dense_weight_grad: null context");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == QGNN_F64) {
    k_wgrad_exact<<<grid1(m * n, 128), 128, 0, s>>>(
        static_cast<const double*>(A), lda, static_cast<const double*>(B), ldb, int(m), int(n),
        rows, row_begin, n_rows, accumulate, static_cast<double*>(out));
  } else if (!rows && use_tc_gemm() && n <= 256 && tma_ok(A, lda, row_begin) &&
             tma_ok(B, ldb, row_begin)) {
    int splits = 0;
    const float* part = tc_gemm_wgrad_partials(
        ctx, static_cast<const float*>(A) + row_begin * lda, lda,
        static_cast<const float*>(B) + row_begin * ldb, ldb, int(m), int(n), n_rows, &splits, s);
    k_splitk_reduce<<<grid1(m * n, 256), 256, 0, s>>>(part, splits, m * n,
                                                       static_cast<float*>(out), accumulate);
  } else {
    // split K (rows) so that tiles x splits ~ 4 waves of the SMs
    const int64_t tiles = ceil_div(m, BM) * ceil_div(n, BN);
    int64_t splits = std::max<int64_t>(1, (4 * ctx->num_sms) / std::max<int64_t>(1, tiles));
    int64_t kps = round_up(ceil_div(std::max<int64_t>(n_rows, 1), splits), BK);
    splits = ceil_div(std::max<int64_t>(n_rows, 1), kps);
    float* part = static_cast<float*>(ctx_scratch(ctx, sizeof(float) * splits * m * n));
    dim3 g(static_cast<unsigned>(ceil_div(m, BM)), static_cast<unsigned>(ceil_div(n, BN)),
           static_cast<unsigned>(splits));
    k_sgemm<true, false><<<g, 256, 0, s>>>(int(m), int(n), int(n_rows),
                                           static_cast<const float*>(A), lda,
                                           static_cast<const float*>(B), ldb, rows, row_begin,
                                           part, n, nullptr, 0, 0, int(kps));
    k_splitk_reduce<<<grid1(m * n, 256), 256, 0, s>>>(part, int(splits), m * n,
                                                       static_cast<float*>(out), accumulate);
  }
  check_launch("dense_weight_grad");
  QGNN_API_END
}

int qgnn_relu_backward(qgnn_ctx* ctx, int dtype, const void* act, int64_t ld_act, const void* dh,
                       int64_t ld_dh, int64_t dim, int64_t row_begin, int64_t n_rows, void* dz,
                       int64_t ld_dz, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "relu_backward: null context");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const dim3 g2(static_cast<unsigned>(ceil_div(dim, 128)),
                static_cast<unsigned>(std::min<int64_t>(n_rows, 65535)));
  const bool v4 = dtype == QGNN_F32 && dim % 4 == 0 && ld_act % 4 == 0 && ld_dh % 4 == 0 &&
                  ld_dz % 4 == 0 && (reinterpret_cast<uintptr_t>(act) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dh) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dz) & 15) == 0;
  if (v4) {
    const int64_t total = n_rows * (dim / 4);
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), 148 * 16));
    k_relu_backward4<<<blocks, 256, 0, s>>>(
        static_cast<const float4*>(act), ld_act / 4, static_cast<const float4*>(dh), ld_dh / 4,
        int(dim / 4), row_begin, n_rows, static_cast<float4*>(dz), ld_dz / 4);
  } else if (dtype == QGNN_F64) {
    k_relu_backward<double><<<g2, 128, 0, s>>>(
        static_cast<const double*>(act), ld_act, static_cast<const double*>(dh), ld_dh, int(dim),
        row_begin, n_rows, static_cast<double*>(dz), ld_dz);
  } else {
    k_relu_backward<float><<<g2, 128, 0, s>>>(
        static_cast<const float*>(act), ld_act, static_cast<const float*>(dh), ld_dh, int(dim),
        row_begin, n_rows, static_cast<float*>(dz), ld_dz);
  }
  check_launch("relu_backward");
  QGNN_API_END
}

int qgnn_masked_ce(qgnn_ctx* ctx, int dtype, const void* logits, int64_t ld, int64_t classes,
                   const int32_t* labels, const int32_t* rows, int64_t n_rows, double inv_denom,
                   void* grad, int64_t ld_grad, double* loss_acc, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "masked_ce: null context");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* terms = static_cast<double*>(ctx_scratch(ctx, sizeof(double) * n_rows));
  const dim3 g = grid1(n_rows * 32, 256);
  if (dtype == QGNN_F64)
    k_ce_rows<double><<<g, 256, 0, s>>>(static_cast<const double*>(logits), ld, int(classes),
                                        labels, rows, n_rows, inv_denom,
                                        static_cast<double*>(grad), ld_grad, terms, ctx->d_err);
  else
    k_ce_rows<float><<<g, 256, 0, s>>>(static_cast<const float*>(logits), ld, int(classes),
                                       labels, rows, n_rows, inv_denom, static_cast<float*>(grad),
                                       ld_grad, terms, ctx->d_err);
  k_sum_fixed<<<1, 1024, 0, s>>>(terms, n_rows, loss_acc);
  check_launch("masked_ce");
  QGNN_API_END
}

int qgnn_count_correct(qgnn_ctx* ctx, int dtype, const void* logits, int64_t ld, int64_t classes,
                       const int32_t* labels, const int32_t* rows, int64_t n_rows,
                       unsigned long long* correct_acc, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "count_correct: null context");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == QGNN_F64)
    k_count_correct<double><<<grid1(n_rows, 256), 256, 0, s>>>(
        static_cast<const double*>(logits), ld, int(classes), labels, rows, n_rows, correct_acc);
  else
    k_count_correct<float><<<grid1(n_rows, 256), 256, 0, s>>>(
        static_cast<const float*>(logits), ld, int(classes), labels, rows, n_rows, correct_acc);
  check_launch("count_correct");
  QGNN_API_END
}

int qgnn_adam_step(qgnn_ctx* ctx, int dtype, void* p, void* m, void* v, const void* g, int64_t n,
                   double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                   void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "adam_step: null context");
  if (n == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == QGNN_F64)
    k_adam<double><<<grid1(n, 256), 256, 0, s>>>(
        static_cast<double*>(p), static_cast<double*>(m), static_cast<double*>(v),
        static_cast<const double*>(g), n, lr, beta1, beta2, eps, bc1, bc2);
  else
    k_adam<float><<<grid1(n, 256), 256, 0, s>>>(
        static_cast<float*>(p), static_cast<float*>(m), static_cast<float*>(v),
        static_cast<const float*>(g), n, float(lr), float(beta1), float(beta2), float(eps),
        float(bc1), float(bc2));
  check_launch("adam_step");
  QGNN_API_END
}

}  // extern "C"

namespace qgnn_b200 {
void input_grad_masked_f32(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int64_t din,
                           int64_t dout, int64_t row_begin, int64_t n_rows, float* out,
                           int64_t ldo, const float* mask, int64_t ldm, cudaStream_t s,
                           const uint32_t* mbits, int64_t ldmb) {
  if (n_rows == 0) return;
  if (use_tc_gemm() && dout <= 4096 && tma_ok(A, lda, row_begin)) {
    if (mask && mbits)  // 32 B of bits per 256-wide row instead of the 1 KB activation row
      tc_gemm_rows(ctx, A + row_begin * lda, lda, W, int(dout), int(din), int(dout), 0, n_rows,
                   0, out + row_begin * ldo, ldo, s, nullptr, 0, nullptr, 0,
                   mbits + row_begin * ldmb, ldmb);
    else
      tc_gemm_rows(ctx, A + row_begin * lda, lda, W, int(dout), int(din), int(dout), 0, n_rows,
                   0, out + row_begin * ldo, ldo, s, mask ? mask + row_begin * ldm : nullptr, ldm);
    return;
  }
  const int st = qgnn_dense_input_grad(ctx, QGNN_F32, A, lda, W, din, dout, nullptr, row_begin,
                                       n_rows, out, ldo, s);
  if (st) throw Status(st, qgnn_last_error());
  if (mask) {
    const int st2 = qgnn_relu_backward(ctx, QGNN_F32, mask, ldm, out, ldo, din, row_begin, n_rows,
                                       out, ldo, s);
    if (st2) throw Status(st2, qgnn_last_error());
  }
}

bool dense_forward_bits_f32(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W,
                            int64_t din, int64_t dout, int64_t row_begin, int64_t n_rows,
                            float* out, int64_t ldo, uint32_t* bits, int64_t ldb, cudaStream_t s) {
  if (n_rows == 0) return true;
  if (use_tc_gemm() && din <= 4096 && tma_ok(A, lda, row_begin)) {
    tc_gemm_rows(ctx, A + row_begin * lda, lda, W, int(dout), int(dout), int(din), 1, n_rows, 1,
                 out + row_begin * ldo, ldo, s, nullptr, 0, bits + row_begin * ldb, ldb);
    return true;
  }
  const int st = qgnn_dense_forward(ctx, QGNN_F32, A, lda, W, din, dout, nullptr, row_begin,
                                    n_rows, 1, out, ldo, s);
  if (st) throw Status(st, qgnn_last_error());
  return false;
}

void adam_step_devbc(int dtype, void* p, void* m, void* v, const void* g, int64_t n, double lr,
                     double beta1, double beta2, double eps, const double* bc, cudaStream_t s) {
  if (n == 0) return;
  if (dtype == QGNN_F64)
    k_adam_devbc<double><<<grid1(n, 256), 256, 0, s>>>(
        static_cast<double*>(p), static_cast<double*>(m), static_cast<double*>(v),
        static_cast<const double*>(g), n, lr, beta1, beta2, eps, bc);
  else
    k_adam_devbc<float><<<grid1(n, 256), 256, 0, s>>>(
        static_cast<float*>(p), static_cast<float*>(m), static_cast<float*>(v),
        static_cast<const float*>(g), n, float(lr), float(beta1), float(beta2), float(eps), bc);
  check_launch("adam_step");
}
}  // namespace qgnn_b200
