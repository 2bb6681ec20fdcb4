// spmm.cu — K4: row-subset CSR aggregation (aggregate.hpp:94-165).
//
// One warp owns one output row and keeps it in registers (lanes split the
// feature dimension in 16-byte vectors).  Neighbour indices/coefficients are
// fetched 32 at a time with one coalesced load and broadcast by shuffle; the
// neighbour rows are gathered four at a time to keep several 16-byte loads in
// flight per lane.  The summation order is the reference's (self, local
// neighbours in CSR order, remote neighbours in CSR order), so the F64
// instantiation is bit-identical to aggregate_rows / aggregate_backward_local
// and the transposed-CSR form of backward_remote_partials; F32 contracts to FMA.
#include <cuda_runtime.h>

#include "common.cuh"

namespace qgnn_b200 {

template <typename T, int VEC>
struct VecT;
template <>
struct VecT<float, 4> {
  using type = float4;
};
template <>
struct VecT<float, 1> {
  using type = float;
};
template <>
struct VecT<double, 1> {
  using type = double;
};

template <typename T, int VEC>
__device__ __forceinline__ void vload(const T* p, T (&v)[VEC]) {
  if constexpr (VEC == 4) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = t.x;
    v[1] = t.y;
    v[2] = t.z;
    v[3] = t.w;
  } else {
    v[0] = __ldg(p);
  }
}

template <typename T, int VEC>
__device__ __forceinline__ void vstore(T* p, const T (&v)[VEC]) {
  if constexpr (VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    p[0] = v[0];
  }
}

template <typename T, int VEC, int NV>
__device__ __forceinline__ void gather_edges(T (&acc)[NV][VEC], const T* __restrict__ src,
                                             int64_t ld, const int64_t beg, const int64_t end,
                                             const int32_t* __restrict__ col,
                                             const T* __restrict__ alpha, int lane, int nvec) {
  for (int64_t e0 = beg; e0 < end; e0 += 32) {
    const int cnt = end - e0 < 32 ? static_cast<int>(end - e0) : 32;
    int my_c = 0;
    T my_a = T(0);
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    int j = 0;
    for (; j + 4 <= cnt; j += 4) {
      int c[4];
      T a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = __shfl_sync(0xffffffffu, my_c, j + u);
        a[u] = __shfl_sync(0xffffffffu, my_a, j + u);
      }
      T v[4][NV][VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const int cv = lane + 32 * i;
          if (cv < nvec) vload<T, VEC>(src + static_cast<int64_t>(c[u]) * ld + cv * VEC, v[u][i]);
        }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int i = 0; i < NV; ++i)
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[i][k] = Arith<T>::madd(a[u], v[u][i][k], acc[i][k]);
    }
    for (; j < cnt; ++j) {
      const int c = __shfl_sync(0xffffffffu, my_c, j);
      const T a = __shfl_sync(0xffffffffu, my_a, j);
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int cv = lane + 32 * i;
        if (cv < nvec) {
          T v[VEC];
          vload<T, VEC>(src + static_cast<int64_t>(c) * ld + cv * VEC, v);
#pragma unroll
          for (int k = 0; k < VEC; ++k) acc[i][k] = Arith<T>::madd(a, v[k], acc[i][k]);
        }
      }
    }
  }
}

template <typename T, int VEC, int NV>
__global__ void __launch_bounds__(256) k_csr_aggregate(
    int dim, const T* __restrict__ x, int64_t ldx, const T* __restrict__ y, int64_t ldy,
    const T* __restrict__ self_alpha, const int64_t* __restrict__ ptr_a,
    const int32_t* __restrict__ col_a, const T* __restrict__ alpha_a,
    const int64_t* __restrict__ ptr_b, const int32_t* __restrict__ col_b,
    const T* __restrict__ alpha_b, const int32_t* __restrict__ rows, int64_t row_begin,
    int64_t n_rows, T* __restrict__ out, int64_t ldo) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (k >= n_rows) return;
  const int64_t r = rows ? static_cast<int64_t>(rows[k]) : row_begin + k;
  const int nvec = (dim + VEC - 1) / VEC;
  T acc[NV][VEC];
  if (self_alpha) {
    const T sa = self_alpha[r];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int cv = lane + 32 * i;
      T v[VEC];
      if (cv < nvec) vload<T, VEC>(x + r * ldx + cv * VEC, v);
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[i][q] = cv < nvec ? Arith<T>::mul(sa, v[q]) : T(0);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i)
#pragma unroll
      for (int q = 0; q < VEC; ++q) acc[i][q] = T(0);
  }
  gather_edges<T, VEC, NV>(acc, x, ldx, ptr_a[r], ptr_a[r + 1], col_a, alpha_a, lane, nvec);
  if (ptr_b) gather_edges<T, VEC, NV>(acc, y, ldy, ptr_b[r], ptr_b[r + 1], col_b, alpha_b, lane, nvec);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int cv = lane + 32 * i;
    if (cv < nvec) vstore<T, VEC>(out + r * ldo + cv * VEC, acc[i]);
  }
}

template <typename T, int VEC>
void launch_csr(int nv, int dim, const T* x, int64_t ldx, const T* y, int64_t ldy, const T* sa,
                const int64_t* pa, const int32_t* ca, const T* aa, const int64_t* pb,
                const int32_t* cb, const T* ab, const int32_t* rows, int64_t rb, int64_t n,
                T* out, int64_t ldo, cudaStream_t s) {
  const int threads = 256;
  const int64_t blocks = ceil_div(n * 32, threads);
#define QGNN_CSR_CASE(NVV)                                                                   \
  case NVV:                                                                                  \
    k_csr_aggregate<T, VEC, NVV><<<blocks, threads, 0, s>>>(dim, x, ldx, y, ldy, sa, pa, ca, \
                                                            aa, pb, cb, ab, rows, rb, n, out, ldo); \
    break;
  switch (nv) {
    QGNN_CSR_CASE(1)
    QGNN_CSR_CASE(2)
    QGNN_CSR_CASE(3)
    QGNN_CSR_CASE(4)
    QGNN_CSR_CASE(5)
    QGNN_CSR_CASE(8)
    case 16:
    case 32:
      if constexpr (VEC == 1) {
        if (nv == 16)
          k_csr_aggregate<T, VEC, 16><<<blocks, threads, 0, s>>>(dim, x, ldx, y, ldy, sa, pa, ca,
                                                                 aa, pb, cb, ab, rows, rb, n, out, ldo);
        else
          k_csr_aggregate<T, VEC, 32><<<blocks, threads, 0, s>>>(dim, x, ldx, y, ldy, sa, pa, ca,
                                                                 aa, pb, cb, ab, rows, rb, n, out, ldo);
        break;
      }
      [[fallthrough]];
    default:
      throw Status(QGNN_EINVAL, "csr_aggregate: feature dim too large");
  }
#undef QGNN_CSR_CASE
  check_launch("k_csr_aggregate");
}

inline int pick_nv(int64_t nvec) {
  const int64_t need = ceil_div(nvec, 32);
  for (int c : {1, 2, 3, 4, 5, 8, 16, 32})
    if (need <= c) return c;
  return 0;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" int qgnn_csr_aggregate(qgnn_ctx* ctx, int dtype, int64_t dim, const void* x,
                                  int64_t ld_x, const void* y, int64_t ld_y,
                                  const void* self_alpha, const int64_t* ptr_a,
                                  const int32_t* col_a, const void* alpha_a,
                                  const int64_t* ptr_b, const int32_t* col_b,
                                  const void* alpha_b, const int32_t* rows, int64_t row_begin,
                                  int64_t n_rows, void* out, int64_t ld_out, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "csr_aggregate: null context");
  QGNN_REQUIRE(dim > 0, QGNN_EINVAL, "csr_aggregate: dim must be > 0");
  if (n_rows == 0) return QGNN_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int d = static_cast<int>(dim);
  if (dtype == QGNN_F64) {
    const int nv = pick_nv(dim);
    launch_csr<double, 1>(nv, d, static_cast<const double*>(x), ld_x,
                          static_cast<const double*>(y), ld_y,
                          static_cast<const double*>(self_alpha), ptr_a, col_a,
                          static_cast<const double*>(alpha_a), ptr_b, col_b,
                          static_cast<const double*>(alpha_b), rows, row_begin, n_rows,
                          static_cast<double*>(out), ld_out, s);
  } else {
    const bool vec4 = dim % 4 == 0 && ld_x % 4 == 0 && ld_out % 4 == 0 && aligned16(x) &&
                      aligned16(out) && (!ptr_b || (ld_y % 4 == 0 && aligned16(y)));
    if (vec4) {
      const int nv = pick_nv(dim / 4);
      launch_csr<float, 4>(nv, d, static_cast<const float*>(x), ld_x,
                           static_cast<const float*>(y), ld_y,
                           static_cast<const float*>(self_alpha), ptr_a, col_a,
                           static_cast<const float*>(alpha_a), ptr_b, col_b,
                           static_cast<const float*>(alpha_b), rows, row_begin, n_rows,
                           static_cast<float*>(out), ld_out, s);
    } else {
      const int nv = pick_nv(dim);
      launch_csr<float, 1>(nv, d, static_cast<const float*>(x), ld_x,
                           static_cast<const float*>(y), ld_y,
                           static_cast<const float*>(self_alpha), ptr_a, col_a,
                           static_cast<const float*>(alpha_a), ptr_b, col_b,
                           static_cast<const float*>(alpha_b), rows, row_begin, n_rows,
                           static_cast<float*>(out), ld_out, s);
    }
  }
  QGNN_API_END
}
