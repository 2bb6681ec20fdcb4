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

#include <algorithm>
#include <cstdlib>

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

// acc += a * v on float4 as two packed fp32x2 FMAs (FFMA2: same rounding as four
// FFMAs, half the issue slots — the narrow-row gathers are issue-bound)
__device__ __forceinline__ void fma4(float4& acc, float a, const float4& v) {
  unsigned long long c0, c1, v0, v1, aa;
  asm("mov.b64 %0, {%1, %2};" : "=l"(c0) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(c1) : "f"(acc.z), "f"(acc.w));
  asm("mov.b64 %0, {%1, %2};" : "=l"(v0) : "f"(v.x), "f"(v.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(v1) : "f"(v.z), "f"(v.w));
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c0) : "l"(aa), "l"(v0));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c1) : "l"(aa), "l"(v1));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.x), "=f"(acc.y) : "l"(c0));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(acc.z), "=f"(acc.w) : "l"(c1));
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
        for (int i = 0; i < NV; ++i) {
          if constexpr (sizeof(T) == 4 && VEC == 4) {
            float4 ac = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            fma4(ac, a[u], make_float4(v[u][i][0], v[u][i][1], v[u][i][2], v[u][i][3]));
            acc[i][0] = ac.x, acc[i][1] = ac.y, acc[i][2] = ac.z, acc[i][3] = ac.w;
          } else {
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc[i][k] = Arith<T>::madd(a[u], v[u][i][k], acc[i][k]);
          }
        }
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

// ReLU backward folded into the producer of dh: dz = dh * 1[h > 0] is linear in
// dh, so every contribution to dh (SpMM rows, decoded remote partials, the
// transform-first input gradient) can be masked by the layer's activation h
// before it is stored or added (model.hpp:128-153).
// (common.cuh: relu_bits4 / apply_bits4 read either form of the mask)

// ----------------------------------------------------------------- F32 v2 ---
// Production fp32 SpMM over a contiguous row range.  Warp w of block b owns
// row r0 + 8b + w, so at any instant the resident warps of the whole GPU sweep
// one window of consecutive rows: with the graph's locality their neighbour
// rows overlap and are served from L2.  Rows with more than `hub_deg`
// neighbours are skipped here and finished by k_spmm_hubs, where a whole CTA
// splits the row's edge list (no single-warp tail on power-law hubs).
template <int NV>
__device__ __forceinline__ void row_gather4(float (&acc)[NV][4], const float* __restrict__ src,
                                            int64_t ld, int64_t beg, int64_t end,
                                            const int32_t* __restrict__ col,
                                            const float* __restrict__ alpha, int lane, int nvec) {
  gather_edges<float, 4, NV>(acc, src, ld, beg, end, col, alpha, lane, nvec);
}

template <int NV>
__global__ void __launch_bounds__(256, (NV <= 2 ? 3 : 1)) k_spmm_f32(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, int64_t r0, int64_t n_rows,
    float* __restrict__ out, int64_t ldo, int64_t hub_deg, const float* __restrict__ mask,
    int64_t ldm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nvec = dim >> 2;
  {
    const int64_t r = r0 + int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
    if (r >= r0 + n_rows) return;
    const int64_t ea0 = pa[r], ea1 = pa[r + 1];
    const int64_t eb0 = pb ? pb[r] : 0, eb1 = pb ? pb[r + 1] : 0;
    if ((ea1 - ea0) + (eb1 - eb0) > hub_deg) return;  // k_spmm_hubs
    float acc[NV][4];
    if (self_alpha) {
      const float sa = self_alpha[r];
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int cv = lane + 32 * i;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (cv < nvec) vload<float, 4>(x + r * ldx + cv * 4, v);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = sa * v[q];
      }
    } else {
#pragma unroll
      for (int i = 0; i < NV; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
    }
    row_gather4<NV>(acc, x, ldx, ea0, ea1, ca, aa, lane, nvec);
    if (pb) row_gather4<NV>(acc, y, ldy, eb0, eb1, cb, ab, lane, nvec);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int cv = lane + 32 * i;
      if (cv >= nvec) continue;
      if (mask) {
        const uint32_t mb = relu_bits4(mask, ldm, r, cv * 4);
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[i][q] = (mb >> q & 1u) ? acc[i][q] : 0.f;
      }
      vstore<float, 4>(out + r * ldo + cv * 4, acc[i]);
    }
  }
}

// Narrow rows (dim <= 128, one float4 per lane): the full-row kernel would
// keep only 4 gathers of <= 400 B per warp in flight and leave lanes idle for
// dim < 128.  Here G = dim/4 lanes cover one row and E = 32/G lane groups take
// consecutive edges round-robin, 8 steps per round, so every lane has 8
// independent 16-byte gathers in flight (the L2 gather ceiling needs ~8,
// profiles/gather_probe.cu).  Groups meet in a fixed order at the end
// (deterministic); self term first, then the local and remote lists.
__device__ __forceinline__ void grp_gather(float4& acc, const float* __restrict__ src, int64_t ld,
                                           int64_t beg, int64_t end,
                                           const int32_t* __restrict__ col,
                                           const float* __restrict__ alpha, int lane, int grp,
                                           int E, bool act) {
  for (int64_t e0 = beg; e0 < end; e0 += 32) {
    const int cnt = end - e0 < 32 ? static_cast<int>(end - e0) : 32;
    int my_c = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    for (int j = 0; j < cnt; j += 8 * E) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = j + u * E + grp;
        const int c = __shfl_sync(0xffffffffu, my_c, k & 31);
        v[u] = (act && k < cnt) ? __ldg(reinterpret_cast<const float4*>(src + int64_t(c) * ld))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, (j + u * E + grp) & 31);
        fma4(acc, a, v[u]);
      }
    }
  }
}

__global__ void __launch_bounds__(256, 4) k_spmm_f32g(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, int64_t r0, int64_t n_rows,
    float* __restrict__ out, int64_t ldo, int64_t hub_deg, const float* __restrict__ mask,
    int64_t ldm, int parts) {
  // `parts` > 1: the row is cut into `parts` column ranges of `dim` floats, handled
  // by the consecutive CTAs blockIdx.x = parts * row_block + part (wide rows keep
  // 8 gathers per lane in flight at a register budget that allows 32 warps/SM)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int G = dim >> 2, E = 32 / G;
  const int grp = lane / G, sub0 = lane - grp * G;
  const bool act = grp < E;
  // parts > 0: column parts interleaved per row block; parts < 0: part-major
  // (all rows of column part 0 first: an L2 working set of rows x dim floats)
  const unsigned np = unsigned(parts < 0 ? -parts : parts);
  const unsigned rb = parts < 0 ? (gridDim.x / np) : 0;
  const int part = int(parts < 0 ? blockIdx.x / rb : blockIdx.x % np);
  const int sub = sub0 + part * G;  // float4 column of this lane in the full row
  const int64_t r = r0 + int64_t(parts < 0 ? blockIdx.x % rb : blockIdx.x / np) * 8 + warp;
  if (r >= r0 + n_rows) return;
  const int64_t ea0 = pa[r], ea1 = pa[r + 1];
  const int64_t eb0 = pb ? pb[r] : 0, eb1 = pb ? pb[r + 1] : 0;
  if ((ea1 - ea0) + (eb1 - eb0) > hub_deg) return;  // k_spmm_hubseg + k_spmm_hubred
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  grp_gather(acc, x + sub * 4, ldx, ea0, ea1, ca, aa, lane, grp, E, act);
  if (pb) grp_gather(acc, y + sub * 4, ldy, eb0, eb1, cb, ab, lane, grp, E, act);
  const float4 mine = acc;  // group g's partial -> group 0, g ascending
  for (int g = 1; g < E; ++g) {
    const int sl = (lane + g * G) & 31;  // same column (sub0) in group g
    acc.x += __shfl_sync(0xffffffffu, mine.x, sl);
    acc.y += __shfl_sync(0xffffffffu, mine.y, sl);
    acc.z += __shfl_sync(0xffffffffu, mine.z, sl);
    acc.w += __shfl_sync(0xffffffffu, mine.w, sl);
  }
  if (grp == 0) {
    float4 o = acc;
    if (self_alpha) {
      const float sa = self_alpha[r];
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x + r * ldx + sub * 4));
      o = make_float4(fmaf(sa, xv.x, acc.x), fmaf(sa, xv.y, acc.y), fmaf(sa, xv.z, acc.z),
                      fmaf(sa, xv.w, acc.w));
    }
    if (mask) o = apply_bits4(o, relu_bits4(mask, ldm, r, sub * 4));
    *reinterpret_cast<float4*>(out + r * ldo + sub * 4) = o;
  }
}

// 32-byte read-only load (LDG.E.256 on sm_100): two consecutive float4 of a row
__device__ __forceinline__ void ldg256(const float* p, float4& a, float4& b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
}

// ---- packed halo rows -------------------------------------------
// The 8 columns [c0, c0 + 8) of remote slot `slot`, dequantized from its chunk in
// the exchange arena exactly as K3 (k_dequant_f32) would have stored them:
// fmaf(code, S, Z), columns >= dim zero (K3 leaves the halo padding zero).
__device__ __forceinline__ void packed_row8(const PackedHalo& pk, int slot, int c0, float4& a,
                                            float4& b) {
  // off / width first (independent), then header and payload together: two
  // dependent round trips, like slot -> row for an fp32 halo row plus one
  int bw;
  const uint8_t* ch;
  if (pk.direct) {  // slot is the chunk word: no index round trip
    const uint32_t w = static_cast<uint32_t>(slot);
    bw = (0x8420 >> (4 * (w >> 30))) & 0xf;  // code 0..3 -> width 0, 2, 4, 8
    ch = pk.arena + (static_cast<uint64_t>(w & 0x3fffffffu) << 4);
  } else {
    bw = __ldg(pk.bits + slot);
    ch = pk.arena + __ldg(pk.off + slot);
  }
  const uint8_t* pl = ch + 16;
  uint2 q = make_uint2(0u, 0u);
  float4 ra = make_float4(0.f, 0.f, 0.f, 0.f), rb = ra;
  uint4 h = make_uint4(0u, 0u, 0u, 0u);
  if (bw == 0) {  // BitMode::kFp: raw fp32 row (no header), padded to 16 bytes
    const float* f = reinterpret_cast<const float*>(ch);
    if (c0 < pk.dim) ra = __ldg(reinterpret_cast<const float4*>(f + c0));
    if (c0 + 4 < pk.dim) rb = __ldg(reinterpret_cast<const float4*>(f + c0 + 4));
  } else {
    h = __ldg(reinterpret_cast<const uint4*>(ch));
    if (bw == 8)
      q = __ldg(reinterpret_cast<const uint2*>(pl + c0));
    else if (bw == 4)
      q.x = __ldg(reinterpret_cast<const uint32_t*>(pl + (c0 >> 1)));
    else
      q.x = __ldg(reinterpret_cast<const uint16_t*>(pl + (c0 >> 2)));
  }
  a = ra, b = rb;
  if (bw == 0) return;
  a = b = make_float4(0.f, 0.f, 0.f, 0.f);
  if (!pk.direct && (static_cast<int>(h.w & 0xffu) != bw || h.z != static_cast<uint32_t>(pk.dim))) {
    atomicOr(pk.err, kErrDecode);  // chunk disagrees with the index (codec.hpp:90-91)
    return;
  }
  if (!pk.direct && pk.env && (h.w >> 8) != __ldg(pk.env + slot)) {
    atomicOr(pk.err, kErrProtocol);  // misrouted payload / plan-version skew (engine.hpp:530-541)
    return;
  }
  const float sc = __uint_as_float(h.x), zp = __uint_as_float(h.y);
  const int sh = bw == 8 ? 8 : bw;  // bits per code
  const uint32_t m = (1u << sh) - 1u;
  float v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t code = bw == 8 ? ((i < 4 ? q.x : q.y) >> (8 * (i & 3))) & 0xffu
                                  : (q.x >> (sh * i)) & m;
    v[i] = c0 + i < pk.dim ? fmaf(static_cast<float>(code), sc, zp) : 0.f;
  }
  a = make_float4(v[0], v[1], v[2], v[3]);
  b = make_float4(v[4], v[5], v[6], v[7]);
}

// In-kernel hub reduction (replaces the k_spmm_hubred launch).  A lane group of
// G lanes has just stored segment u's partial row; after a fence its leader counts
// the arrival, and the group that brings the last segment of hub h reduces it:
// out[r] = x[r]·α_rr + Σ_s part[s] in segment order, masked — the same arithmetic
// and order as k_spmm_hubred, so the result does not depend on which group does
// it.  The counter is reset by that group for the next launch (stream order).
// All 32 lanes must call this (it shuffles); `mine` marks lanes of a segment unit.
__device__ __noinline__ void hub_finish(bool mine, int64_t u, int sub, int G, int leader,
                                           int dim, const float* __restrict__ x, int64_t ldx,
                                           const float* __restrict__ self_alpha,
                                           const int32_t* __restrict__ hubs,
                                           const int32_t* __restrict__ seg_ptr,
                                           const int32_t* __restrict__ seg_hub,
                                           int32_t* __restrict__ cnt,
                                           const float* __restrict__ part, int64_t ldp,
                                           float* __restrict__ out, int64_t ldo,
                                           const float* __restrict__ mask, int64_t ldm) {
  __threadfence();  // this lane's partial stores before the arrival count
  __syncwarp();
  int last = 0, h = 0;
  if (mine && sub == 0) {
    h = seg_hub[u];
    last = atomicAdd(cnt + h, 1) == seg_ptr[h + 1] - seg_ptr[h] - 1;
  }
  last = __shfl_sync(0xffffffffu, last, leader & 31);
  h = __shfl_sync(0xffffffffu, h, leader & 31);
  if (!(mine && last)) return;
  __threadfence();  // the other groups' partials (their fences precede their counts)
  const int64_t r = hubs[h];
  const float sa = self_alpha ? self_alpha[r] : 0.f;
  const int s0 = seg_ptr[h], s1 = seg_ptr[h + 1];
  for (int c = sub * 4; c < dim; c += 4 * G) {
    float4 v = self_alpha ? *reinterpret_cast<const float4*>(x + r * ldx + c)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
    v.x *= sa, v.y *= sa, v.z *= sa, v.w *= sa;
    for (int sg = s0; sg < s1; ++sg) {
      const float4 p = __ldcg(reinterpret_cast<const float4*>(part + int64_t(sg) * ldp + c));
      v.x += p.x, v.y += p.y, v.z += p.z, v.w += p.w;
    }
    if (mask) v = apply_bits4(v, relu_bits4(mask, ldm, r, c));
    *reinterpret_cast<float4*>(out + r * ldo + c) = v;
  }
  if (sub == 0) cnt[h] = 0;
}

// Narrow rows, two float4 per lane: G = ceil(F/2) lanes per row, E = 32/G
// lane groups, 4 steps per round (8 loads per lane in flight).  Per step a
// warp issues the same index shuffles and address math as k_spmm_f32g but moves
// twice the bytes per lane, so per gathered byte it issues ~half the
// instructions (the 100- and 48-wide layers are issue-bound in k_spmm_f32g).
__device__ __forceinline__ void grp2_gather(float4 (&acc)[2], const float* __restrict__ src,
                                            int ld, int n, const int32_t* __restrict__ col,
                                            const float* __restrict__ alpha, int lane, int grp,
                                            int E, bool act, bool has2, bool v8) {
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int cnt = min(32, n - e0);
    int my_c = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    for (int j = 0; j < cnt; j += 4 * E) {
      float4 v[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = j + u * E + grp;
        const int c = __shfl_sync(0xffffffffu, my_c, k & 31);
        const bool ok = act && k < cnt;
        const float4* p = reinterpret_cast<const float4*>(src + int64_t(c) * ld);
        v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok) {
          if (v8 && has2) {  // adjacent float4 pair: one 32-byte load
            ldg256(reinterpret_cast<const float*>(p), v[u][0], v[u][1]);
          } else {
            v[u][0] = __ldg(p);
            if (has2) v[u][1] = __ldg(p + 1);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, (j + u * E + grp) & 31);
#pragma unroll
        for (int h = 0; h < 2; ++h) fma4(acc[h], a, v[u][h]);
      }
    }
  }
}

// grp2_gather with the rows read from the packed arena (lane columns cx..cx+7)
__device__ __forceinline__ void grp2_gather_pk(float4 (&acc)[2], const PackedHalo& pk, int cx,
                                               int n, const int32_t* __restrict__ col,
                                               const float* __restrict__ alpha, int lane, int grp,
                                               int E, bool act) {
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int cnt = min(32, n - e0);
    int my_c = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    for (int j = 0; j < cnt; j += 4 * E) {
      float4 v[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = j + u * E + grp;
        const int c = __shfl_sync(0xffffffffu, my_c, k & 31);
        v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (act && k < cnt) packed_row8(pk, c, cx, v[u][0], v[u][1]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, (j + u * E + grp) & 31);
#pragma unroll
        for (int h = 0; h < 2; ++h) fma4(acc[h], a, v[u][h]);
      }
    }
  }
}

template <int MINB, bool PK = false>
__global__ void __launch_bounds__(256, MINB) k_spmm_f32g2(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, int64_t r0, int64_t n_rows,
    float* __restrict__ out, int64_t ldo, int64_t hub_deg, const float* __restrict__ mask,
    int64_t ldm, const int64_t* __restrict__ seg, int64_t n_segs, float* __restrict__ part,
    int64_t ldp, const int32_t* __restrict__ hubs, const int32_t* __restrict__ seg_ptr,
    const int32_t* __restrict__ seg_hub, int32_t* __restrict__ cnt, bool v8,
    PackedHalo pk = PackedHalo{}) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int F = dim >> 2, G = (F + 1) >> 1, E = 32 / G;
  const int grp = lane / G, sub = lane - grp * G;
  const bool act = grp < E;
  const bool has2 = 2 * sub + 1 < F;
  // warps [0, n_segs): hub segments into `part` (as k_spmm_wide); then the rows
  const int64_t w = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  const bool is_seg = w < n_segs;
  const int64_t r = is_seg ? -1 : r0 + (w - n_segs);
  if (r >= r0 + n_rows) return;
  int64_t ea0;  // edge ranges rebased to pointers + 32-bit counts
  int na, nb;
  if (is_seg) {
    const int64_t* sg = seg + 4 * w;
    ea0 = sg[0], na = int(sg[1] - ea0), nb = int(sg[3] - sg[2]);
  } else {
    ea0 = pa[r], na = int(pa[r + 1] - ea0), nb = pb ? int(pb[r + 1] - pb[r]) : 0;
    if (na + nb > hub_deg) return;  // segments + k_spmm_hubred
  }
  float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  const int cx = sub * 8;  // first float of this lane's two columns
  grp2_gather(acc, x + cx, int(ldx), na, ca + ea0, aa + ea0, lane, grp, E, act, has2, v8);
  if (nb) {  // b range start re-read here rather than held across the first gather
    const int64_t eb0 = is_seg ? seg[4 * w + 2] : pb[r];
    if constexpr (PK)
      grp2_gather_pk(acc, pk, cx, nb, cb + eb0, ab + eb0, lane, grp, E, act);
    else
      grp2_gather(acc, y + cx, int(ldy), nb, cb + eb0, ab + eb0, lane, grp, E, act, has2, v8);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const float4 mine = acc[h];  // group g's partial -> group 0, g ascending
    for (int g = 1; g < E; ++g) {
      const int sl = (lane + g * G) & 31;
      acc[h].x += __shfl_sync(0xffffffffu, mine.x, sl);
      acc[h].y += __shfl_sync(0xffffffffu, mine.y, sl);
      acc[h].z += __shfl_sync(0xffffffffu, mine.z, sl);
      acc[h].w += __shfl_sync(0xffffffffu, mine.w, sl);
    }
  }
  if (grp == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (h == 1 && !has2) break;
      const int c = cx + 4 * h;
      float4 o = acc[h];
      if (is_seg) {
        *reinterpret_cast<float4*>(part + w * ldp + c) = o;
        continue;
      }
      if (self_alpha) {
        const float sa = self_alpha[r];
        const float4 xv = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
        o = make_float4(fmaf(sa, xv.x, o.x), fmaf(sa, xv.y, o.y), fmaf(sa, xv.z, o.z),
                        fmaf(sa, xv.w, o.w));
      }
      if (mask) o = apply_bits4(o, relu_bits4(mask, ldm, r, c));
      *reinterpret_cast<float4*>(out + r * ldo + c) = o;
    }
  }
  if (is_seg && cnt)  // warp-uniform: the whole warp worked on segment w
    hub_finish(true, w, lane, 32, 0, dim, x, ldx, self_alpha, hubs, seg_ptr, seg_hub, cnt, part,
               ldp, out, ldo, mask, ldm);
}

// Narrow rows (D <= 128), several rows per warp: G = ceil(F/2) lanes (two float4
// each) own one row, R = 32/G rows per warp, no cross-group reduction.  Rows come
// from HubPlan::order — the range's non-hub rows sorted by descending degree — so
// the R rows of a warp have (nearly) the same length and the warp-uniform edge
// loop wastes little; hub segments (256 edges) are the first units.  Per lane 4
// edges x 2 float4 in flight; each step's 4 edge indices are loaded by 4 lanes of
// the group and shuffled to the rest (G >= 4, i.e. D >= 28).
__device__ __forceinline__ void sorted_gather(float4 (&acc)[2], const float* __restrict__ src,
                                              int ld, int n, int nmax,
                                              const int32_t* __restrict__ col,
                                              const float* __restrict__ alpha, bool has2,
                                              int sub, int base, bool v8) {
  for (int j = 0; j < nmax; j += 4) {
    // lanes 0..3 of the group load the step's 4 edge indices, the group shuffles them
    int my_c = 0;
    float my_a = 0.f;
    if (sub < 4 && j + sub < n) my_c = __ldg(col + j + sub), my_a = __ldg(alpha + j + sub);
    int c[4];
    float a[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      c[u] = __shfl_sync(0xffffffffu, my_c, (base + u) & 31);
      a[u] = __shfl_sync(0xffffffffu, my_a, (base + u) & 31);
    }
    float4 v[4][2];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float4* p = reinterpret_cast<const float4*>(src + int64_t(c[u]) * ld);
      v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j + u < n) {
        if (v8 && has2) {  // the lane's two float4 are adjacent: one 32-byte load
          ldg256(reinterpret_cast<const float*>(p), v[u][0], v[u][1]);
        } else {
          v[u][0] = __ldg(p);
          if (has2) v[u][1] = __ldg(p + 1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      fma4(acc[0], a[u], v[u][0]);
      fma4(acc[1], a[u], v[u][1]);
    }
  }
}

template <int MINB>
__global__ void __launch_bounds__(64, MINB) k_spmm_sorted(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab,
    const int32_t* __restrict__ order, int64_t n_order, float* __restrict__ out, int64_t ldo,
    const float* __restrict__ mask, int64_t ldm, const int64_t* __restrict__ seg, int64_t n_segs,
    float* __restrict__ part, int64_t ldp, const int32_t* __restrict__ hubs, const int32_t* __restrict__ seg_ptr,
    const int32_t* __restrict__ seg_hub, int32_t* __restrict__ cnt, bool v8) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int F = dim >> 2, G = (F + 1) >> 1, R = 32 / G;
  const int grp = lane / G, sub = lane - grp * G;
  const bool act = grp < R;
  const bool has2 = 2 * sub + 1 < F;
  const int64_t u = (int64_t(blockIdx.x) * (blockDim.x >> 5) + warp) * R + grp;
  const bool is_seg = u < n_segs;
  const bool live = act && u < n_segs + n_order;
  int64_t ea = 0, eb = 0, r = -1;
  int na = 0, nb = 0;
  if (live) {
    if (is_seg) {
      const int64_t* sg = seg + 4 * u;
      ea = sg[0], na = int(sg[1] - ea), eb = sg[2], nb = int(sg[3] - eb);
    } else {
      r = order[u - n_segs];
      ea = pa[r], na = int(pa[r + 1] - ea);
      if (pb) eb = pb[r], nb = int(pb[r + 1] - eb);
    }
  }
  int ma = na, mb = nb;  // warp-uniform trip counts (rows of a warp have ~equal degree)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ma = max(ma, __shfl_xor_sync(0xffffffffu, ma, o));
    mb = max(mb, __shfl_xor_sync(0xffffffffu, mb, o));
  }
  float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  const int cx = sub * 8;
  // all lanes stay for the shuffles; dead lanes load nothing (n = 0)
  sorted_gather(acc, x + cx, int(ldx), na, ma, ca + ea, aa + ea, has2, sub, grp * G, v8);
  if (mb) sorted_gather(acc, y + cx, int(ldy), nb, mb, cb + eb, ab + eb, has2, sub, grp * G, v8);
  if (n_segs && cnt) {  // kernel-uniform: segment partials, then the in-kernel hub finish
    const bool mine = live && is_seg;
    if (mine) {
      *reinterpret_cast<float4*>(part + u * ldp + cx) = acc[0];
      if (has2) *reinterpret_cast<float4*>(part + u * ldp + cx + 4) = acc[1];
    }
    hub_finish(mine, u, sub, G, grp * G, dim, x, ldx, self_alpha, hubs, seg_ptr, seg_hub, cnt,
               part, ldp, out, ldo, mask, ldm);
    if (is_seg) return;
  }
  if (!live) return;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1 && !has2) break;
    const int c = cx + 4 * h;
    float4 o = acc[h];
    if (is_seg) {
      *reinterpret_cast<float4*>(part + u * ldp + c) = o;
      continue;
    }
    if (self_alpha) {
      const float sa = self_alpha[r];
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
      o = make_float4(fmaf(sa, xv.x, o.x), fmaf(sa, xv.y, o.y), fmaf(sa, xv.z, o.z),
                      fmaf(sa, xv.w, o.w));
    }
    if (mask) o = apply_bits4(o, relu_bits4(mask, ldm, r, c));
    *reinterpret_cast<float4*>(out + r * ldo + c) = o;
  }
}

// 256-wide rows (two float4 per lane, every lane active), register-lean: 32-bit
// edge offsets within the row (pointers rebased once per row), no per-lane column
// bounds, alphas shuffled after the loads — to fit 64 registers (32 warps/SM)
// with the same 8 gathers per lane in flight as k_spmm_f32<2>.
template <bool V8>
__device__ __forceinline__ void wide_gather(float4 (&acc)[2], const float* __restrict__ src,
                                            int ld, int n, const int32_t* __restrict__ col,
                                            const float* __restrict__ alpha, int lane) {
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int cnt = min(32, n - e0);
    int my_c = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    for (int j = 0; j < cnt; j += 4) {
      float4 v[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = __shfl_sync(0xffffffffu, my_c, (j + u) & 31);
        const bool ok = j + u < cnt;
        if (V8) {  // lane owns columns 8 lane .. 8 lane + 7: one 32-byte load
          v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok) ldg256(src + int64_t(c) * ld + 8 * lane, v[u][0], v[u][1]);
        } else {
          const float4* p = reinterpret_cast<const float4*>(src + int64_t(c) * ld) + lane;
          v[u][0] = ok ? __ldg(p) : make_float4(0.f, 0.f, 0.f, 0.f);
          v[u][1] = ok ? __ldg(p + 32) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, (j + u) & 31);
        fma4(acc[0], a, v[u][0]);
        fma4(acc[1], a, v[u][1]);
      }
    }
  }
}

// wide_gather with the rows read from the packed arena (lane columns 8 lane .. +7)
__device__ __forceinline__ void wide_gather_pk(float4 (&acc)[2], const PackedHalo& pk, int n,
                                               const int32_t* __restrict__ col,
                                               const float* __restrict__ alpha, int lane) {
  for (int e0 = 0; e0 < n; e0 += 32) {
    const int cnt = min(32, n - e0);
    int my_c = 0;
    float my_a = 0.f;
    if (lane < cnt) {
      my_c = __ldg(col + e0 + lane);
      my_a = __ldg(alpha + e0 + lane);
    }
    for (int j = 0; j < cnt; j += 4) {
      float4 v[4][2];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = __shfl_sync(0xffffffffu, my_c, (j + u) & 31);
        v[u][0] = v[u][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j + u < cnt) packed_row8(pk, c, 8 * lane, v[u][0], v[u][1]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float a = __shfl_sync(0xffffffffu, my_a, (j + u) & 31);
        fma4(acc[0], a, v[u][0]);
        fma4(acc[1], a, v[u][1]);
      }
    }
  }
}

template <int MINB, bool V8, bool PK = false>
__global__ void __launch_bounds__(64, MINB) k_spmm_wide(
    const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, int64_t r0, int64_t n_rows,
    float* __restrict__ out, int64_t ldo, int64_t hub_deg, const float* __restrict__ mask,
    int64_t ldm, const int64_t* __restrict__ seg, int64_t n_segs, float* __restrict__ part,
    int64_t ldp, const int32_t* __restrict__ hubs, const int32_t* __restrict__ seg_ptr,
    const int32_t* __restrict__ seg_hub, int32_t* __restrict__ cnt, PackedHalo pk = PackedHalo{}) {
  static_assert(!PK || V8, "packed rows use the 8-columns-per-lane layout");
  // warps [0, n_segs) reduce hub segments into `part` (k_spmm_hubred finishes those
  // rows); they take the lowest block ids so the long lists start first and overlap
  // the ordinary rows instead of running as a separate tail launch
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t w = int64_t(blockIdx.x) * (blockDim.x >> 5) + warp;
  const bool is_seg = w < n_segs;
  const int64_t r = r0 + (w - n_segs);
  if (!is_seg && r >= r0 + n_rows) return;
  int64_t ea;
  int na, nb;
  if (is_seg) {
    const int64_t* sg = seg + 4 * w;  // [a0, a1, b0, b1]
    ea = sg[0], na = int(sg[1] - ea), nb = int(sg[3] - sg[2]);
  } else {
    ea = pa[r], na = int(pa[r + 1] - ea), nb = pb ? int(pb[r + 1] - pb[r]) : 0;
    if (na + nb > hub_deg) return;  // segments + k_spmm_hubred
  }
  float4 acc[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  wide_gather<V8>(acc, x, int(ldx), na, ca + ea, aa + ea, lane);
  if (nb) {  // b range start re-read here rather than held across the first gather
    const int64_t eb = is_seg ? seg[4 * w + 2] : pb[r];
    if constexpr (PK)
      wide_gather_pk(acc, pk, nb, cb + eb, ab + eb, lane);
    else
      wide_gather<V8>(acc, y, int(ldy), nb, cb + eb, ab + eb, lane);
  }
  if (is_seg) {
    float* dst = part + w * ldp;
    *reinterpret_cast<float4*>(dst + (V8 ? 8 * lane : 4 * lane)) = acc[0];
    *reinterpret_cast<float4*>(dst + (V8 ? 8 * lane + 4 : 4 * lane + 128)) = acc[1];
    if (cnt)
      hub_finish(true, w, lane, 32, 0, 256, x, ldx, self_alpha, hubs, seg_ptr, seg_hub, cnt, part,
                 ldp, out, ldo, mask, ldm);
    return;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = V8 ? 8 * lane + 4 * h : 4 * (lane + 32 * h);
    float4 o = acc[h];
    if (self_alpha) {
      const float sa = self_alpha[r];
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
      o = make_float4(fmaf(sa, xv.x, o.x), fmaf(sa, xv.y, o.y), fmaf(sa, xv.z, o.z),
                      fmaf(sa, xv.w, o.w));
    }
    if (mask) o = apply_bits4(o, relu_bits4(mask, ldm, r, c));
    *reinterpret_cast<float4*>(out + r * ldo + c) = o;
  }
}

// 256-wide rows of low degree (the remote-partial rows: ~1 edge each), two rows
// per warp: a half-warp owns a row (16 lanes x 16 columns, two 32-byte loads per
// edge), so twice the rows' dependent index -> gather chains are in flight.
// Hub rows are left to k_spmm_wide's segments; no shuffles, halves run freely.
__device__ __forceinline__ void half_gather(float4 (&acc)[4], const float* __restrict__ src,
                                            int ld, int n, const int32_t* __restrict__ col,
                                            const float* __restrict__ alpha, int c0) {
  for (int e = 0; e < n; e += 2) {
    float4 v[2][4];
    float a[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      a[u] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e + u < n) {
        const int c = __ldg(col + e + u);
        a[u] = __ldg(alpha + e + u);
        const float* p = src + int64_t(c) * ld + c0;
        ldg256(p, v[u][0], v[u][1]);
        ldg256(p + 8, v[u][2], v[u][3]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) fma4(acc[q], a[u], v[u][q]);
  }
}

__device__ __forceinline__ void half_gather_pk(float4 (&acc)[4], const PackedHalo& pk, int n,
                                               const int32_t* __restrict__ col,
                                               const float* __restrict__ alpha, int c0) {
  for (int e = 0; e < n; e += 2) {
    float4 v[2][4];
    float a[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      a[u] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e + u < n) {
        const int c = __ldg(col + e + u);
        a[u] = __ldg(alpha + e + u);
        packed_row8(pk, c, c0, v[u][0], v[u][1]);
        packed_row8(pk, c, c0 + 8, v[u][2], v[u][3]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) fma4(acc[q], a[u], v[u][q]);
  }
}

template <bool PK = false>
__global__ void __launch_bounds__(64, 16) k_spmm_wide_half(
    const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, int64_t r0, int64_t n_rows,
    float* __restrict__ out, int64_t ldo, int64_t hub_deg, const float* __restrict__ mask,
    int64_t ldm, PackedHalo pk = PackedHalo{}) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int hl = lane & 15;
  const int64_t r = r0 + (int64_t(blockIdx.x) * (blockDim.x >> 5) + warp) * 2 + (lane >> 4);
  if (r >= r0 + n_rows) return;
  const int64_t ea = pa[r];
  const int na = int(pa[r + 1] - ea), nb = pb ? int(pb[r + 1] - pb[r]) : 0;
  if (na + nb > hub_deg) return;  // k_spmm_wide's segments + in-kernel finish
  const int c0 = 16 * hl;         // this lane's 16 columns
  float4 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  half_gather(acc, x, int(ldx), na, ca + ea, aa + ea, c0);
  if (nb) {
    const int64_t eb = pb[r];
    if constexpr (PK)
      half_gather_pk(acc, pk, nb, cb + eb, ab + eb, c0);
    else
      half_gather(acc, y, int(ldy), nb, cb + eb, ab + eb, c0);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c = c0 + 4 * q;
    float4 o = acc[q];
    if (self_alpha) {
      const float sa = self_alpha[r];
      const float4 xv = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
      o = make_float4(fmaf(sa, xv.x, o.x), fmaf(sa, xv.y, o.y), fmaf(sa, xv.z, o.z),
                      fmaf(sa, xv.w, o.w));
    }
    if (mask) o = apply_bits4(o, relu_bits4(mask, ldm, r, c));
    *reinterpret_cast<float4*>(out + r * ldo + c) = o;
  }
}

// One CTA per hub row: 8 warps take contiguous eighths of the edge lists,
// partial sums meet in shared memory and are added in warp order (deterministic).
template <int NV>
__global__ void __launch_bounds__(256) k_spmm_hubs(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const float* __restrict__ self_alpha, const int64_t* __restrict__ pa,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int64_t* __restrict__ pb,
    const int32_t* __restrict__ cb, const float* __restrict__ ab, const int32_t* __restrict__ hubs,
    float* __restrict__ out, int64_t ldo) {
  extern __shared__ float part[];  // [8][NV * 128]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = hubs[blockIdx.x];
  const int nvec = dim >> 2;
  float acc[NV][4];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
  {
    const int64_t e0 = pa[r], e1 = pa[r + 1], len = e1 - e0;
    const int64_t b = e0 + len * warp / 8, e = e0 + len * (warp + 1) / 8;
    row_gather4<NV>(acc, x, ldx, b, e, ca, aa, lane, nvec);
  }
  if (pb) {
    const int64_t e0 = pb[r], e1 = pb[r + 1], len = e1 - e0;
    const int64_t b = e0 + len * warp / 8, e = e0 + len * (warp + 1) / 8;
    row_gather4<NV>(acc, y, ldy, b, e, cb, ab, lane, nvec);
  }
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) part[warp * NV * 128 + (lane + 32 * i) * 4 + q] = acc[i][q];
  __syncthreads();
  const float sa = self_alpha ? self_alpha[r] : 0.f;
  for (int c = threadIdx.x; c < nvec * 4; c += blockDim.x) {
    float v = self_alpha ? sa * x[r * ldx + c] : 0.f;
    for (int w = 0; w < 8; ++w) v += part[w * NV * 128 + c];
    out[r * ldo + c] = v;
  }
}

// Hub rows, segmented: each 256-edge segment of a hub row's (local, then
// remote) edge list is one warp's work; partial rows are then added in segment
// order with the self term (deterministic).  A 17k-neighbour hub becomes ~70
// independent warps instead of one CTA.
template <int NV>
__global__ void __launch_bounds__(256) k_spmm_hubseg(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ y, int64_t ldy,
    const int32_t* __restrict__ ca, const float* __restrict__ aa, const int32_t* __restrict__ cb,
    const float* __restrict__ ab, const int64_t* __restrict__ seg, int64_t n_segs,
    float* __restrict__ part, int64_t ldp) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (g >= n_segs) return;
  const int nvec = dim >> 2;
  const int64_t* sg = seg + 4 * g;  // [a0, a1, b0, b1]
  float acc[NV][4];
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[i][q] = 0.f;
  row_gather4<NV>(acc, x, ldx, sg[0], sg[1], ca, aa, lane, nvec);
  if (sg[3] > sg[2]) row_gather4<NV>(acc, y, ldy, sg[2], sg[3], cb, ab, lane, nvec);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int cv = lane + 32 * i;
    if (cv < nvec) vstore<float, 4>(part + g * ldp + cv * 4, acc[i]);
  }
}

__global__ void __launch_bounds__(256) k_spmm_hubred(
    int dim, const float* __restrict__ x, int64_t ldx, const float* __restrict__ self_alpha,
    const int32_t* __restrict__ hubs, const int32_t* __restrict__ seg_ptr, int64_t n_hubs,
    const float* __restrict__ part, int64_t ldp, float* __restrict__ out, int64_t ldo,
    const float* __restrict__ mask, int64_t ldm) {
  const int lane = threadIdx.x & 31;
  const int64_t h = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (h >= n_hubs) return;
  const int64_t r = hubs[h];
  const float sa = self_alpha ? self_alpha[r] : 0.f;
  for (int c = lane * 4; c < dim; c += 128) {
    float4 v = self_alpha ? *reinterpret_cast<const float4*>(x + r * ldx + c) : make_float4(0, 0, 0, 0);
    v.x *= sa, v.y *= sa, v.z *= sa, v.w *= sa;
    for (int s = seg_ptr[h]; s < seg_ptr[h + 1]; ++s) {
      const float4 p = *reinterpret_cast<const float4*>(part + int64_t(s) * ldp + c);
      v.x += p.x, v.y += p.y, v.z += p.z, v.w += p.w;
    }
    if (mask) v = apply_bits4(v, relu_bits4(mask, ldm, r, c));
    *reinterpret_cast<float4*>(out + r * ldo + c) = v;
  }
}

// QGNN_SPMM_SPLIT=1: two warps per 256-wide row, interleaved (measured slower);
// =2: the two column halves as two sweeps over all rows (half the L2 working set)
static int split_wide() {
  const char* e = std::getenv("QGNN_SPMM_SPLIT");
  return e ? std::atoi(e) : 0;
}

static bool two_per_lane() {  // QGNN_SPMM_G2=0: one float4 per lane (k_spmm_f32g)
  const char* e = std::getenv("QGNN_SPMM_G2");
  return !e || std::atoi(e) != 0;
}

static int spmm_tpb() {  // threads per block of the full-row kernel (QGNN_SPMM_TPB)
  const char* e = std::getenv("QGNN_SPMM_TPB");
  return e ? std::max(32, std::min(256, std::atoi(e))) : 64;  // small blocks: a straggler row
                                                                  // holds 1 warp slot, not 8
}

static int wide_lean() {  // QGNN_SPMM_WIDE=0: 256-wide rows via k_spmm_f32<2>
  const char* e = std::getenv("QGNN_SPMM_WIDE");
  return e ? std::atoi(e) : 1;
}

static int g2_minb() {  // QGNN_G2_MINB=3: 85-register k_spmm_f32g2 (no spills, 24 warps/SM)
  const char* e = std::getenv("QGNN_G2_MINB");
  return e ? std::atoi(e) : 4;
}

static int sorted_rows() {  // QGNN_SPMM_SORTED=0: narrow rows via k_spmm_f32g2 (2: 64 regs)
  const char* e = std::getenv("QGNN_SPMM_SORTED");
  return e ? std::atoi(e) : 1;
}

static int sorted_max_dim() {  // widest rows sent to k_spmm_sorted (QGNN_SPMM_SORTED_MAXD)
  const char* e = std::getenv("QGNN_SPMM_SORTED_MAXD");
  return e ? std::atoi(e) : 64;
}

static bool hub_finish_inline() {  // QGNN_HUB_FINISH=0: hub rows reduced by k_spmm_hubred
  const char* e = std::getenv("QGNN_HUB_FINISH");
  return !e || std::atoi(e) != 0;
}

static bool load256() {  // QGNN_SPMM_LD256=0: 16-byte gathers only
  const char* e = std::getenv("QGNN_SPMM_LD256");
  return !e || std::atoi(e) != 0;
}

static double half_rows_deg() {  // QGNN_SPMM_HALF_DEG: mean degree below which 256-wide
  const char* e = std::getenv("QGNN_SPMM_HALF_DEG");  // ranges run two rows per warp
  return e ? std::atof(e) : 4.0;
}

static bool merge_hubs() {  // QGNN_HUB_MERGE=0: hub segments as a separate k_spmm_hubseg launch
  const char* e = std::getenv("QGNN_HUB_MERGE");
  return !e || std::atoi(e) != 0;
}

static bool grouped_narrow() {  // QGNN_SPMM_GROUPED=0 selects the one-row-per-warp kernel
  const char* e = std::getenv("QGNN_SPMM_GROUPED");
  return !e || std::atoi(e) != 0;
}

// fp32 row-range SpMM with optional hub list (rows with > hub_deg neighbours).
bool spmm_packed_ok(int dim, const HubPlan* hp, const float* x, int64_t ldx) {
  if (hp && hp->order && dim <= sorted_max_dim() && dim / 4 >= 7 && sorted_rows()) return false;
  if (hp && hp->n_hubs > 0 && !merge_hubs()) return false;
  const int nv = int(ceil_div(dim / 4, 32));
  if (nv == 1) return grouped_narrow() && dim / 4 >= 5 && two_per_lane();
  const bool v8 = load256() && (reinterpret_cast<uintptr_t>(x) & 31) == 0 && ldx % 8 == 0;
  return dim == 256 && wide_lean() && split_wide() == 0 && v8;
}

int spmm_f32(qgnn_ctx* ctx, int dim, const float* x, int64_t ldx, const float* y, int64_t ldy,
              const float* sa, const int64_t* pa, const int32_t* ca, const float* aa,
              const int64_t* pb, const int32_t* cb, const float* ab, int64_t row_begin,
              int64_t n_rows, float* out, int64_t ldo, const HubPlan* hp, cudaStream_t s,
              const float* mask, int64_t ldm, const PackedHalo* pk) {
  if (n_rows <= 0) return 0;
  if (pk && !spmm_packed_ok(dim, hp, x, ldx))
    throw Status(QGNN_EINVAL, "spmm_f32: no packed-halo kernel for this row range");
  const int nv = int(ceil_div(dim / 4, 32));
  const int64_t blocks = ceil_div(n_rows, 8);
  const bool hubs = hp && hp->n_hubs > 0;
  const int64_t hd = hubs ? hp->hub_deg : (int64_t(1) << 62);
#define QGNN_SPMM_CASE(NVV)                                                                    \
  case NVV:                                                                                    \
    k_spmm_f32<NVV><<<unsigned(ceil_div(n_rows, spmm_tpb() / 32)), spmm_tpb(), 0, s>>>(         \
                                                     dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, \
                                                     ab, row_begin, n_rows, out, ldo, hd, mask, ldm); \
    if (hubs) {                                                                                \
      k_spmm_hubseg<NVV><<<unsigned(ceil_div(hp->n_segs * 32, 256)), 256, 0, s>>>(             \
          dim, x, ldx, y, ldy, ca, aa, cb, ab, hp->seg, hp->n_segs, hp->part, hp->ldp);        \
      k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(                  \
          dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask, ldm); \
    }                                                                                          \
    break;
  if (hp && hp->order && dim <= sorted_max_dim() && dim / 4 >= 7 && sorted_rows()) {
    const int G = (dim / 4 + 1) / 2, R = 32 / G;
    const int64_t ns = hp->n_hubs > 0 ? hp->n_segs : 0;
    const int64_t units = ns + hp->n_order;
    const unsigned nb = unsigned(ceil_div(ceil_div(units, R), 2));
    int32_t* cnt = ns && hp->cnt && hub_finish_inline() ? hp->cnt : nullptr;
    const bool v8 = load256() && (reinterpret_cast<uintptr_t>(x) & 31) == 0 && ldx % 8 == 0 &&
                    (!y || ((reinterpret_cast<uintptr_t>(y) & 31) == 0 && ldy % 8 == 0));
    if (sorted_rows() == 2)
      k_spmm_sorted<16><<<nb, 64, 0, s>>>(dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab,
                                          hp->order, hp->n_order, out, ldo, mask, ldm, hp->seg, ns,
                                          hp->part, hp->ldp, hp->hubs, hp->seg_ptr, hp->seg_hub,
                                          cnt, v8);
    else
      k_spmm_sorted<12><<<nb, 64, 0, s>>>(dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab,
                                          hp->order, hp->n_order, out, ldo, mask, ldm, hp->seg, ns,
                                          hp->part, hp->ldp, hp->hubs, hp->seg_ptr, hp->seg_hub,
                                          cnt, v8);
    if (hp->n_hubs > 0 && !cnt)
      k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(
          dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask,
          ldm);
    check_launch("k_spmm_sorted");
    return 1 + (hp->n_hubs > 0 && !cnt ? 1 : 0);
  }
  const int sw = split_wide();
  const int parts = nv == 1 ? 1 : (nv == 2 && dim % 8 == 0 && sw) ? (sw == 2 ? -2 : 2) : 0;
  if (parts && grouped_narrow()) {
    const int np = parts < 0 ? -parts : parts;
    if (parts == 1 && dim / 4 >= 5 && two_per_lane()) {
      const bool mg = hubs && merge_hubs();
      const int64_t ns = mg ? hp->n_segs : 0;
      if (hubs && !mg)
        k_spmm_hubseg<1><<<unsigned(ceil_div(hp->n_segs * 32, 256)), 256, 0, s>>>(
            dim, x, ldx, y, ldy, ca, aa, cb, ab, hp->seg, hp->n_segs, hp->part, hp->ldp);
      const unsigned nb2 = unsigned(ceil_div(ns + n_rows, spmm_tpb() / 32));
      int32_t* cnt = ns && hp->cnt && hub_finish_inline() ? hp->cnt : nullptr;
      const int32_t* hh = hubs ? hp->hubs : nullptr;
      const int32_t* hsp = hubs ? hp->seg_ptr : nullptr;
      const int32_t* hsh = hubs ? hp->seg_hub : nullptr;
      const bool v8 = load256() && (reinterpret_cast<uintptr_t>(x) & 31) == 0 && ldx % 8 == 0 &&
                      (!y || ((reinterpret_cast<uintptr_t>(y) & 31) == 0 && ldy % 8 == 0));
      if (pk)
        k_spmm_f32g2<4, true><<<nb2, spmm_tpb(), 0, s>>>(
            dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask,
            ldm, hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0, hh,
            hsp, hsh, cnt, v8, *pk);
      else if (g2_minb() == 3)
        k_spmm_f32g2<3><<<nb2, spmm_tpb(), 0, s>>>(
            dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask,
            ldm, hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0, hh,
            hsp, hsh, cnt, v8);
      else
        k_spmm_f32g2<4><<<nb2, spmm_tpb(), 0, s>>>(
            dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask,
            ldm, hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0, hh,
            hsp, hsh, cnt, v8);
      if (hubs && !cnt)
        k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(
            dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask,
            ldm);
      check_launch("k_spmm_f32g2");
      return 1 + (hubs ? (cnt ? 0 : mg ? 1 : 2) : 0);
    }
    k_spmm_f32g<<<unsigned(blocks * np), 256, 0, s>>>(dim / np, x, ldx, y, ldy, sa, pa, ca, aa,
                                                      pb, cb, ab, row_begin, n_rows, out, ldo, hd,
                                                      mask, ldm, parts);
    if (hubs) {
      if (nv == 1)
        k_spmm_hubseg<1><<<unsigned(ceil_div(hp->n_segs * 32, 256)), 256, 0, s>>>(
            dim, x, ldx, y, ldy, ca, aa, cb, ab, hp->seg, hp->n_segs, hp->part, hp->ldp);
      else
        k_spmm_hubseg<2><<<unsigned(ceil_div(hp->n_segs * 32, 256)), 256, 0, s>>>(
            dim, x, ldx, y, ldy, ca, aa, cb, ab, hp->seg, hp->n_segs, hp->part, hp->ldp);
      k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(
          dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask,
          ldm);
    }
    check_launch("k_spmm_f32g");
    return 1 + (hubs ? 2 : 0);
  }
  if (dim == 256 && wide_lean()) {
    const bool mg = hubs && merge_hubs();
    const int64_t ns = mg ? hp->n_segs : 0;
    if (hubs && !mg)
      k_spmm_hubseg<2><<<unsigned(ceil_div(hp->n_segs * 32, 256)), 256, 0, s>>>(
          dim, x, ldx, y, ldy, ca, aa, cb, ab, hp->seg, hp->n_segs, hp->part, hp->ldp);
    int32_t* cnt = ns && hp->cnt && hub_finish_inline() ? hp->cnt : nullptr;
    // 32-byte loads need 32-byte aligned rows (engine buffers: ld multiple of 8 floats)
    const bool v8 = load256() && (reinterpret_cast<uintptr_t>(x) & 31) == 0 && ldx % 8 == 0 &&
                    (!y || ((reinterpret_cast<uintptr_t>(y) & 31) == 0 && ldy % 8 == 0));
    if (v8 && hp && hp->avg_deg < half_rows_deg()) {
      // low-degree rows: two per warp; hub segments (if any) through k_spmm_wide
      if (pk)
        k_spmm_wide_half<true><<<unsigned(ceil_div(n_rows, 4)), 64, 0, s>>>(
            x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask, ldm,
            *pk);
      else
        k_spmm_wide_half<<<unsigned(ceil_div(n_rows, 4)), 64, 0, s>>>(
            x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask, ldm);
      if (ns && pk)
        k_spmm_wide<16, true, true><<<unsigned(ceil_div(ns, 2)), 64, 0, s>>>(
            x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, 0, out, ldo, hd, mask, ldm,
            hp->seg, ns, hp->part, hp->ldp, hp->hubs, hp->seg_ptr, hp->seg_hub, cnt, *pk);
      else if (ns)
        k_spmm_wide<16, true><<<unsigned(ceil_div(ns, 2)), 64, 0, s>>>(
            x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, 0, out, ldo, hd, mask, ldm,
            hp->seg, ns, hp->part, hp->ldp, hp->hubs, hp->seg_ptr, hp->seg_hub, cnt);
      if (hubs && !cnt)
        k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(
            dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask,
            ldm);
      check_launch("k_spmm_wide_half");
      return 1 + (ns ? 1 : 0) + (hubs && !cnt ? 1 : 0);
    }
    if (pk)
      k_spmm_wide<16, true, true><<<unsigned(ceil_div(ns + n_rows, 2)), 64, 0, s>>>(
          x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask, ldm,
          hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0,
          hubs ? hp->hubs : nullptr, hubs ? hp->seg_ptr : nullptr, hubs ? hp->seg_hub : nullptr,
          cnt, *pk);
    else if (v8)
      k_spmm_wide<16, true><<<unsigned(ceil_div(ns + n_rows, 2)), 64, 0, s>>>(
          x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask, ldm,
          hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0,
          hubs ? hp->hubs : nullptr, hubs ? hp->seg_ptr : nullptr, hubs ? hp->seg_hub : nullptr,
          cnt);
    else
      k_spmm_wide<16, false><<<unsigned(ceil_div(ns + n_rows, 2)), 64, 0, s>>>(
          x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, row_begin, n_rows, out, ldo, hd, mask, ldm,
          hubs ? hp->seg : nullptr, ns, hubs ? hp->part : nullptr, hubs ? hp->ldp : 0,
          hubs ? hp->hubs : nullptr, hubs ? hp->seg_ptr : nullptr, hubs ? hp->seg_hub : nullptr,
          cnt);
    if (hubs && !cnt) {
      k_spmm_hubred<<<unsigned(ceil_div(hp->n_hubs * 32, 64)), 64, 0, s>>>(
          dim, x, ldx, sa, hp->hubs, hp->seg_ptr, hp->n_hubs, hp->part, hp->ldp, out, ldo, mask,
          ldm);
    }
    check_launch("k_spmm_wide");
    return 1 + (hubs ? (cnt ? 0 : mg ? 1 : 2) : 0);
  }
  switch (nv) {
    QGNN_SPMM_CASE(1)
    QGNN_SPMM_CASE(2)
    QGNN_SPMM_CASE(3)
    QGNN_SPMM_CASE(4)
    QGNN_SPMM_CASE(5)
    QGNN_SPMM_CASE(8)
    default:
      throw Status(QGNN_EINVAL, "spmm_f32: feature dim too large");
  }
#undef QGNN_SPMM_CASE
  check_launch("k_spmm_f32");
  return 1 + (hubs ? 2 : 0);
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
    if (vec4 && !rows && pick_nv(dim / 4) <= 5) {
      spmm_f32(ctx, d, static_cast<const float*>(x), ld_x, static_cast<const float*>(y), ld_y,
               static_cast<const float*>(self_alpha), ptr_a, col_a,
               static_cast<const float*>(alpha_a), ptr_b, col_b,
               static_cast<const float*>(alpha_b), row_begin, n_rows, static_cast<float*>(out),
               ld_out, nullptr, s);
    } else if (vec4) {
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
