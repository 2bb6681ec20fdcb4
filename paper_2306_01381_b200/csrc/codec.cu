// codec.cu — K1 (stochastic quantize + LSB-first pack + trace window) and
// K3 (unpack + dequantize + scatter/accumulate) for sm_100a.
//
// Work decomposition: one warp per message (row, destination).  The row is
// read once for the extrema (warp-shuffle min/max), then each lane produces
// whole 32-bit payload words (32/b codes each), so the payload store of a
// warp is a contiguous, coalesced run.  Every element draws its own uniform
// from the counter-based generator, u_i = mix(key + (i+1)*phi) >> 11, so the
// draws are embarrassingly parallel and bit-identical to the reference's
// sequential stream (quant.hpp:81-87).  The per-element arithmetic is the
// reference's fp64 sequence x=(h-lo)/S, floor, frac, u<frac, clamp.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "rng.cuh"

namespace qgnn_b200 {

constexpr int kHdrGpu = 16;

// GPU-layout chunk envelope (header word 3 above the width byte): source
// partition, destination partition and plan version, each mod 256 — the
// per-message form of the reference payload's routing fields (source, target,
// plan_version; engine.hpp:530-541).  `env` = source | version << 8;
// the destination is the message's set index.
__device__ __forceinline__ uint32_t env_word(int b, uint32_t env, const uint16_t* set_of,
                                             int64_t m) {
  const uint32_t dst = set_of ? set_of[m] : 0u;
  return static_cast<uint32_t>(b) | (env & 0xffu) << 8 | (dst & 0xffu) << 16 |
         ((env >> 8) & 0xffu) << 24;
}
constexpr int kHdrRef = 25;

__host__ __device__ inline uint64_t packed_bytes(uint64_t count, int b) {
  return (count * static_cast<uint64_t>(b) + 7) / 8;
}
__host__ __device__ inline uint64_t chunk_bytes(uint64_t count, int b, int layout, int elem) {
  if (b == 0) {  // raw row; GPU layout pads it to 16 bytes so every chunk stays 16-aligned
    const uint64_t raw = count * static_cast<uint64_t>(elem);
    return layout == QGNN_WIRE_REF ? raw : (raw + 15) / 16 * 16;
  }
  if (layout == QGNN_WIRE_REF) return kHdrRef + packed_bytes(count, b);
  return kHdrGpu + ((packed_bytes(count, b) + 15) / 16) * 16;
}

template <typename T>
__device__ __forceinline__ bool is_finite_t(T v) {
  return isfinite(v);
}

// Warp-wide first-occurrence fix-up for signed zeros: the reference's
// sequential std::min/std::max keep the FIRST element equal to the extremum
// (quant.hpp:63-68), which only matters for +0.0 vs -0.0.
template <typename T>
__device__ __forceinline__ T first_zero(const T* row, int dim, int lane) {
  for (int base = 0; base < dim; base += 32) {
    const int j = base + lane;
    const bool z = j < dim && row[j] == T(0);
    const unsigned mask = __ballot_sync(0xffffffffu, z);
    if (mask) return row[base + __ffs(mask) - 1];
  }
  return T(0);
}

template <typename T>
__device__ __forceinline__ void row_extrema(const T* __restrict__ row, int dim, int lane, T& lo,
                                            T& hi, bool& finite) {
  lo = INFINITY;
  hi = -INFINITY;
  finite = true;
  for (int j = lane; j < dim; j += 32) {
    const T v = row[j];
    finite &= is_finite_t(v);
    lo = v < lo ? v : lo;
    hi = hi < v ? v : hi;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const T h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = hi < h2 ? h2 : hi;
  }
  finite = __all_sync(0xffffffffu, finite);
  if (lo == T(0)) lo = first_zero(row, dim, lane);
  if (hi == T(0)) hi = first_zero(row, dim, lane);
}

__device__ __forceinline__ void store_u64_bytes(uint8_t* p, uint64_t v, int lane_byte, int base) {
  // writes byte (lane_byte - base) of v when in range
  const int k = lane_byte - base;
  if (k >= 0 && k < 8) p[lane_byte] = static_cast<uint8_t>(v >> (8 * k));
}

template <typename T>
__global__ void __launch_bounds__(256) k_quantize_pack(
    const T* __restrict__ values, int64_t ld, int dim, int64_t n, const int32_t* __restrict__ rows,
    const uint32_t* __restrict__ ids, const uint8_t* __restrict__ bits,
    const uint64_t* __restrict__ offsets, const uint16_t* __restrict__ set_of,
    const uint64_t* __restrict__ set_keys, int layout, uint8_t* __restrict__ out,
    T* __restrict__ win_lo, T* __restrict__ win_hi, int* __restrict__ err, uint32_t env) {
  const int lane = threadIdx.x & 31;
  const int64_t m = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (m >= n) return;
  const T* row = values + static_cast<int64_t>(rows[m]) * ld;
  const int b = bits[m];
  uint8_t* chunk = out + offsets[m];

  T lo, hi;
  bool finite;
  row_extrema(row, dim, lane, lo, hi, finite);
  if (lane == 0 && win_lo) {  // trace.hpp:86-91 (update precedes encode, engine.hpp:487)
    const T wl = win_lo[m], wh = win_hi[m];
    win_lo[m] = lo < wl ? lo : wl;
    win_hi[m] = wh < hi ? hi : wh;
  }
  if (b == 0) {  // BitMode::kFp: raw row (engine.hpp:473-481)
    T* dst = reinterpret_cast<T*>(chunk);
    for (int j = lane; j < dim; j += 32) dst[j] = row[j];
    return;
  }
  if (b != 2 && b != 4 && b != 8) {
    if (lane == 0) atomicOr(err, kErrBadWidth);
    return;
  }
  if (!finite) {
    if (lane == 0) atomicOr(err, kErrNonFinite);
    return;
  }
  const double lo_d = static_cast<double>(lo), hi_d = static_cast<double>(hi);
  const uint32_t levels = (1u << b) - 1;
  const bool constant = hi_d == lo_d;
  const double scale = constant ? 0.0 : (hi_d - lo_d) / static_cast<double>(levels);

  uint8_t* payload;
  if (layout == QGNN_WIRE_GPU) {
    if (lane == 0) {
      uint4 h;
      h.x = __float_as_uint(static_cast<float>(scale));
      h.y = __float_as_uint(static_cast<float>(lo_d));
      h.z = static_cast<uint32_t>(dim);
      h.w = env_word(b, env, set_of, m);
      *reinterpret_cast<uint4*>(chunk) = h;
    }
    payload = chunk + kHdrGpu;
  } else {  // quant.hpp:109-119, byte-identical
    if (lane < kHdrRef) {
      if (lane == 0) chunk[0] = static_cast<uint8_t>(b);
      store_u64_bytes(chunk, static_cast<uint64_t>(dim), lane, 1);
      store_u64_bytes(chunk, __double_as_longlong(scale), lane, 9);
      store_u64_bytes(chunk, __double_as_longlong(lo_d), lane, 17);
    }
    payload = chunk + kHdrRef;
  }

  const int nbytes = static_cast<int>(packed_bytes(dim, b));
  const int epw = 32 / b;
  const int nwords =
      layout == QGNN_WIRE_GPU ? ((nbytes + 15) / 16) * 4 : (nbytes + 3) / 4;
  const uint64_t key = rng_fork(set_keys[set_of ? set_of[m] : 0], ids[m]);
  const double lv = static_cast<double>(levels);

  for (int w = lane; w < nwords; w += 32) {
    uint32_t word = 0;
    if (!constant) {
      const int e0 = w * epw;
      const int e1 = min(e0 + epw, dim);
      for (int e = e0; e < e1; ++e) {
        const double x = __ddiv_rn(__dsub_rn(static_cast<double>(row[e]), lo_d), scale);
        double base = floor(x);
        const double frac = __dsub_rn(x, base);
        const double u = static_cast<double>(rng_u53(key, static_cast<uint64_t>(e) + 1)) *
                         0x1.0p-53;
        if (u < frac) base = __dadd_rn(base, 1.0);
        const uint32_t code = static_cast<uint32_t>(base < lv ? base : lv);
        word |= code << ((e - e0) * b);
      }
    }
    if (layout == QGNN_WIRE_GPU) {
      reinterpret_cast<uint32_t*>(payload)[w] = word;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * w + k < nbytes) payload[4 * w + k] = static_cast<uint8_t>(word >> (8 * k));
    }
  }
}

__device__ __forceinline__ uint64_t load_u64_bytes(const uint8_t* p) {
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) v |= static_cast<uint64_t>(p[k]) << (8 * k);
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) k_dequant_scatter(
    const uint8_t* __restrict__ in, int64_t n, int dim, const uint8_t* __restrict__ bits,
    const uint64_t* __restrict__ offsets, int layout, const int32_t* __restrict__ dst_rows,
    int accumulate, T* __restrict__ out, int64_t ld, int* __restrict__ err,
    const uint32_t* __restrict__ expect) {
  const int lane = threadIdx.x & 31;
  const int64_t m = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (m >= n) return;
  const uint8_t* chunk = in + offsets[m];
  const int b = bits[m];
  T* dst = out + (dst_rows ? static_cast<int64_t>(dst_rows[m]) : m) * ld;
  if (b == 0) {
    const T* src = reinterpret_cast<const T*>(chunk);
    for (int j = lane; j < dim; j += 32) dst[j] = accumulate ? dst[j] + src[j] : src[j];
    return;
  }
  int hb;
  uint64_t count;
  double scale_d, zero_d;
  float scale_f = 0.f, zero_f = 0.f;
  const uint8_t* payload;
  if (layout == QGNN_WIRE_GPU) {
    const uint4 h = *reinterpret_cast<const uint4*>(chunk);
    scale_f = __uint_as_float(h.x);
    zero_f = __uint_as_float(h.y);
    scale_d = scale_f;
    zero_d = zero_f;
    count = h.z;
    hb = static_cast<int>(h.w & 0xff);
    payload = chunk + kHdrGpu;
    if (expect && (h.w >> 8) != expect[m]) {  // engine.hpp:530-541
      if (lane == 0) atomicOr(err, kErrProtocol);
      return;
    }
  } else {
    hb = chunk[0];
    count = load_u64_bytes(chunk + 1);
    scale_d = __longlong_as_double(load_u64_bytes(chunk + 9));
    zero_d = __longlong_as_double(load_u64_bytes(chunk + 17));
    payload = chunk + kHdrRef;
  }
  if (hb != b || count != static_cast<uint64_t>(dim)) {  // codec.hpp:88-89
    if (lane == 0) atomicOr(err, kErrDecode);
    return;
  }
  const int nbytes = static_cast<int>(packed_bytes(dim, b));
  const int epw = 32 / b;
  const uint32_t mask = (1u << b) - 1;
  const int nwords = (nbytes + 3) / 4;
  for (int w = lane; w < nwords; w += 32) {
    uint32_t word;
    if (layout == QGNN_WIRE_GPU) {
      word = reinterpret_cast<const uint32_t*>(payload)[w];
    } else {
      word = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * w + k < nbytes) word |= static_cast<uint32_t>(payload[4 * w + k]) << (8 * k);
    }
    const int e0 = w * epw;
    const int e1 = min(e0 + epw, dim);
    for (int e = e0; e < e1; ++e) {
      const uint32_t code = (word >> ((e - e0) * b)) & mask;
      T v;
      if (sizeof(T) == 4 && layout == QGNN_WIRE_GPU) {
        v = static_cast<T>(fmaf(static_cast<float>(code), scale_f, zero_f));
      } else {  // quant.hpp:97: code*S then +Z, both rounded
        v = static_cast<T>(__dadd_rn(__dmul_rn(static_cast<double>(code), scale_d), zero_d));
      }
      if (accumulate) {
        if (sizeof(T) == 8)
          dst[e] = static_cast<T>(__dadd_rn(static_cast<double>(dst[e]), static_cast<double>(v)));
        else
          dst[e] = dst[e] + v;
      } else {
        dst[e] = v;
      }
    }
  }
}


// ------------------------------------------------------------------ fast path ---
// fp32 rows, GPU wire layout: lane l owns the float4 chunks c = l + 32 i of the
// row, held in registers for both the extrema and the encode (one row read).
// Chunk c's 4 codes occupy 4b bits at payload byte c*b/2, so a lane stores 1, 2
// or 4 bytes per chunk and a warp instruction writes a contiguous run.  The
// draw counter of element e is e + 1; consecutive elements advance the
// generator input by +phi (64-bit add) instead of a multiply.
// Element math.  Reference: x = RN((h - lo) / S), base = floor(x),
// frac = x - base, base += (u < frac), code = min(base, levels) (quant.hpp:81-87).
// Fast path: x' = RN(a * RN(1/S)) satisfies |x' - x| < 2^-43 for x <= 255, so
// floor(x') == floor(x) and (u < frac') == (u < frac) whenever frac' and
// u - frac' stay 2^-40 away from the decision boundaries.  h == lo gives x = 0
// exactly (code 0); h == hi uses x_hi = RN((hi - lo) / S), computed once per
// message with the exact division.  Anything else within 2^-40 of a boundary
// (probability ~1e-12 per element) is flagged and recomputed by quant_exact.
// The draw u = (mix(z) >> 11) * 2^-53 with z = key + (e + 1) * phi.
struct QRow {
  double lo, scale, rcp, x_hi;
  float hi;
  uint32_t levels;
};

__device__ __forceinline__ uint32_t quant_fast(float h, const QRow& R, uint64_t z, bool& slow) {
  constexpr double tol = 0x1.0p-40;
  const double a = __dsub_rn(static_cast<double>(h), R.lo);
  const double u = static_cast<double>(rng_mix(z) >> 11) * 0x1.0p-53;
  const bool top = h == R.hi;
  const double x = top ? R.x_hi : __dmul_rn(a, R.rcp);
  const double base = floor(x);
  const double frac = __dsub_rn(x, base);
  const double d = fabs(u - frac);
  slow = !top && a != 0.0 && !(frac >= tol && frac <= 1.0 - tol && d > tol);
  const uint32_t code = static_cast<uint32_t>(base) + (u < frac ? 1u : 0u);
  return code < R.levels ? code : R.levels;
}

__device__ __noinline__ uint32_t quant_exact(float h, double lo_d, double scale, double lv,
                                             uint64_t z) {
  const double a = __dsub_rn(static_cast<double>(h), lo_d);
  const double u = static_cast<double>(rng_mix(z) >> 11) * 0x1.0p-53;
  const double x = __ddiv_rn(a, scale);
  double base = floor(x);
  const double frac = __dsub_rn(x, base);
  if (u < frac) base = __dadd_rn(base, 1.0);
  return static_cast<uint32_t>(base < lv ? base : lv);
}

// First-occurrence signed zero from registers (quant.hpp:63-68 keeps the FIRST
// element equal to the extremum; only +0.0 vs -0.0 can differ): the lowest
// element index holding a zero, warp-wide, and that element's sign.
template <int NV>
__device__ __forceinline__ float first_zero_reg(const float (&v)[NV][4], int lane, int dim) {
  int key = 0x7fffffff;  // (index << 1) | sign
#pragma unroll
  for (int i = NV - 1; i >= 0; --i)
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      const int e = 4 * (lane + 32 * i) + q;
      if (e < dim && v[i][q] == 0.f) key = (e << 1) | int(__float_as_uint(v[i][q]) >> 31);
    }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
  return (key & 1) ? -0.f : 0.f;
}

template <int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) k_quantize_pack_f32(
    const float* __restrict__ values, int64_t ld, int dim, int64_t n,
    const int32_t* __restrict__ rows, const uint32_t* __restrict__ ids,
    const uint8_t* __restrict__ bits, const uint64_t* __restrict__ offsets,
    const uint16_t* __restrict__ set_of, const uint64_t* __restrict__ set_keys,
    uint8_t* __restrict__ out, float* __restrict__ win_lo, float* __restrict__ win_hi,
    int* __restrict__ err, uint32_t env) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t m = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; m < n;
       m += wstride) {
  const float* row = values + static_cast<int64_t>(rows[m]) * ld;
  const int b = bits[m];
  uint8_t* chunk = out + offsets[m];
  const int nchunk = (dim + 3) >> 2;
  float v[NV][4];
  float lo = INFINITY, hi = -INFINITY;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nchunk) {
      const float4 t = __ldg(reinterpret_cast<const float4*>(row) + c);
      v[i][0] = t.x, v[i][1] = t.y, v[i][2] = t.z, v[i][3] = t.w;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (4 * c + q < dim) {
          finite &= isfinite(v[i][q]);
          lo = v[i][q] < lo ? v[i][q] : lo;
          hi = hi < v[i][q] ? v[i][q] : hi;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const float h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = hi < h2 ? h2 : hi;
  }
  finite = __all_sync(0xffffffffu, finite);
  if (lo == 0.f || hi == 0.f) {  // signed-zero first occurrence, from registers
    const float z0 = first_zero_reg<NV>(v, lane, dim);
    if (lo == 0.f) lo = z0;
    if (hi == 0.f) hi = z0;
  }
  if (lane == 0 && win_lo) {
    const float wl = win_lo[m], wh = win_hi[m];
    win_lo[m] = lo < wl ? lo : wl;
    win_hi[m] = wh < hi ? hi : wh;
  }
  if (b == 0) {
    float* dst = reinterpret_cast<float*>(chunk);
    for (int j = lane; j < dim; j += 32) dst[j] = row[j];
    continue;
  }
  if (b != 2 && b != 4 && b != 8) {
    if (lane == 0) atomicOr(err, kErrBadWidth);
    continue;
  }
  if (!finite) {
    if (lane == 0) atomicOr(err, kErrNonFinite);
    continue;
  }
  const double lo_d = lo, hi_d = hi;
  const uint32_t levels = (1u << b) - 1;
  const bool constant = hi_d == lo_d;
  const double scale = constant ? 0.0 : (hi_d - lo_d) / static_cast<double>(levels);
  if (lane == 0) {
    uint4 h;
    h.x = __float_as_uint(static_cast<float>(scale));
    h.y = __float_as_uint(lo);
    h.z = static_cast<uint32_t>(dim);
    h.w = env_word(b, env, set_of, m);
    *reinterpret_cast<uint4*>(chunk) = h;
  }
  uint8_t* payload = chunk + kHdrGpu;
  const int padded = static_cast<int>(((packed_bytes(dim, b) + 15) / 16) * 16);
  const int units = padded * 2 / b;  // chunk-sized store units incl. zero padding
  const uint64_t key = rng_fork(set_keys[set_of ? set_of[m] : 0], ids[m]);
  QRow R;
  R.lo = lo_d;
  R.scale = scale;
  R.rcp = constant ? 0.0 : __drcp_rn(scale);
  R.x_hi = constant ? 0.0 : __ddiv_rn(__dsub_rn(hi_d, lo_d), scale);
  R.hi = hi;
  R.levels = levels;
#pragma unroll
  for (int i = 0; i < NV + 1; ++i) {
    const int c = lane + 32 * i;
    if (c >= units) break;
    uint32_t word = 0;
    if (i < NV && c < nchunk && !constant) {
      const uint64_t z0 = key + static_cast<uint64_t>(4 * c + 1) * kPhi;
      uint64_t z = z0;
      uint32_t slow_mask = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        bool sl;
        const uint32_t code = quant_fast(v[i][q], R, z, sl);
        if (4 * c + q < dim) {
          word |= code << (q * b);
          slow_mask |= uint32_t(sl) << q;
        }
        z += kPhi;
      }
      if (slow_mask) {  // ~1e-12 per element: exact division for the flagged ones
        const double lv = static_cast<double>(levels);
        for (int q = 0; q < 4; ++q)
          if (slow_mask >> q & 1) {
            const uint32_t code = quant_exact(v[i][q], lo_d, scale, lv, z0 + uint64_t(q) * kPhi);
            word = (word & ~(((1u << b) - 1) << (q * b))) | (code << (q * b));
          }
      }
    }
    if (b == 8)
      reinterpret_cast<uint32_t*>(payload)[c] = word;
    else if (b == 4)
      reinterpret_cast<uint16_t*>(payload)[c] = static_cast<uint16_t>(word);
    else
      payload[c] = static_cast<uint8_t>(word);
  }
  }
}

// Payload of one message from the row in registers (lane l holds float4 chunks
// c = l + 32 i): per element one counter draw and the branch-free fp64 decision,
// flagged elements (~1e-12) recomputed exactly; zero padding to 16 bytes.
template <int NV>
__device__ __forceinline__ void encode_payload(const float (&v)[NV][4], int lane, int dim, int b,
                                               double lo_d, float hi, double scale, double rcp,
                                               double x_hi, uint64_t key, uint8_t* payload) {
  const int nchunk = dim >> 2;
  const uint32_t levels = (1u << b) - 1;
  const bool constant = scale == 0.0;
  const int padded = static_cast<int>(((packed_bytes(dim, b) + 15) / 16) * 16);
  const int units = (padded * 2) >> (b == 8 ? 3 : b == 4 ? 2 : 1);
  constexpr double tol = 0x1.0p-40;
#pragma unroll
  for (int i = 0; i < NV + 1; ++i) {
    const int c = lane + 32 * i;
    if (c >= units) break;
    uint32_t word = 0;
    if (i < NV && c < nchunk && !constant) {
      const uint64_t z0 = key + static_cast<uint64_t>(4 * c + 1) * kPhi;
      bool slow = false;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float hq = v[i][q];
        const double a = __dsub_rn(static_cast<double>(hq), lo_d);
        const double u = static_cast<double>(rng_mix(z0 + uint64_t(q) * kPhi) >> 11) * 0x1.0p-53;
        const double x = hq == hi ? x_hi : __dmul_rn(a, rcp);
        const double base = floor(x);
        const double frac = __dsub_rn(x, base);
        const uint32_t code = static_cast<uint32_t>(base) + (u < frac ? 1u : 0u);
        word |= min(code, levels) << (q * b);
        // x' within 2^-43 of x: the decision can only differ near a boundary;
        // non-short-circuit: predicate logic instead of a branch per element
        slow |= (hq != hi) & (a != 0.0) &
                ((frac < tol) | (frac > 1.0 - tol) | (fabs(u - frac) < tol));
      }
      if (slow) {  // ~1e-12 per element: recompute the chunk exactly
        const double lv = static_cast<double>(levels);
        word = 0;
        for (int q = 0; q < 4; ++q)
          word |= quant_exact(v[i][q], lo_d, scale, lv, z0 + uint64_t(q) * kPhi) << (q * b);
      }
    }
    if (b == 8)
      reinterpret_cast<uint32_t*>(payload)[c] = word;
    else if (b == 4)
      reinterpret_cast<uint16_t*>(payload)[c] = static_cast<uint16_t>(word);
    else
      payload[c] = static_cast<uint8_t>(word);
  }
}

// Lean variant for dim % 4 == 0 (every production width): the profile of the
// general kernel showed the integer ALU pipe at 64 % with ~116 instructions per
// element (bounds checks, compare/select chains, divergence bookkeeping).
// Here: no per-element bounds, extrema with FMNMX, the signed-zero search only
// when the row holds a -0.0 (the first-occurrence rule can only differ then),
// and per element one counter draw plus a branch-free fp64 decision whose
// exactness is checked arithmetically (see quant_fast); flagged elements
// (~1e-12, and never h == lo) take quant_exact.  Same codes and headers.
template <int NV, int MINB>
__global__ void __launch_bounds__(256, MINB) k_quantize_pack_lean(
    const float* __restrict__ values, int64_t ld, int dim, int64_t n,
    const int32_t* __restrict__ rows, const uint32_t* __restrict__ ids,
    const uint8_t* __restrict__ bits, const uint64_t* __restrict__ offsets,
    const uint16_t* __restrict__ set_of, const uint64_t* __restrict__ set_keys,
    uint8_t* __restrict__ out, float* __restrict__ win_lo, float* __restrict__ win_hi,
    int* __restrict__ err, uint32_t env) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  const int nchunk = dim >> 2;
  for (int64_t m = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; m < n;
       m += wstride) {
    const float* row = values + static_cast<int64_t>(rows[m]) * ld;
    const int b = bits[m];
    uint8_t* chunk = out + offsets[m];
    float v[NV][4];
    float lo = INFINITY, hi = -INFINITY;
    bool finite = true, negz = false;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + 32 * i;
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < nchunk) t = __ldg(reinterpret_cast<const float4*>(row) + c);
      v[i][0] = t.x, v[i][1] = t.y, v[i][2] = t.z, v[i][3] = t.w;
      if (c < nchunk) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          lo = fminf(lo, v[i][q]);
          hi = fmaxf(hi, v[i][q]);
          finite &= fabsf(v[i][q]) < INFINITY;
          negz |= __float_as_uint(v[i][q]) == 0x80000000u;
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    finite = __all_sync(0xffffffffu, finite);
    // fminf/fmaxf may pick either signed zero; the reference keeps the first
    // occurrence (quant.hpp:63-68), which only matters if a -0.0 is present
    if (lo == 0.f || hi == 0.f) {
      float z0 = 0.f;
      if (__any_sync(0xffffffffu, negz)) z0 = first_zero_reg<NV>(v, lane, dim);
      if (lo == 0.f) lo = z0;
      if (hi == 0.f) hi = z0;
    }
    if (lane == 0 && win_lo) {  // trace.hpp:86-91 (update precedes encode, engine.hpp:487)
      const float wl = win_lo[m], wh = win_hi[m];
      win_lo[m] = lo < wl ? lo : wl;
      win_hi[m] = wh < hi ? hi : wh;
    }
    if (b == 0) {  // BitMode::kFp: raw row (engine.hpp:473-481)
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        if (c < nchunk)
          reinterpret_cast<float4*>(chunk)[c] = make_float4(v[i][0], v[i][1], v[i][2], v[i][3]);
      }
      continue;
    }
    if (b != 2 && b != 4 && b != 8) {
      if (lane == 0) atomicOr(err, kErrBadWidth);
      continue;
    }
    if (!finite) {
      if (lane == 0) atomicOr(err, kErrNonFinite);
      continue;
    }
    const double lo_d = lo, hi_d = hi;
    const uint32_t levels = (1u << b) - 1;
    const bool constant = hi_d == lo_d;
    const double scale = constant ? 0.0 : (hi_d - lo_d) / static_cast<double>(levels);
    if (lane == 0) {
      uint4 h;
      h.x = __float_as_uint(static_cast<float>(scale));
      h.y = __float_as_uint(lo);
      h.z = static_cast<uint32_t>(dim);
      h.w = env_word(b, env, set_of, m);
      *reinterpret_cast<uint4*>(chunk) = h;
    }
    const uint64_t key = rng_fork(set_keys[set_of ? set_of[m] : 0], ids[m]);
    const double rcp = constant ? 0.0 : __drcp_rn(scale);
    const double x_hi = constant ? 0.0 : __ddiv_rn(__dsub_rn(hi_d, lo_d), scale);
    encode_payload<NV>(v, lane, dim, b, lo_d, hi, scale, rcp, x_hi, key, chunk + kHdrGpu);
  }
}

// ------------------------------------------------------------ grouped K1 ---
// Production K1 (fp32 rows, GPU layout).  G = 2^lg lanes own one message (G *
// EPL >= dim) and a warp carries 32 / G messages, so lane j holds the EPL
// contiguous elements [j*EPL, (j+1)*EPL): its payload is one contiguous run of
// EPL*b/8 bytes (16 B at 8 bits -> one 128-bit store), and the per-message
// scalars (key fork, S, 1/S) are amortized over EPL elements per lane instead
// of 4-8 (D = 256: 2 messages per warp; D = 100: 4).
//
// Element decision in fp32 with a proven error bound, exact fallback.  The
// reference computes x = RN(RN(h - lo) / S) in fp64 and code = min(floor(x) +
// (u < frac(x)), levels) (quant.hpp:81-87); that is ceil(T) - 1 for T = x + 1 - u.
// Here (YD, the default) y = fma_f(RN_f(h - lo), RN_f(1/S), 1 - u_f) with u_f
// the draw's top 23 bits (u_f <= u < u_f + 2^-23, and 1 - u_f exact), so
// |y - T| <= 2.01 * 2^-24 * levels + ulp(y) / 2 + 2^-23 < 4.6e-5 < 2^-14 at 8
// bits.  t = RZ_f(512 + y) holds floor(y * 2^14) in its mantissa: code =
// floor(y) = t >> 14, exact whenever y's fraction is at least 2^-13 away from
// 0 and 1 (then T is not an integer and floor(T) == floor(y), and floor(y) <=
// levels); the rest (4 * 2^-14 = 2.4e-4 of the elements, lattice points and
// u_f = 0 among them) take quant_fast / quant_exact, the fp64 path of the lean
// kernel, so every code is the reference's.  h == lo (y = 1 - u_f) and h == hi
// (x next to levels) need no special case.  The x-domain form (YD = false,
// QGNN_K1_YDOM=0) decides floor(x_f) and u_f < frac(x_f) separately with the
// bound dl = levels * 2^-22 and special-cases h == hi.  The top 23 bits of the
// draw are bits 41..63 of the second multiply: the final xorshift (z ^ z >> 31)
// does not touch them, and only the high word of that product is formed.
// 32-bit form: 14 integer ops.
__device__ __forceinline__ uint32_t draw_top32(uint32_t lo, uint32_t hi) {  // z = key+(e+2)phi
  const uint32_t tl = lo ^ __funnelshift_r(lo, hi, 30);  // z ^= z >> 30
  const uint32_t th = hi ^ (hi >> 30);
  const uint64_t w = static_cast<uint64_t>(tl) * 0x1ce4e5b9u;  // z *= 0xbf58476d1ce4e5b9
  const uint32_t ml = static_cast<uint32_t>(w);
  const uint32_t mh = static_cast<uint32_t>(w >> 32) + tl * 0xbf58476du + th * 0x1ce4e5b9u;
  const uint32_t sl = ml ^ __funnelshift_r(ml, mh, 27);  // z ^= z >> 27
  const uint32_t sh = mh ^ (mh >> 27);
  return __umulhi(sl, 0x133111ebu) + sl * 0x94d049bbu + sh * 0x133111ebu;  // hi(z * C2)
}

__device__ __noinline__ uint32_t quant_slow(float h, float lo, float hi, uint32_t levels,
                                            uint64_t z0, int q) {
  const uint64_t z = z0 + static_cast<uint64_t>(q - 1) * kPhi;  // counter e0 + q + 1
  QRow R;
  R.lo = lo;
  R.scale = (static_cast<double>(hi) - R.lo) / static_cast<double>(levels);
  R.rcp = __drcp_rn(R.scale);
  R.x_hi = __ddiv_rn(__dsub_rn(static_cast<double>(hi), R.lo), R.scale);
  R.hi = hi;
  R.levels = levels;
  bool sl;
  const uint32_t c = quant_fast(h, R, z, sl);
  return sl ? quant_exact(h, R.lo, R.scale, static_cast<double>(levels), z) : c;
}

__device__ __forceinline__ float fmin_nan(float a, float b) {  // NaN-propagating min
  float r;
  asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// 4 byte containers (codes < 2^b) -> 4*b packed bits, LSB first
// (flagged elements hold arbitrary bytes until patched: mask them to the width)
__device__ __forceinline__ uint32_t pack4x4(uint32_t w) {
  w &= 0x0f0f0f0fu;
  w = (w | (w >> 4)) & 0x00ff00ffu;
  return (w | (w >> 8)) & 0xffffu;
}
__device__ __forceinline__ uint32_t pack4x2(uint32_t w) {
  w &= 0x03030303u;
  w = (w | (w >> 6)) & 0x000f000fu;
  return (w | (w >> 12)) & 0xffu;
}

template <int EPL, int MINB, bool YD>
__global__ void __launch_bounds__(256, MINB) k_quantize_pack_grp(
    const float* __restrict__ values, int64_t ld, int dim, int64_t n, int lg,
    const int32_t* __restrict__ rows, const uint32_t* __restrict__ ids,
    const uint8_t* __restrict__ bits, const uint64_t* __restrict__ offsets,
    const uint16_t* __restrict__ set_of, const uint64_t* __restrict__ set_keys,
    uint8_t* __restrict__ out, float* __restrict__ win_lo, float* __restrict__ win_hi,
    int* __restrict__ err, uint32_t env) {
  constexpr int CPL = EPL / 4;  // float4 chunks per lane
  constexpr int NW = EPL / 4;   // byte-container words per lane
  const int lane = threadIdx.x & 31;
  const int G = 1 << lg;
  const int j = lane & (G - 1);
  const int mpw = 32 >> lg;
  const unsigned gm = G == 32 ? 0xffffffffu : ((1u << G) - 1u) << (lane & ~(G - 1));
  const int nchunk = (dim + 3) >> 2;
  const int e0 = j * EPL;
  const int nvalid = min(max(dim - e0, 0), EPL);  // valid elements of this lane
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarp = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t base = warp * mpw; base < n; base += nwarp * mpw) {
    int64_t m = base + (lane >> lg);
    const bool live = m < n;
    if (!live) m = n - 1;  // idle group: recompute the last message, store nothing
    const float* row = values + static_cast<int64_t>(rows[m]) * ld;
    float v[EPL];
#pragma unroll
    for (int k = 0; k < CPL; ++k) {
      const int c = j * CPL + k;
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < nchunk) t = __ldg(reinterpret_cast<const float4*>(row) + c);
      v[4 * k] = t.x, v[4 * k + 1] = t.y, v[4 * k + 2] = t.z, v[4 * k + 3] = t.w;
    }
    if (nvalid < EPL && nvalid > 0) {  // tail lane: pad with a valid element
#pragma unroll
      for (int q = 1; q < EPL; ++q)
        if (q >= nvalid) v[q] = v[0];
    }
    // extrema; NaN propagates into lo, +-inf shows in lo/hi: finite <=> both finite
    float lo = INFINITY, hi = -INFINITY;
    bool negz = false;
    if (nvalid > 0) {
#pragma unroll
      for (int q = 0; q < EPL; ++q) {
        lo = fmin_nan(lo, v[q]);
        hi = fmaxf(hi, v[q]);
        negz |= __float_as_uint(v[q]) == 0x80000000u;
      }
    }
    for (int o = G >> 1; o > 0; o >>= 1) {
      lo = fmin_nan(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    const bool finite = fabsf(lo) < INFINITY && fabsf(hi) < INFINITY;
    negz = (__ballot_sync(0xffffffffu, negz) & gm) != 0;
    // first-occurrence signed zero (quant.hpp:63-68); only when a -0.0 is present
    const bool needz = negz && (lo == 0.f || hi == 0.f);
    if (__any_sync(0xffffffffu, needz)) {
      int zk = 0x7fffffff;  // (index << 1) | sign of this lane's first zero
#pragma unroll
      for (int q = EPL - 1; q >= 0; --q)
        if (q < nvalid && v[q] == 0.f) zk = ((e0 + q) << 1) | int(__float_as_uint(v[q]) >> 31);
      for (int o = G >> 1; o > 0; o >>= 1) zk = min(zk, __shfl_xor_sync(0xffffffffu, zk, o));
      if (needz) {
        const float z0 = (zk & 1) ? -0.f : 0.f;
        if (lo == 0.f) lo = z0;
        if (hi == 0.f) hi = z0;
      }
    }
    if (!live) continue;
    if (j == 0 && win_lo) {  // trace.hpp:86-91 (update precedes encode, engine.hpp:487)
      const float wl = win_lo[m], wh = win_hi[m];
      win_lo[m] = lo < wl ? lo : wl;
      win_hi[m] = wh < hi ? hi : wh;
    }
    const int b = bits[m];
    uint8_t* chunk = out + offsets[m];
    if (b == 0) {  // BitMode::kFp: raw row (engine.hpp:473-481)
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int c = j * CPL + k;
        if (c < nchunk)
          reinterpret_cast<float4*>(chunk)[c] =
              make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      }
      continue;
    }
    if (b != 2 && b != 4 && b != 8) {
      if (j == 0) atomicOr(err, kErrBadWidth);
      continue;
    }
    if (!finite) {
      if (j == 0) atomicOr(err, kErrNonFinite);
      continue;
    }
    const double lo_d = lo, hi_d = hi;
    const uint32_t levels = (1u << b) - 1;
    const bool constant = hi_d == lo_d;
    const double scale = constant ? 0.0 : (hi_d - lo_d) / static_cast<double>(levels);
    if (j == 0) {
      uint4 h;
      h.x = __float_as_uint(static_cast<float>(scale));
      h.y = __float_as_uint(lo);
      h.z = static_cast<uint32_t>(dim);
      h.w = env_word(b, env, set_of, m);
      *reinterpret_cast<uint4*>(chunk) = h;
    }
    uint32_t w8[NW];  // codes in byte containers, element q in byte q & 3 of word q >> 2
#pragma unroll
    for (int k = 0; k < NW; ++k) w8[k] = 0;
    // elements left to the exact path: bit q = element e0 + q (patched after the stores)
    uint32_t slow = 0, hib = 0, Tb = 0, Ab = 0;
    uint64_t z0 = 0;
    bool f32ok = true;
    if (!constant && nvalid > 0) {  // hi == lo: S = 0, zero payload, no draws (quant.hpp:74-78)
      if (nvalid < EPL) {  // tail lane: padding elements encode as h == lo (code 0)
#pragma unroll
        for (int q = 1; q < EPL; ++q)
          if (q >= nvalid) v[q] = lo;
      }
      const uint64_t key = rng_fork(set_keys[set_of ? set_of[m] : 0], ids[m]);
      f32ok = scale >= 0x1.0p-100 && scale <= 0x1.0p+100;
      const float rf = __double2float_rn(__drcp_rn(scale));
      z0 = key + static_cast<uint64_t>(e0 + 2) * kPhi;  // pre-mix state, counter e0 + 1
      if constexpr (YD) {
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          uint32_t c4[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int q = 4 * k + r;
            const uint64_t zq = z0 + static_cast<uint64_t>(q) * kPhi;
            const uint32_t top = draw_top32(static_cast<uint32_t>(zq), static_cast<uint32_t>(zq >> 32));
            const float vv = 2.f - __uint_as_float(__funnelshift_r(top, 0x7fu, 9));  // 1 - u_f
            const float y = __fmaf_rn(v[q] - lo, rf, vv);
            const uint32_t t = __float_as_uint(__fadd_rz(y, 512.f));  // 512 + floor(y * 2^14) / 2^14
            c4[r] = t >> 14;                                        // floor(y) in the low byte
            if (((t + 2u) & 0x3fffu) < 4u) slow |= 1u << q;         // within 2^-13 of an integer
          }
          w8[k] = __byte_perm(__byte_perm(c4[0], c4[1], 0x0040), __byte_perm(c4[2], c4[3], 0x0040),
                              0x5410);
        }
        if (nvalid < EPL) {  // tail lane: padding bytes are zero, never patched
#pragma unroll
          for (int k = 0; k < NW; ++k) {
            const int nb = nvalid - 4 * k;
            w8[k] &= nb >= 4 ? 0xffffffffu : nb <= 0 ? 0u : (1u << (8 * nb)) - 1u;
          }
          slow &= (1u << nvalid) - 1u;
        }
      } else {
      // h == hi has x = x_hi exactly: code = floor(x_hi) + (u < frac_hi).  With
      // K = frac_hi * 2^23 and k the draw's top 23 bits, u < frac_hi <=> k < floor(K)
      // unless K is fractional and k == floor(K) (probability 2^-23: exact path).
      const double x_hi = __ddiv_rn(__dsub_rn(hi_d, lo_d), scale);
      const double hbd = floor(x_hi);
      if (hbd < static_cast<double>(levels)) {
        const double K = __dmul_rn(__dsub_rn(x_hi, hbd), 8388608.0);
        const double Kf = floor(K);
        hib = static_cast<uint32_t>(hbd);
        Tb = 0x3f800000u | static_cast<uint32_t>(Kf);
        Ab = K != Kf ? Tb : 0u;
      } else {
        hib = levels;  // min(floor(x_hi) + inc, levels) = levels
      }
      const float dl = static_cast<float>(levels) * 0x1.0p-22f;
      const float hw = 0.5f - dl - 0x1.0p-24f;  // |fr - 1/2| > hw  <=>  dl <= fr <= 1 - dl
      const float dd = dl + 0x1.0p-22f;
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        uint32_t c4[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int q = 4 * k + r;
          const uint64_t zq = z0 + static_cast<uint64_t>(q) * kPhi;
          const uint32_t top = draw_top32(static_cast<uint32_t>(zq), static_cast<uint32_t>(zq >> 32));
          const float u = __uint_as_float(__funnelshift_r(top, 0x7fu, 9)) - 1.f;  // u_f in [0,1)
          const float h = v[q];
          const float a = h - lo;
          const float x = a * rf;
          const float mm = __fadd_rz(x, 8388608.f);  // 2^23 + floor(x) for 0 <= x < 2^23
          const float fr = x - (mm - 8388608.f);
          const float d = u - fr;
          // low byte: floor(x) + (u < fr), the sign of d (d = +0 when equal)
          c4[r] = __float_as_uint(mm) + (__float_as_uint(d) >> 31);
          const bool s = ((a != 0.f) & ((fabsf(fr - 0.5f) > hw) | (fabsf(d) <= dd))) | (h == hi);
          if (s) slow |= 1u << q;
        }
        w8[k] = __byte_perm(__byte_perm(c4[0], c4[1], 0x0040), __byte_perm(c4[2], c4[3], 0x0040),
                            0x5410);
      }
      }
      if (!f32ok) slow = nvalid == 32 ? 0xffffffffu : (1u << nvalid) - 1u;
    }
    // LSB-first payload, zero padded to 16 bytes; the lane's run is EPL*b/8 bytes
    uint8_t* payload = chunk + kHdrGpu;
    const int pb = static_cast<int>(((packed_bytes(dim, b) + 15) / 16) * 16);
    if (b == 8) {
#pragma unroll
      for (int k = 0; k < NW; k += 4) {
        const int off = e0 + 4 * k;
        if (off < pb)
          *reinterpret_cast<uint4*>(payload + off) = make_uint4(w8[k], w8[k + 1], w8[k + 2], w8[k + 3]);
      }
    } else if (b == 4) {
      uint32_t p[NW / 2];
#pragma unroll
      for (int k = 0; k < NW / 2; ++k) p[k] = pack4x4(w8[2 * k]) | pack4x4(w8[2 * k + 1]) << 16;
      const int off = e0 / 2;
      if constexpr (NW / 2 == 2) {
        if (off < pb) *reinterpret_cast<uint2*>(payload + off) = make_uint2(p[0], p[1]);
      } else {
#pragma unroll
        for (int k = 0; k < NW / 2; k += 4)
          if (off + 4 * k < pb)
            *reinterpret_cast<uint4*>(payload + off + 4 * k) = make_uint4(p[k], p[k + 1], p[k + 2], p[k + 3]);
      }
    } else {
      uint32_t p[NW / 4];
#pragma unroll
      for (int k = 0; k < NW / 4; ++k)
        p[k] = pack4x2(w8[4 * k]) | pack4x2(w8[4 * k + 1]) << 8 | pack4x2(w8[4 * k + 2]) << 16 |
               pack4x2(w8[4 * k + 3]) << 24;
      const int off = e0 / 4;
      if constexpr (NW / 4 == 1) {
        if (off < pb) *reinterpret_cast<uint32_t*>(payload + off) = p[0];
      } else {
        if (off < pb) *reinterpret_cast<uint2*>(payload + off) = make_uint2(p[0], p[1]);
      }
    }
    // lanes cover G*EPL*b/8 bytes; the rest of the 16-byte padding (small dims)
    for (int off = G * EPL * b / 8 + 4 * j; off < pb; off += 4 * G)
      *reinterpret_cast<uint32_t*>(payload + off) = 0u;
    // flagged elements (h == hi, ~2e-4 near a decision boundary, or every element
    // when S is outside the fp32 window): exact code patched into the payload this
    // lane just wrote (its own bytes; same-thread order)
    while (slow) {
      const int q = __ffs(slow) - 1;
      slow &= slow - 1;
      const float h = row[e0 + q];
      uint32_t c;
      const uint32_t ub = !YD && f32ok && h == hi
                              ? __funnelshift_r(draw_top32(static_cast<uint32_t>(z0 + q * kPhi),
                                                           static_cast<uint32_t>((z0 + q * kPhi) >> 32)),
                                                0x7fu, 9)
                              : 0u;
      if (ub != 0u && ub != Ab)
        c = min(hib + (ub < Tb ? 1u : 0u), levels);
      else
        c = quant_slow(h, lo, hi, levels, z0, q);
      const int e = e0 + q;
      if (b == 8) {
        payload[e] = static_cast<uint8_t>(c);
      } else {
        const int sh = b == 4 ? (e & 1) * 4 : (e & 3) * 2;
        uint8_t* p = payload + (b == 4 ? e >> 1 : e >> 2);
        *p = static_cast<uint8_t>((*p & ~(levels << sh)) | (c << sh));
      }
    }
  }
}

// Decode counterpart: lane l writes the float4 chunks c = l + 32 i of the row.
__global__ void __launch_bounds__(256) k_dequant_f32(
    const uint8_t* __restrict__ in, int64_t n, int dim, const uint8_t* __restrict__ bits,
    const uint64_t* __restrict__ offsets, const int32_t* __restrict__ dst_rows, int accumulate,
    float* __restrict__ out, int64_t ld, int* __restrict__ err, const uint32_t* __restrict__ expect,
    const float* __restrict__ mask,
    int64_t ldm) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t m = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; m < n;
       m += wstride) {
  const uint8_t* chunk = in + offsets[m];
  const int b = bits[m];
  float* dst = out + (dst_rows ? static_cast<int64_t>(dst_rows[m]) : m) * ld;
  const int nchunk = (dim + 3) >> 2;
  if (b == 0) {
    const float* src = reinterpret_cast<const float*>(chunk);
    const int64_t mr = dst_rows ? static_cast<int64_t>(dst_rows[m]) : m;
    for (int j = lane; j < dim; j += 32) {
      bool keep = true;
      if (mask)
        keep = ldm < 0 ? ((__ldg(reinterpret_cast<const uint32_t*>(mask) + mr * (-ldm) + (j >> 5)) >>
                           (j & 31)) & 1u) != 0
                       : mask[mr * ldm + j] > 0.f;
      const float v = keep ? src[j] : 0.f;
      dst[j] = accumulate ? dst[j] + v : v;
    }
    continue;
  }
  const uint4 h = *reinterpret_cast<const uint4*>(chunk);
  if (static_cast<int>(h.w & 0xff) != b || h.z != static_cast<uint32_t>(dim)) {
    if (lane == 0) atomicOr(err, kErrDecode);
    continue;
  }
  if (expect && (h.w >> 8) != expect[m]) {  // misrouted / plan-version skew (engine.hpp:530-541)
    if (lane == 0) atomicOr(err, kErrProtocol);
    continue;
  }
  const float sc = __uint_as_float(h.x), zp = __uint_as_float(h.y);
  const uint8_t* payload = chunk + kHdrGpu;
  const uint32_t cmask = (1u << b) - 1;
  for (int c = lane; c < nchunk; c += 32) {
    uint32_t word;
    if (b == 8)
      word = reinterpret_cast<const uint32_t*>(payload)[c];
    else if (b == 4)
      word = reinterpret_cast<const uint16_t*>(payload)[c];
    else
      word = payload[c];
    float r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = fmaf(static_cast<float>((word >> (q * b)) & cmask), sc, zp);
    if (mask) {  // ReLU backward folded into the scatter-add (see spmm.cu:relu_mask4)
      const uint32_t mb =
          relu_bits4(mask, ldm, dst_rows ? static_cast<int64_t>(dst_rows[m]) : m, 4 * c);
      r[0] = (mb & 1u) ? r[0] : 0.f;
      r[1] = (mb & 2u) ? r[1] : 0.f;
      r[2] = (mb & 4u) ? r[2] : 0.f;
      r[3] = (mb & 8u) ? r[3] : 0.f;
    }
    if (4 * c + 3 < dim) {
      float4* d4 = reinterpret_cast<float4*>(dst) + c;
      if (accumulate) {
        const float4 o = *d4;
        *d4 = make_float4(o.x + r[0], o.y + r[1], o.z + r[2], o.w + r[3]);
      } else {
        *d4 = make_float4(r[0], r[1], r[2], r[3]);
      }
    } else {
      for (int q = 0; q < 4 && 4 * c + q < dim; ++q)
        dst[4 * c + q] = accumulate ? dst[4 * c + q] + r[q] : r[q];
    }
  }
  }
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" {

uint64_t qgnn_packed_bytes(uint64_t count, int bits) { return packed_bytes(count, bits); }

uint64_t qgnn_chunk_wire_bytes(uint64_t count, int bits, int layout, int dtype) {
  return chunk_bytes(count, bits, layout, dtype == QGNN_F64 ? 8 : 4);
}

int qgnn_wire_layout(const int32_t* bits, int64_t n, int64_t dim, int layout, int dtype,
                     int64_t* wire_pos, uint64_t* offsets, uint64_t* total) {
  QGNN_API_BEGIN
  const int elem = dtype == QGNN_F64 ? 8 : 4;
  uint64_t off = 0;
  int64_t k = 0;
  for (int64_t i = 0; i < n; ++i)
    QGNN_REQUIRE(bits[i] == 0 || bits[i] == 2 || bits[i] == 4 || bits[i] == 8, QGNN_EINVAL,
                 "encode_message_set: bit width must be 2, 4, or 8");
  for (int b : {0, 2, 4, 8}) {
    for (int64_t i = 0; i < n; ++i) {
      if (bits[i] != b) continue;
      if (wire_pos) wire_pos[k] = i;
      ++k;
      offsets[i] = off;
      off += chunk_bytes(static_cast<uint64_t>(dim), b, layout, elem);
    }
  }
  *total = off;
  QGNN_API_END
}

int qgnn_decode_validate(const uint8_t* bits, const uint64_t* offsets, const uint64_t* dims,
                         int64_t n, int layout, int dtype, uint64_t total_bytes,
                         uint64_t n_bytes) {
  QGNN_API_BEGIN
  const int elem = dtype == QGNN_F64 ? 8 : 4;
  QGNN_REQUIRE(n_bytes == total_bytes, QGNN_EDECODE, "message set: byte count mismatch");
  uint64_t expect = 0;
  for (int64_t k = 0; k < n; ++k) {
    QGNN_REQUIRE(offsets[k] == expect, QGNN_EDECODE, "message set: index offsets not contiguous");
    const int b = bits[k];
    QGNN_REQUIRE(b == 2 || b == 4 || b == 8 || b == 0, QGNN_EDECODE, "chunk: bad bit width");
    const uint64_t cb = chunk_bytes(dims[k], b, layout, elem);
    QGNN_REQUIRE(b == 0 || offsets[k] + (layout == QGNN_WIRE_REF ? kHdrRef : kHdrGpu) <= n_bytes,
                 QGNN_EDECODE, "chunk: truncated header");
    QGNN_REQUIRE(offsets[k] + cb <= n_bytes, QGNN_EDECODE, "chunk: truncated payload");
    expect = offsets[k] + cb;
  }
  QGNN_REQUIRE(expect == n_bytes, QGNN_EDECODE, "message set: trailing bytes");
  QGNN_API_END
}

int qgnn_quantize_pack(qgnn_ctx* ctx, const void* values, int dtype, int64_t ld, int64_t dim,
                       int64_t n, const int32_t* rows, const uint32_t* ids, const uint8_t* bits,
                       const uint64_t* offsets, const uint16_t* set_of, const uint64_t* set_keys,
                       int layout, uint8_t* out, void* win_lo, void* win_hi, uint32_t envelope,
                       void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "quantize_pack: null context");
  QGNN_REQUIRE(dim > 0, QGNN_EINVAL, "quantize: empty input");
  if (n == 0) return QGNN_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(n * 32, threads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool fast = dtype == QGNN_F32 && layout == QGNN_WIRE_GPU && ld % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(values) & 15) == 0 && dim <= 1024;
  static const int grp = [] {
    const char* e = std::getenv("QGNN_K1_GRP");  // 0: the round-1 lean kernel
    return e ? std::atoi(e) : 1;
  }();
  if (fast && grp) {
    static const int epl_env = [] {
      const char* e = std::getenv("QGNN_K1_EPL");  // 16 or 32 elements per lane (default 32)
      return e ? std::atoi(e) : 32;
    }();
    const int epl = (epl_env == 16 && dim <= 512) ? 16 : 32;
    int lg = 0;
    while ((int64_t(1) << lg) * epl < dim) ++lg;
    const int64_t per_cta = (256 / 32) * (32 >> lg);  // messages per CTA per sweep
    const int minb = epl == 16 ? 4 : 3;
    const int64_t gblocks = std::min<int64_t>(ceil_div(n, per_cta), int64_t(ctx->num_sms) * minb);
    auto* v = static_cast<const float*>(values);
    auto* wl = static_cast<float*>(win_lo);
    auto* wh = static_cast<float*>(win_hi);
    const int d = static_cast<int>(dim);
    static const bool yd = [] {  // QGNN_K1_YDOM=0: the x-domain decision (round 2 first cut)
      const char* e = std::getenv("QGNN_K1_YDOM");
      return !e || std::atoi(e) != 0;
    }();
#define QGNN_K1_GRP(E, MB, Y)                                                                       \
  k_quantize_pack_grp<E, MB, Y><<<gblocks, 256, 0, s>>>(v, ld, d, n, lg, rows, ids, bits, offsets,  \
                                                       set_of, set_keys, out, wl, wh, ctx->d_err,  \
                                                       envelope)
    if (epl == 16) {
      if (yd)
        QGNN_K1_GRP(16, 4, true);
      else
        QGNN_K1_GRP(16, 4, false);
    } else {
      if (yd)
        QGNN_K1_GRP(32, 3, true);
      else
        QGNN_K1_GRP(32, 3, false);
    }
#undef QGNN_K1_GRP
  } else if (fast) {
    const int64_t fblocks = std::min<int64_t>(blocks, int64_t(ctx->num_sms) * 16);
    const int nv = static_cast<int>(ceil_div(ceil_div(dim, 4), 32));
    auto* v = static_cast<const float*>(values);
    auto* wl = static_cast<float*>(win_lo);
    auto* wh = static_cast<float*>(win_hi);
    const int d = static_cast<int>(dim);
    static const int minb = [] {
      const char* e = std::getenv("QGNN_K1_MINB");  // occupancy target (measured best: 4)
      return e ? std::atoi(e) : 4;
    }();
    static const bool lean = [] {
      const char* e = std::getenv("QGNN_K1_LEAN");
      return !e || std::atoi(e) != 0;
    }();
#define QGNN_K1_LAUNCH(NVV, MB)                                                                     \
  if (lean && d % 4 == 0)                                                                           \
    k_quantize_pack_lean<NVV, MB><<<fblocks, threads, 0, s>>>(v, ld, d, n, rows, ids, bits, offsets, \
                                                             set_of, set_keys, out, wl, wh,         \
                                                             ctx->d_err, envelope);                 \
  else                                                                                              \
    k_quantize_pack_f32<NVV, MB><<<fblocks, threads, 0, s>>>(v, ld, d, n, rows, ids, bits, offsets,  \
                                                            set_of, set_keys, out, wl, wh, ctx->d_err, \
                                                            envelope)
#define QGNN_K1_NV(NVV)                 \
  if (minb >= 4)                        \
    QGNN_K1_LAUNCH(NVV, 4);             \
  else if (minb == 3)                   \
    QGNN_K1_LAUNCH(NVV, 3);             \
  else                                  \
    QGNN_K1_LAUNCH(NVV, 1);
    if (nv <= 1) {
      QGNN_K1_NV(1)
    } else if (nv <= 2) {
      QGNN_K1_NV(2)
    } else if (nv <= 4) {
      QGNN_K1_NV(4)
    } else {
      QGNN_K1_NV(8)
    }
#undef QGNN_K1_NV
#undef QGNN_K1_LAUNCH
  } else if (dtype == QGNN_F64)
    k_quantize_pack<double><<<blocks, threads, 0, s>>>(
        static_cast<const double*>(values), ld, static_cast<int>(dim), n, rows, ids, bits, offsets,
        set_of, set_keys, layout, out, static_cast<double*>(win_lo), static_cast<double*>(win_hi),
        ctx->d_err, envelope);
  else
    k_quantize_pack<float><<<blocks, threads, 0, s>>>(
        static_cast<const float*>(values), ld, static_cast<int>(dim), n, rows, ids, bits, offsets,
        set_of, set_keys, layout, out, static_cast<float*>(win_lo), static_cast<float*>(win_hi),
        ctx->d_err, envelope);
  check_launch("k_quantize_pack");
  QGNN_API_END
}

int qgnn_dequant_scatter(qgnn_ctx* ctx, const uint8_t* in, int64_t n, int64_t dim,
                         const uint8_t* bits, const uint64_t* offsets, int layout,
                         const int32_t* dst_rows, int accumulate, void* out, int dtype,
                         int64_t ld, const uint32_t* expect_envelope, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx, QGNN_EINVAL, "dequant_scatter: null context");
  if (n == 0) return QGNN_OK;
  const int threads = 256;
  const int64_t blocks = ceil_div(n * 32, threads);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool fast = dtype == QGNN_F32 && layout == QGNN_WIRE_GPU && ld % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (fast)
    k_dequant_f32<<<std::min<int64_t>(blocks, int64_t(ctx->num_sms) * 16), threads, 0, s>>>(
        in, n, static_cast<int>(dim), bits, offsets, dst_rows, accumulate, static_cast<float*>(out),
        ld, ctx->d_err, layout == QGNN_WIRE_GPU ? expect_envelope : nullptr, nullptr, 0);
  else if (dtype == QGNN_F64)
    k_dequant_scatter<double><<<blocks, threads, 0, s>>>(in, n, static_cast<int>(dim), bits,
                                                         offsets, layout, dst_rows, accumulate,
                                                         static_cast<double*>(out), ld, ctx->d_err,
                                                         layout == QGNN_WIRE_GPU ? expect_envelope
                                                                                 : nullptr);
  else
    k_dequant_scatter<float><<<blocks, threads, 0, s>>>(in, n, static_cast<int>(dim), bits,
                                                        offsets, layout, dst_rows, accumulate,
                                                        static_cast<float*>(out), ld, ctx->d_err,
                                                        layout == QGNN_WIRE_GPU ? expect_envelope
                                                                                : nullptr);
  check_launch("k_dequant_scatter");
  QGNN_API_END
}

}  // extern "C"

namespace qgnn_b200 {
// Backward scatter-add, one launch: warp per destination row; the row's
// incoming chunks (ascending source, engine.hpp:720-734) are decoded and summed
// in registers, masked by the ReLU of h (when given) and added to out once.
// The kernel is a chain of dependent loads (row list -> message -> offset ->
// chunk), so everything that does not depend on the messages — the destination
// row and its mask bits — is loaded before the chain starts, and a chunk's
// header and payload are loaded together (the payload is used only if the
// header checks pass; its bytes lie inside the arena either way).  KC float4
// chunks per lane: 128 * KC columns per grid.y slice.
// 24 CTAs (48 warps) per SM: 38 registers, +40 % warps in flight for the load
// chains over the unconstrained 49 (profiles/ab_k3_occ_r2.txt)
template <int KC>
__global__ void __launch_bounds__(64, 24) k_dequant_rows_f32(
    const uint8_t* __restrict__ in, int64_t n_rows, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ ptr, const int32_t* __restrict__ msg,
    const int32_t* __restrict__ words, int dim,
    const uint8_t* __restrict__ bits, const uint64_t* __restrict__ offsets,
    float* __restrict__ out, int64_t ld, const float* __restrict__ mask, int64_t ldm,
    int* __restrict__ err, const uint32_t* __restrict__ expect) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (g >= n_rows) return;
  const int nchunk = (dim + 3) >> 2;
  constexpr int kMaxC = KC;
  const int cbase = blockIdx.y * 32 * KC;
  const int64_t r = rows[g];
  const int j0 = ptr[g], j1 = ptr[g + 1];
  float4 prev[kMaxC];
  uint32_t mb[kMaxC];
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = cbase + lane + 32 * i;
    prev[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    mb[i] = 0xfu;
    if (c < nchunk && 4 * c + 3 < dim) {
      prev[i] = *reinterpret_cast<const float4*>(out + r * ld + 4 * c);
      if (mask) mb[i] = relu_bits4(mask, ldm, r, 4 * c);
    }
  }
  float4 acc[kMaxC];
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int j = j0; j < j1; ++j) {
    int m = -1;
    const uint8_t* chunk;
    int b;
    if (words) {  // chunk word: offset / 16 and width code, one load (rebuilt per plan)
      const uint32_t w = static_cast<uint32_t>(words[j]);
      chunk = in + (static_cast<uint64_t>(w & 0x3fffffffu) << 4);
      b = (0x8420 >> (4 * (w >> 30))) & 0xf;  // code 0..3 -> width 0, 2, 4, 8
    } else {
      m = msg[j];
      chunk = in + offsets[m];
      b = bits[m];
    }
    if (b == 0) {  // raw fp32 row (BitMode::kFp)
      const float4* src = reinterpret_cast<const float4*>(chunk);
#pragma unroll
      for (int i = 0; i < kMaxC; ++i) {
        const int c = cbase + lane + 32 * i;
        if (c < nchunk) {
          const float4 v = src[c];
          acc[i].x += v.x, acc[i].y += v.y, acc[i].z += v.z, acc[i].w += v.w;
        }
      }
      continue;
    }
    const uint4 h = *reinterpret_cast<const uint4*>(chunk);
    const uint8_t* payload = chunk + kHdrGpu;
    uint32_t word[kMaxC];
#pragma unroll
    for (int i = 0; i < kMaxC; ++i) {
      const int c = cbase + lane + 32 * i;
      word[i] = 0;
      if (c < nchunk)
        word[i] = b == 8 ? reinterpret_cast<const uint32_t*>(payload)[c]
                : b == 4 ? reinterpret_cast<const uint16_t*>(payload)[c]
                         : payload[c];
    }
    if (static_cast<int>(h.w & 0xff) != b || h.z != static_cast<uint32_t>(dim)) {
      if (lane == 0) atomicOr(err, kErrDecode);
      continue;
    }
    if (expect && (h.w >> 8) != expect[m < 0 ? msg[j] : m]) {
      if (lane == 0) atomicOr(err, kErrProtocol);
      continue;
    }
    const float sc = __uint_as_float(h.x), zp = __uint_as_float(h.y);
    const uint32_t cmask = (1u << b) - 1;
#pragma unroll
    for (int i = 0; i < kMaxC; ++i) {
      const int c = cbase + lane + 32 * i;
      if (c >= nchunk) continue;
      const uint32_t w = word[i];
      acc[i].x += fmaf(static_cast<float>(w & cmask), sc, zp);
      acc[i].y += fmaf(static_cast<float>((w >> b) & cmask), sc, zp);
      acc[i].z += fmaf(static_cast<float>((w >> (2 * b)) & cmask), sc, zp);
      acc[i].w += fmaf(static_cast<float>((w >> (3 * b)) & cmask), sc, zp);
    }
  }
#pragma unroll
  for (int i = 0; i < kMaxC; ++i) {
    const int c = cbase + lane + 32 * i;
    if (c >= nchunk) continue;
    float* o = out + r * ld + 4 * c;
    if (4 * c + 3 < dim) {
      const float4 a = apply_bits4(acc[i], mb[i]);
      float4 p = prev[i];
      p.x += a.x, p.y += a.y, p.z += a.z, p.w += a.w;
      *reinterpret_cast<float4*>(o) = p;
    } else {
      float4 a = acc[i];
      if (mask) a = apply_bits4(a, relu_bits4(mask, ldm, r, 4 * c));
      const float av[4] = {a.x, a.y, a.z, a.w};
      for (int q = 0; q < 4 && 4 * c + q < dim; ++q) o[q] += av[q];
    }
  }
}

// Chunk words for the packed-halo gathers (PackedHalo::direct): offset / 16 and the
// width code of message idx[e], one word per gather entry, rebuilt with every plan.
__global__ void k_encode_chunk_words(const int32_t* __restrict__ idx, int64_t n,
                                     const uint64_t* __restrict__ off,
                                     const uint8_t* __restrict__ bits, int32_t* __restrict__ out) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int32_t m = idx[e];
    const int b = bits[m];
    const uint32_t code = b == 8 ? 3u : b == 4 ? 2u : b == 2 ? 1u : 0u;
    out[e] = static_cast<int32_t>(static_cast<uint32_t>(off[m] >> 4) | code << 30);
  }
}
void encode_chunk_words(const int32_t* idx, int64_t n, const uint64_t* off, const uint8_t* bits,
                        int32_t* out, cudaStream_t s) {
  if (n <= 0) return;
  k_encode_chunk_words<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 148 * 32)), 256, 0, s>>>(
      idx, n, off, bits, out);
  check_launch("k_encode_chunk_words");
}

// Once per received message: the header's width and count against the index
// (DecodeError, codec.hpp:82-95) and its envelope against the receiver's
// expectation (ProtocolError, engine.hpp:530-541) — the checks the slot-indexed
// gather made per entry.
__global__ void k_check_chunk_headers(const uint8_t* __restrict__ arena,
                                      const uint64_t* __restrict__ off,
                                      const uint8_t* __restrict__ bits,
                                      const uint32_t* __restrict__ env, int64_t n, int dim,
                                      int* __restrict__ err) {
  for (int64_t m = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; m < n;
       m += int64_t(gridDim.x) * blockDim.x) {
    const int b = bits[m];
    if (b == 0) continue;  // raw rows carry no header
    const uint4 h = __ldg(reinterpret_cast<const uint4*>(arena + off[m]));
    if (static_cast<int>(h.w & 0xffu) != b || h.z != static_cast<uint32_t>(dim))
      atomicOr(err, kErrDecode);
    else if (env && (h.w >> 8) != env[m])
      atomicOr(err, kErrProtocol);
  }
}
void check_chunk_headers(const uint8_t* arena, const uint64_t* off, const uint8_t* bits,
                         const uint32_t* env, int64_t n, int dim, int* err, cudaStream_t s) {
  if (n <= 0) return;
  k_check_chunk_headers<<<unsigned(std::min<int64_t>(ceil_div(n, 256), 148 * 32)), 256, 0, s>>>(
      arena, off, bits, env, n, dim, err);
  check_launch("k_check_chunk_headers");
}

void dequant_rows_add_f32(qgnn_ctx* ctx, const uint8_t* in, int64_t n_rows, const int32_t* rows,
                          const int32_t* ptr, const int32_t* msg, const int32_t* words, int dim,
                          const uint8_t* bits,
                          const uint64_t* offsets, float* out, int64_t ld, const float* mask,
                          int64_t ldm, const uint32_t* expect, cudaStream_t s) {
  if (n_rows == 0) return;
  if (dim <= 256) {
    const dim3 grid(unsigned(ceil_div(n_rows * 32, 64)), 1);
    k_dequant_rows_f32<2><<<grid, 64, 0, s>>>(
        in, n_rows, rows, ptr, msg, words, dim, bits, offsets, out, ld, mask, ldm, ctx->d_err, expect);
  } else {
    const dim3 grid(unsigned(ceil_div(n_rows * 32, 64)), unsigned(ceil_div(dim, 512)));
    k_dequant_rows_f32<4><<<grid, 64, 0, s>>>(
        in, n_rows, rows, ptr, msg, words, dim, bits, offsets, out, ld, mask, ldm, ctx->d_err, expect);
  }
  check_launch("k_dequant_rows_f32");
}

// fp32 GPU-layout decode + scatter-add with the ReLU-backward mask (engine)
void dequant_add_masked_f32(qgnn_ctx* ctx, const uint8_t* in, int64_t n, int dim,
                            const uint8_t* bits, const uint64_t* offsets, const int32_t* dst_rows,
                            float* out, int64_t ld, const float* mask, int64_t ldm,
                            const uint32_t* expect, cudaStream_t s) {
  if (n == 0) return;
  const int64_t blocks = ceil_div(n * 32, 256);
  k_dequant_f32<<<std::min<int64_t>(blocks, int64_t(ctx->num_sms) * 16), 256, 0, s>>>(
      in, n, dim, bits, offsets, dst_rows, 1, out, ld, ctx->d_err, expect, mask, ldm);
  check_launch("k_dequant_f32");
}
}  // namespace qgnn_b200
