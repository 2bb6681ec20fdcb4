// gemm_tc.cu — K5 dense transform on the 5th-gen tensor cores (tcgen05, sm_100a).
//
// fp32-faithful GEMM via the 3xTF32 split: every operand x = hi + lo with
// hi = x with the low 13 mantissa bits cleared (exactly representable in
// TF32) and lo = x - hi; D = Ahi*Bhi + Ahi*Blo + Alo*Bhi accumulated in fp32
// in TMEM (relative error ~2^-21, vs ~2^-11 for plain TF32).
//
// Pipeline (one persistent CTA per SM, 12 warps):
//   warp 0      TMA producer: A tile (and, for the weight gradient, B tile)
//               for each 16-deep K chunk into a 2..6-stage smem ring
//   warp 1      MMA issuer: one elected thread issues 2 k-steps x 3 products of
//               tcgen05.mma.cta_group::1.kind::tf32 (M=128, N=BN) per chunk
//   warp 2      TMEM allocator (2 x BN fp32 accumulator columns, double buffer)
//   warps 4-7   epilogue: tcgen05.ld 32x32b -> ReLU -> global stores, while the
//               MMA warp already accumulates the next tile in the other buffer
//   warps 8-11  converters: lo = x - tf32(x) of the landed fp32 tile into a
//               second buffer (the MMA reads the tile itself as hi: kind::tf32
//               ignores the low 13 mantissa bits), fence.proxy.async, release
// Shapes: forward z = A W (A rows x din, K-major), input gradient dz W^T
// (K-major, SWIZZLE_128B), weight gradient A^T B over rows (both operands
// MN-major; 32-bit MN-major operands require the 128B swizzle with 32-byte
// atoms, TMA SWIZZLE_128B_ATOM_32B / UMMA SWIZZLE_128B_BASE32B; split-K over
// rows with a fixed-order reduction).  B for the first two is the small
// weight matrix, pre-split into padded hi/lo K-major copies by k_prep_b.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"

namespace qgnn_b200 {
namespace tc {

constexpr int kBM = 128;
constexpr int kBK = 16;         // fp32 K elements per chunk (64-byte K-major rows)
constexpr int kMaxStages = 6;   // ring depth is chosen per launch from the smem budget
constexpr int kThreads = 512;  // 16 warps: warps 12-15 are the optional second epilogue group

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// Multicast variant: the box lands at the same smem offset in every CTA of
// `mask` and completes tx bytes on each destination's barrier at `bar`'s offset.
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar,
                                               int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::"
      "cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// arrive once on the barrier at `bar`'s offset in every CTA of `mask`
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// 16 consecutive accumulator columns of this thread's TMEM lane (no wait)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// SW128 shared-memory matrix descriptor (tcgen05 "version 1")
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout = 2) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t{1} << 46;  // version
  d |= uint64_t(layout) << 61;  // 2 = SW128, 4 = SW64, 1 = SW128_BASE32B
  return d;
}

__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

// lo = x - tf32(x) for `n16` 16-byte vectors, strided over `nthr` threads.  The hi
// part needs no copy: kind::tf32 reads only the top 19 bits of each 32-bit
// operand (verified bit-identical against an explicit truncated copy,
// profiles/chk_tc_trunc.py), so the landed fp32 tile is used as hi in place.
__device__ __forceinline__ void st_shared4(uint32_t a, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}
__device__ __forceinline__ float4 ld_shared4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
// buf / lo: shared-space byte addresses (explicit ld/st.shared, not generic)
__device__ __forceinline__ void split_tile(uint32_t buf, uint32_t lo, int n16, int t, int nthr) {
  for (int i = t; i < n16; i += nthr) {
    const float4 v = ld_shared4(buf + 16u * uint32_t(i));
    st_shared4(lo + 16u * uint32_t(i), make_float4(v.x - tf32_hi(v.x), v.y - tf32_hi(v.y),
                                                   v.z - tf32_hi(v.z), v.w - tf32_hi(v.w)));
  }
}

struct Params {
  int M, N, K;          // logical GEMM (C[M x N] = A[M x K] B[K x N])
  int BN;               // N tile (multiple of 16 / 32 for MN-major B), <= 256
  int tmem_cols;        // columns per accumulator buffer (pow2 >= BN)
  int m_tiles, splits, k_chunks, chunks_per_split;
  int stages;
  float* out;
  int64_t ldo;
  int relu;
  const float* mask;  // optional ReLU-backward mask: out = v * 1[mask > 0] (same row/col layout)
  int64_t ldm;
  int mh;  // M halves per tile (MN-major path): 2 = 256-row tiles, the two TMEM buffers hold
           // the two halves, so the N operand is read once per 256 output rows
  int dbg;  // QGNN_GEMM_DEBUG bit mask for bottleneck isolation (results invalid when set):
            // 1 = no MMAs, 2 = no output stores, 4 = no lo split, 8 = TMA producer only
  int bk;  // K elements per chunk: 16 (SW64, 64-byte rows) or 32 (SW128, K-major only)
  uint32_t* bits_out;        // relu: 1[out > 0] as 32-column words per row (pitch ldbo)
  int64_t ldbo;
  const uint32_t* bits_in;   // ReLU-backward mask as such words (pitch ldbi), or mask
  int64_t ldbi;
  int conv2;  // warps 12-15 join the converters (8 warps split each landed tile): the
              // weight gradient, whose converters split both operands of every chunk
  int epi2;  // K-major: a second epilogue warp group (warps 12-15) drains the upper half
             // of each tile's columns (wide outputs of short-K products, where the
             // epilogue, not the MMA, paces the tile)
  int cs;  // K-major: CTAs per cluster sharing each B stage (1, 2, 4).  Rank r loads
           // B rows [r BN/cs, (r+1) BN/cs) once and multicasts them to the cluster; a
           // stage is refilled when every CTA's MMAs have drained it (empty count = cs)
};

// kMN = false: A K-major (tmA box {32, 128}), B/Blo K-major prepared (box {32, BN})
// kMN = true : A MN-major (box {32 m, 32 k}), B MN-major (box {32 n, 32 k}); both split here
template <bool kMN>
__global__ void __launch_bounds__(kThreads, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmBlo, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int bk = kMN ? kBK : p.bk;
  const int a_bytes = kBM * bk * 4 * p.mh;  // 8 / 16 KB per 128-row half
  const int b_bytes = p.BN * bk * 4;       // BN x 64 / 128 B
  const int stage_bytes = 2 * a_bytes + 2 * b_bytes;
  const int kStages = p.stages;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * stage_bytes);
  uint64_t* full = bars;                    // [kMaxStages]
  uint64_t* conv = bars + kMaxStages;       // [kMaxStages]
  uint64_t* empty = bars + 2 * kMaxStages;  // [kMaxStages]
  uint64_t* tfull = bars + 3 * kMaxStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // epilogue staging: per epilogue warp a 32 x 32 fp32 block, row pitch 36 floats
  float* stage_out = reinterpret_cast<float*>(smem + kStages * stage_bytes + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = p.m_tiles * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], p.conv2 ? 8 : 4);  // one arrival per converter warp
      mbar_init(&empty[s], uint32_t(p.cs));
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], p.epi2 ? 8 : 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(2 * p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  if (p.cs > 1) cluster_sync();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint16_t cmask = uint16_t((1u << p.cs) - 1u);
  const int crank = p.cs > 1 ? int(cluster_rank()) : 0;

  auto tile_chunks = [&](int tile, int& m0, int& kc0, int& kc1, int& split) {
    const int mt = tile % p.m_tiles;
    split = tile / p.m_tiles;
    m0 = mt * kBM * p.mh;
    kc0 = split * p.chunks_per_split;
    kc1 = min(p.k_chunks, kc0 + p.chunks_per_split);
  };

  if ((p.dbg & 8) && warp != 0) {
    // isolation: producer alone (it waits for its own loads before reusing a stage)
  } else if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        int m0, kc0, kc1, split;
        tile_chunks(tile, m0, kc0, kc1, split);
        for (int kc = kc0; kc < kc1; ++kc) {
          if (p.dbg & 8)
            mbar_wait(&full[s], ph ^ 1);
          else
            mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * stage_bytes;
          uint8_t* A = st;
          uint8_t* B = st + 2 * a_bytes;
          uint8_t* Blo = B + b_bytes;
          const int k0 = kc * bk;
          if (!kMN) {
            mbar_expect_tx(&full[s], a_bytes + 2 * b_bytes);
            for (int h = 0; h < p.mh; ++h)
              tma_load_2d(A + h * (kBM * bk * 4), &tmA, &full[s], k0, m0 + kBM * h);
            if (p.cs == 1) {
              tma_load_2d(B, &tmB, &full[s], k0, 0);
              tma_load_2d(Blo, &tmBlo, &full[s], k0, 0);
            } else {  // this rank's slice of B rows, to every CTA of the cluster
              const int rows = p.BN / p.cs, off = crank * rows * bk * 4;
              tma_load_2d_mc(B + off, &tmB, &full[s], k0, crank * rows, cmask);
              tma_load_2d_mc(Blo + off, &tmBlo, &full[s], k0, crank * rows, cmask);
            }
          } else {
            mbar_expect_tx(&full[s], a_bytes + b_bytes);
            // 32-bit MN-major operands must use the 128B swizzle with 32-byte atoms
            // (TMA SWIZZLE_128B_ATOM_32B <-> UMMA SWIZZLE_128B_BASE32B): one box per
            // 32-wide MN group, kBK K rows of 128 B, groups 2 KB apart
            for (int j = 0; j < kBM * p.mh / 32; ++j)
              tma_load_2d(A + j * 2048, &tmA, &full[s], m0 + 32 * j, k0);
            for (int j = 0; j < p.BN / 32; ++j) tma_load_2d(B + j * 2048, &tmB, &full[s], 32 * j, k0);
          }
          if (++s == kStages) s = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kMN ? 1u : 0u) << 15) |
                           ((kMN ? 1u : 0u) << 16) | (uint32_t(p.BN >> 3) << 17) |
                           (uint32_t(kBM >> 4) << 24);
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      int m0, kc0, kc1, split;
      tile_chunks(tile, m0, kc0, kc1, split);
      // two accumulator buffers alternate between tiles, or (mh = 2) hold the
      // two 128-row halves of one tile
      const int acc = p.mh == 2 ? 0 : it & 1;
      const uint32_t aph = p.mh == 2 ? (it & 1) : ((it >> 1) & 1);
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + uint32_t(acc * p.tmem_cols);
      bool first = true;
      for (int kc = kc0; kc < kc1; ++kc) {
        mbar_wait(&full[s], ph);
        mbar_wait(&conv[s], ph);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* st = smem + s * stage_bytes;
          const uint32_t aH = smem_u32(st), aL = smem_u32(st + a_bytes);
          const uint32_t bH = smem_u32(st + 2 * a_bytes), bL = smem_u32(st + 2 * a_bytes + b_bytes);
#pragma unroll
          for (int j = 0; j < bk / 8; ++j) {
            uint64_t dAh, dAl, dBh, dBl;
            if (!kMN) {  // K-major SWIZZLE_64B / 128B: 8-row atoms of 64 / 128 B, +32 B per k-step
              const uint32_t sbo = bk == 32 ? 1024 : 512, lay = bk == 32 ? 2 : 4;
              dAh = sdesc(aH + 32 * j, 16, sbo, lay);
              dAl = sdesc(aL + 32 * j, 16, sbo, lay);
              dBh = sdesc(bH + 32 * j, 16, sbo, lay);
              dBl = sdesc(bL + 32 * j, 16, sbo, lay);
            } else {  // MN-major BASE32B: 4-row K atoms (SBO 512 B), MN groups 2 KB (LBO)
              dAh = sdesc(aH + 1024 * j, 2048, 512, 1);
              dAl = sdesc(aL + 1024 * j, 2048, 512, 1);
              dBh = sdesc(bH + 1024 * j, 2048, 512, 1);
              dBl = sdesc(bL + 1024 * j, 2048, 512, 1);
            }
            for (int h = 0; h < p.mh; ++h) {  // half h: rows 128h.. (MN groups 4h.. / SW64 atoms 16h..)
              const uint64_t hoff = uint64_t(h * (kBM * bk * 4)) >> 4;
              const uint32_t dh = d + uint32_t(h * p.tmem_cols);
              if (p.dbg & 1) continue;
              tc_mma(dh, dAh + hoff, dBh, idesc, first ? 0u : 1u);
              tc_mma(dh, dAh + hoff, dBl, idesc, 1u);
              tc_mma(dh, dAl + hoff, dBh, idesc, 1u);
            }
            first = false;
          }
          if (p.cs == 1)
            tc_commit(&empty[s]);
          else
            tc_commit_mc(&empty[s], cmask);  // frees stage s in every CTA's ring
        }
        __syncwarp();
        if (++s == kStages) s = 0, ph ^= 1;
      }
      if (lane == 0) tc_commit(&tfull[acc]);
      __syncwarp();
    }
  } else if ((warp >= 4 && warp < 8) || (warp >= 12 && p.epi2 && !kMN)) {
    // ---------------- epilogue (group 0: warps 4-7; with epi2, group 1: warps 12-15
    // takes the upper half of the 32-column groups)
    const int q = warp & 3;
    const int grp = warp >= 12 ? 1 : 0;
    const int ngrp = (p.BN + 31) / 32;
    const int cg0 = p.epi2 ? (grp ? (ngrp + 1) / 2 : 0) : 0;
    const int cg1 = p.epi2 ? (grp ? ngrp : (ngrp + 1) / 2) : ngrp;
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      int m0, kc0, kc1, split;
      tile_chunks(tile, m0, kc0, kc1, split);
      const int acc0 = p.mh == 2 ? 0 : it & 1;
      mbar_wait(&tfull[acc0], p.mh == 2 ? (it & 1) : ((it >> 1) & 1));
      tc_fence_after();
      for (int h = 0; h < p.mh; ++h) {
      const int acc = acc0 + h;  // TMEM buffer: tile parity, or the tile's half
      const int row0 = m0 + 128 * h + 32 * q;  // this warp's 32 rows (TMEM lanes 32q..)
      float* out_base = p.out + (kMN ? int64_t(split) * p.M * p.N : 0);
      // explicit shared-space accesses (the uintptr-aligned base would otherwise
      // compile to generic LD/ST)
      const uint32_t st_s = smem_u32(stage_out + (4 * grp + q) * (32 * 36));
      // 32-column groups: TMEM -> registers (thread = row) -> ReLU / mask -> smem
      // -> registers (8 lanes = one 128-byte row segment) -> coalesced stores
      for (int c0 = 32 * cg0; c0 < 32 * cg1; c0 += 32) {
        const int cc = c0 + 4 * (lane & 7);
        // ReLU-backward mask of this lane's 8 output segments, loaded up front
        float4 mk[8];
        uint32_t mb[8];  // bits_in: this lane's 4 columns of each of its 8 rows
        if (p.bits_in) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int row = row0 + 4 * j + (lane >> 3);
            mb[j] = row < p.M ? (__ldg(p.bits_in + int64_t(row) * p.ldbi + (c0 >> 5)) >>
                                 (4 * (lane & 7))) : 0xfu;
          }
        }
        if (p.mask) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int row = row0 + 4 * j + (lane >> 3);
            mk[j] = make_float4(1.f, 1.f, 1.f, 1.f);
            if (row < p.M && cc + 4 <= p.N && (p.ldm & 3) == 0)
              mk[j] = __ldg(reinterpret_cast<const float4*>(p.mask + int64_t(row) * p.ldm + cc));
            else if (row < p.M && cc < p.N) {
              const float* mrow = p.mask + int64_t(row) * p.ldm + cc;
              mk[j].x = mrow[0];
              if (cc + 1 < p.N) mk[j].y = mrow[1];
              if (cc + 2 < p.N) mk[j].z = mrow[2];
              if (cc + 3 < p.N) mk[j].w = mrow[3];
            }
          }
        }
        uint32_t r[2][16];
        tmem_ld16_nowait(tmem_base + uint32_t(acc * p.tmem_cols + c0) + (uint32_t(32 * q) << 16),
                         r[0]);
        if (c0 + 16 < p.BN)
          tmem_ld16_nowait(tmem_base + uint32_t(acc * p.tmem_cols + c0 + 16) +
                               (uint32_t(32 * q) << 16),
                           r[1]);
        tmem_wait_ld();
        uint32_t bw = 0;  // bits_out: 1[v > 0] of this thread's row, columns c0 .. c0 + 31
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int i = 0; i < 16; i += 4) {
            float4 v = make_float4(__uint_as_float(r[h][i]), __uint_as_float(r[h][i + 1]),
                                   __uint_as_float(r[h][i + 2]), __uint_as_float(r[h][i + 3]));
            if (p.relu) {
              v.x = v.x > 0.f ? v.x : 0.f;
              v.y = v.y > 0.f ? v.y : 0.f;
              v.z = v.z > 0.f ? v.z : 0.f;
              v.w = v.w > 0.f ? v.w : 0.f;
            }
            bw |= (v.x > 0.f ? 1u : 0u) << (16 * h + i) | (v.y > 0.f ? 2u : 0u) << (16 * h + i) |
                  (v.z > 0.f ? 4u : 0u) << (16 * h + i) | (v.w > 0.f ? 8u : 0u) << (16 * h + i);
            st_shared4(st_s + 4u * uint32_t(lane * 36 + 16 * h + i), v);
          }
        if (p.bits_out && row0 + lane < p.M && !(p.dbg & 2))
          p.bits_out[int64_t(row0 + lane) * p.ldbo + (c0 >> 5)] = bw;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int rr = 4 * j + (lane >> 3);
          const int row = row0 + rr;
          if (row >= p.M || cc >= p.N) continue;
          float4 v = ld_shared4(st_s + 4u * uint32_t(rr * 36 + 4 * (lane & 7)));
          if (p.mask) {
            v.x = mk[j].x > 0.f ? v.x : 0.f;
            v.y = mk[j].y > 0.f ? v.y : 0.f;
            v.z = mk[j].z > 0.f ? v.z : 0.f;
            v.w = mk[j].w > 0.f ? v.w : 0.f;
          }
          if (p.bits_in) {
            v.x = (mb[j] & 1u) ? v.x : 0.f;
            v.y = (mb[j] & 2u) ? v.y : 0.f;
            v.z = (mb[j] & 4u) ? v.z : 0.f;
            v.w = (mb[j] & 8u) ? v.w : 0.f;
          }
          if (p.dbg & 2) continue;
          float* o = out_base + int64_t(row) * p.ldo + cc;
          if (cc + 4 <= p.N && (p.ldo & 3) == 0) {
            *reinterpret_cast<float4*>(o) = v;
          } else {
            o[0] = v.x;
            if (cc + 1 < p.N) o[1] = v.y;
            if (cc + 2 < p.N) o[2] = v.z;
            if (cc + 3 < p.N) o[3] = v.w;
          }
        }
        __syncwarp();
      }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc0]);
    }
  } else if ((warp >= 8 && warp < 12) || (warp >= 12 && p.conv2)) {
    // ---------------- converters (warps 8-11, with conv2 also 12-15)
    const int t = threadIdx.x - 256;  // 0..127, or 0..255 with conv2
    const int nthr = p.conv2 ? 256 : 128;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      int m0, kc0, kc1, split;
      tile_chunks(tile, m0, kc0, kc1, split);
      for (int kc = kc0; kc < kc1; ++kc) {
        mbar_wait(&full[s], ph);
        uint8_t* st = smem + s * stage_bytes;
        if (!(p.dbg & 4))
          split_tile(smem_u32(st), smem_u32(st + a_bytes), a_bytes / 16, t, nthr);
        if (kMN)
          split_tile(smem_u32(st + 2 * a_bytes), smem_u32(st + 2 * a_bytes + b_bytes),
                     b_bytes / 16, t, nthr);
        fence_proxy_async();
        __syncwarp();
        if ((t & 31) == 0) mbar_arrive(&conv[s]);
        if (++s == kStages) s = 0, ph ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (p.cs > 1) cluster_sync();  // no peer still multicasting into / arriving on this CTA
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(2 * p.tmem_cols));
  }
}

// B(n, k) for the K-major paths, padded to Kp columns and split into hi / lo:
//   transpose == 1: B(n, k) = W[k][n]  (forward: W is K x N)
//   transpose == 0: B(n, k) = W[n][k]  (input gradient: W is N x K)
__global__ void k_prep_b(const float* __restrict__ W, int wcols, int N, int K, int Kp, int transpose,
                         float* __restrict__ bhi, float* __restrict__ blo) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(N) * Kp) return;
  const int n = int(i / Kp), k = int(i % Kp);
  float x = 0.f;
  if (k < K) x = transpose ? W[int64_t(k) * wcols + n] : W[int64_t(n) * wcols + k];
  const float h = tf32_hi(x);
  bhi[i] = h;
  blo[i] = x - h;
}

}  // namespace tc

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  QGNN_REQUIRE(fn, QGNN_ECUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D fp32 tensor map: inner (contiguous) extent x outer extent, row pitch in elements
CUtensorMap make_map(const float* base, uint64_t inner, uint64_t outer, uint64_t pitch_elems,
                     uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * 4};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  QGNN_REQUIRE((pitch_elems * 4) % 16 == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0,
               QGNN_EINVAL, "tensor map: 16-byte aligned base/pitch required");
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  QGNN_REQUIRE(r == CUDA_SUCCESS, QGNN_ECUDA, "cuTensorMapEncodeTiled failed");
  return m;
}

// 256-row tiles for the K-major path: the B stage is then loaded once per 256
// output rows.  Default: only for narrow outputs (BN <= 64, e.g. the 47-class
// layer: -12 % in profiles/gemm_micro_r1.txt); at BN = 256 the halved ring depth
// and the lost TMEM double buffer cost more (+20 %).  QGNN_GEMM_M256=0/1 forces.
bool gemm_m256(int bn) {
  const char* e = std::getenv("QGNN_GEMM_M256");
  if (e) return std::atoi(e) != 0;
  return bn <= 64;
}

int gemm_debug() {
  const char* e = std::getenv("QGNN_GEMM_DEBUG");
  return e ? std::atoi(e) : 0;
}

int gemm_bk() {  // QGNN_GEMM_BK=32: 128-byte K-major rows (SW128) for z = A W / dz W^T
  const char* e = std::getenv("QGNN_GEMM_BK");
  return e && std::atoi(e) == 32 ? 32 : 16;
}

bool gemm_conv2() {  // QGNN_GEMM_CONV2=0: four converter warps for the weight gradient too
  const char* e = std::getenv("QGNN_GEMM_CONV2");
  return !e || std::atoi(e) != 0;
}

bool gemm_epi2() {  // QGNN_GEMM_EPI2=0: one epilogue warp group for every shape
  const char* e = std::getenv("QGNN_GEMM_EPI2");
  return !e || std::atoi(e) != 0;
}

int gemm_cluster() {  // QGNN_GEMM_CLUSTER: CTAs sharing each B stage (1, 2, 4 or 8)
  const char* e = std::getenv("QGNN_GEMM_CLUSTER");
  const int v = e ? std::atoi(e) : 2;
  return v == 8 ? 8 : v == 4 ? 4 : v == 2 ? 2 : 1;
}

bool wgrad_m256() {  // QGNN_WGRAD_M256=0: 128-row tiles (A/B)
  const char* e = std::getenv("QGNN_WGRAD_M256");
  return !e || std::atoi(e) != 0;
}

int pow2_cols(int bn) {
  int c = 32;
  while (c < bn) c <<= 1;
  return c;
}

constexpr size_t kSmemBudget = 200 * 1024;  // + 18 KB epilogue staging (<= 227 KB)
constexpr size_t kStaging = 4 * 32 * 36 * sizeof(float);  // one epilogue group's blocks
// the second epilogue group's staging comes out of the ring's budget
int stages_for(int BN, int mh = 1, int bk = tc::kBK, int epi2 = 0) {
  const size_t stage = 2 * tc::kBM * bk * 4 * size_t(mh) + 2 * size_t(BN) * bk * 4;
  const size_t budget = kSmemBudget - (epi2 ? kStaging : 0);
  return int(std::max<size_t>(2, std::min<size_t>(tc::kMaxStages, budget / stage)));
}
size_t smem_bytes(int BN, int mh = 1, int bk = tc::kBK, int epi2 = 0) {
  const size_t stage = 2 * tc::kBM * bk * 4 * size_t(mh) + 2 * size_t(BN) * bk * 4;
  return size_t(stages_for(BN, mh, bk, epi2)) * stage + 1024 + 256 + (epi2 ? 2 : 1) * kStaging;
}

template <bool kMN>
void launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& blo, const tc::Params& p,
            int num_sms, cudaStream_t s) {
  const size_t sm = smem_bytes(p.BN, p.mh, kMN ? tc::kBK : p.bk, p.epi2);
  static bool attr_set = false;
  if (!attr_set) {
    QGNN_CUDA(cudaFuncSetAttribute(tc::k_tc_gemm<kMN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(kSmemBudget + 1024 + 256 + 4 * 32 * 36 * sizeof(float))));
    attr_set = true;
  }
  const int tiles = p.m_tiles * p.splits;
  if (p.cs == 1) {
    const int grid = std::max(1, std::min(tiles, num_sms));
    tc::k_tc_gemm<kMN><<<grid, tc::kThreads, sm, s>>>(a, b, blo, p);
  } else {
    // every CTA of a cluster runs the same number of tiles (p.m_tiles is a multiple
    // of cs; rows past M load as TMA zero fill and are not stored)
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(tc::kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(p.cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // persistent grid = the clusters that are co-resident (GPC sizes need not be
    // multiples of cs, so this can be below num_sms / cs)
    static int resident[2][9] = {};  // [kMN][cs], per process (one device per engine)
    int& rc = resident[kMN ? 1 : 0][p.cs];
    if (rc == 0) {
      cfg.gridDim = dim3(unsigned(num_sms / p.cs * p.cs));
      int n = 0;
      QGNN_CUDA(cudaOccupancyMaxActiveClusters(&n, tc::k_tc_gemm<kMN>, &cfg));
      rc = std::max(1, n);
    }
    const int grid = std::max(p.cs, std::min(tiles, rc * p.cs));
    cfg.gridDim = dim3(unsigned(grid));
    QGNN_CUDA(cudaLaunchKernelEx(&cfg, tc::k_tc_gemm<kMN>, a, b, blo, p));
  }
  check_launch("k_tc_gemm");
}
}  // namespace

// C[rows x N] = A[rows x K] B  with B(n,k) from W (see k_prep_b); relu optional.
namespace {
void tc_gemm_block(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int wcols, int N,
                   int K, int transpose_w, int64_t n_rows, int relu, float* out, int64_t ldo,
                   cudaStream_t s, const float* mask, int64_t ldm, uint32_t* bits_out,
                   int64_t ldbo, const uint32_t* bits_in, int64_t ldbi);
}  // namespace

// Outputs wider than one TMEM tile (N > 256) run as 256-column blocks of B.
void tc_gemm_rows(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int wcols, int N,
                  int K, int transpose_w, int64_t n_rows, int relu, float* out, int64_t ldo,
                  cudaStream_t s, const float* mask, int64_t ldm, uint32_t* bits_out,
                  int64_t ldbo, const uint32_t* bits_in, int64_t ldbi) {
  QGNN_REQUIRE(K <= 4096, QGNN_EINVAL, "tc_gemm: K must be <= 4096");
  int launches = 0;
  for (int n0 = 0; n0 < N; n0 += 256) {
    const int nb = std::min(256, N - n0);
    // B(n, k) = W[k][n] (transpose_w) or W[n][k]: block n0 starts n0 columns / rows in
    const float* Wb = transpose_w ? W + n0 : W + int64_t(n0) * wcols;
    tc_gemm_block(ctx, A, lda, Wb, wcols, nb, K, transpose_w, n_rows, relu, out + n0, ldo, s,
                  mask ? mask + n0 : nullptr, ldm, bits_out ? bits_out + n0 / 32 : nullptr, ldbo,
                  bits_in ? bits_in + n0 / 32 : nullptr, ldbi);
    launches += ctx->last_gemm_launches;
  }
  ctx->last_gemm_launches = launches;
}

namespace {
void tc_gemm_block(qgnn_ctx* ctx, const float* A, int64_t lda, const float* W, int wcols, int N,
                   int K, int transpose_w, int64_t n_rows, int relu, float* out, int64_t ldo,
                   cudaStream_t s, const float* mask, int64_t ldm, uint32_t* bits_out,
                   int64_t ldbo, const uint32_t* bits_in, int64_t ldbi) {
  QGNN_REQUIRE(N <= 256 && K <= 4096, QGNN_EINVAL, "tc_gemm: N must be <= 256");
  const int BN = int(round_up(N, 16));
  const int Kp = int(round_up(K, 4));
  float* bhi = static_cast<float*>(ctx_gemm_b(ctx, size_t(2) * BN * Kp * sizeof(float)));
  float* blo = bhi + size_t(BN) * Kp;
  auto& bp = ctx->bprep;
  const bool reuse = ctx->b_reuse && bp.W == W && bp.buf == bhi && bp.wcols == wcols &&
                     bp.N == N && bp.K == K && bp.transpose == transpose_w && bp.gen == ctx->wgen;
  ctx->last_gemm_launches = reuse ? 1 : 2;
  if (!reuse) {  // same stream as every GEMM that reuses it: ordered before them
    tc::k_prep_b<<<unsigned(ceil_div(int64_t(N) * Kp, 256)), 256, 0, s>>>(W, wcols, N, K, Kp,
                                                                          transpose_w, bhi, blo);
    bp.W = W, bp.buf = bhi, bp.wcols = wcols, bp.N = N, bp.K = K, bp.transpose = transpose_w;
    bp.gen = ctx->wgen;
  }
  const int bk = gemm_bk();
  const CUtensorMapSwizzle swz = bk == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const CUtensorMap ta = make_map(A, uint64_t(K), uint64_t(n_rows), uint64_t(lda), uint32_t(bk),
                                  tc::kBM, swz);
  const bool m256 = gemm_m256(BN) && n_rows > tc::kBM;
  int cs = (gemm_debug() & 8) || m256 ? 1 : gemm_cluster();  // producer-only isolation is per CTA
  while (cs > 1 && (BN % (8 * cs) != 0 || ceil_div(n_rows, tc::kBM) < 2 * cs)) cs >>= 1;
  const CUtensorMap tb = make_map(bhi, uint64_t(Kp), uint64_t(N), uint64_t(Kp), uint32_t(bk),
                                  uint32_t(BN / cs), swz);
  const CUtensorMap tbl = make_map(blo, uint64_t(Kp), uint64_t(N), uint64_t(Kp), uint32_t(bk),
                                   uint32_t(BN / cs), swz);
  tc::Params p{};
  p.M = int(n_rows);
  p.N = N;
  p.K = K;
  p.BN = BN;
  p.tmem_cols = pow2_cols(BN);
  p.m_tiles = int(ceil_div(n_rows, tc::kBM));
  p.splits = 1;
  p.k_chunks = int(ceil_div(K, bk));
  p.bk = bk;
  p.chunks_per_split = p.k_chunks;
  p.out = out;
  p.ldo = ldo;
  p.relu = relu;
  p.mask = mask;
  p.ldm = ldm;
  p.bits_out = relu ? bits_out : nullptr;
  p.ldbo = ldbo;
  p.bits_in = bits_in;
  p.ldbi = ldbi;
  p.mh = m256 ? 2 : 1;
  p.m_tiles = int(ceil_div(n_rows, tc::kBM * p.mh));
  p.cs = cs;
  p.dbg = gemm_debug();
  if (cs > 1) p.m_tiles = int(round_up(p.m_tiles, cs));
  p.epi2 = gemm_epi2() && p.k_chunks <= 8 && BN >= 128 && !(p.dbg & 8) ? 1 : 0;
  p.conv2 = 0;  // K-major rings are not conversion-paced (profiles/ab_gemm_conv2_r2.txt)
  p.stages = stages_for(BN, p.mh, bk, p.epi2);
  launch<false>(ta, tb, tbl, p, ctx->num_sms, s);
}

}  // namespace

// Partial tiles of out[M x N] = A[rows x M]^T B[rows x N], split-K over rows:
// returns the workspace holding *splits consecutive M x N partial products
// (the caller reduces them in fixed order).
float* tc_gemm_wgrad_partials(qgnn_ctx* ctx, const float* A, int64_t lda, const float* B,
                              int64_t ldb, int M, int N, int64_t n_rows, int* splits_out,
                              cudaStream_t s) {
  QGNN_REQUIRE(N <= 256, QGNN_EINVAL, "tc_gemm_wgrad: N must be <= 256");
  const int BN = int(round_up(N, 32));
  // 256-row tiles when M > 128 (the N operand streams once per 256 output rows)
  const int mh = M > tc::kBM && wgrad_m256() ? 2 : 1;
  const int m_tiles = int(ceil_div(M, tc::kBM * mh));
  const int k_chunks = int(ceil_div(std::max<int64_t>(n_rows, 1), tc::kBK));
  int splits = std::max(1, std::min(k_chunks, ctx->num_sms / std::max(1, m_tiles)));
  const int cps = int(ceil_div(k_chunks, splits));
  splits = int(ceil_div(k_chunks, cps));
  float* part = static_cast<float*>(ctx_scratch(ctx, sizeof(float) * size_t(splits) * M * N));
  const CUtensorMap ta = make_map(A, uint64_t(M), uint64_t(n_rows), uint64_t(lda), 32, tc::kBK,
                                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  const CUtensorMap tb = make_map(B, uint64_t(N), uint64_t(n_rows), uint64_t(ldb), 32, tc::kBK,
                                  CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
  tc::Params p{};
  p.M = M;
  p.N = N;
  p.K = int(n_rows);
  p.BN = BN;
  p.tmem_cols = pow2_cols(BN);
  p.m_tiles = m_tiles;
  p.splits = splits;
  p.k_chunks = k_chunks;
  p.chunks_per_split = cps;
  p.out = part;
  p.ldo = N;
  p.relu = 0;
  p.mask = nullptr;
  p.ldm = 0;
  p.mh = mh;
  p.cs = 1;
  p.bk = tc::kBK;
  p.dbg = gemm_debug();
  p.conv2 = gemm_conv2() ? 1 : 0;
  p.stages = stages_for(BN, mh);
  launch<true>(ta, tb, tb, p, ctx->num_sms, s);
  *splits_out = splits;
  return part;
}

}  // namespace qgnn_b200
