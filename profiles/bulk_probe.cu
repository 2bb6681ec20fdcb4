// bulk_probe.cu — random-row gathers of W-byte rows from an L2-resident table
// into shared memory, three ways, to pick the SpMM gather mechanism on B200:
//   ldg   : register loads (16 B/lane), UNR in flight
//   lgsts : cp.async 16 B/lane into a per-warp smem ring
//   bulk  : cp.async.bulk (TMA bulk copy) of one whole W-byte row per lane,
//           32 rows per warp step, mbarrier completion, DEPTH steps in flight
// Prints gathered GB/s.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int W, int DEPTH>
__global__ void __launch_bounds__(128) k_bulk(const char* __restrict__ tab, const int* __restrict__ idx,
                                              long m, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* ring = sm + warp * (DEPTH * 32 * W + DEPTH * 8);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + DEPTH * 32 * W);
  if (lane < DEPTH)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bars + lane)));
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long gw = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (long(gridDim.x) * blockDim.x) >> 5;
  float acc = 0.f;
  int slot = 0, filled = 0;
  uint32_t phase = 0;  // bit s = parity of slot s
  auto consume = [&](int s) {
    const uint32_t par = (phase >> s) & 1u;
    asm volatile(
        "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(
            su32(bars + s)),
        "r"(par)
        : "memory");
    phase ^= 1u << s;
    const float4* d = reinterpret_cast<const float4*>(ring + s * 32 * W);
#pragma unroll
    for (int k = 0; k < W / 16; ++k) {
      const float4 v = d[k * 32 + lane];
      acc += v.x + v.y + v.z + v.w;
    }
  };
  int cn = gw * 32 < m ? idx[gw * 32 + lane] : 0;
  for (long e0 = gw * 32; e0 < m; e0 += nw * 32) {
    const int c = cn;
    if (e0 + nw * 32 < m) cn = idx[e0 + nw * 32 + lane];
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bars + slot)),
                   "r"(32 * W)
                   : "memory");
    __syncwarp();
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(ring + slot * 32 * W + lane * W)),
        "l"(tab + long(c) * W), "n"(W), "r"(su32(bars + slot))
        : "memory");
    if (++slot == DEPTH) slot = 0;
    if (filled < DEPTH - 1) ++filled;
    else { consume(slot); __syncwarp(); }
  }
  int s = slot - filled; if (s < 0) s += DEPTH;
  for (int k = 0; k < filled; ++k) { consume(s); if (++s == DEPTH) s = 0; }
  if (acc == 123.456f) sink[0] = acc;
}

template <int W, int DEPTH>
__global__ void __launch_bounds__(256) k_lgsts(const char* __restrict__ tab, const int* __restrict__ idx,
                                               long m, float* sink) {
  // G = W/16 lanes per row, 32/G rows per step
  constexpr int G = W / 16, E = 32 / G;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float4* ring = reinterpret_cast<float4*>(sm) + warp * DEPTH * 32;
  const long gw = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (long(gridDim.x) * blockDim.x) >> 5;
  float acc = 0.f;
  int slot = 0, filled = 0;
  int cn = gw * E < m ? idx[gw * E + lane / G] : 0;
  for (long e0 = gw * E; e0 < m; e0 += nw * E) {
    const int c = cn;
    if (e0 + nw * E < m) cn = idx[e0 + nw * E + lane / G];
    const uint32_t d = su32(ring + slot * 32 + lane);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(tab + long(c) * W + (lane % G) * 16) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    if (++slot == DEPTH) slot = 0;
    if (filled < DEPTH - 1) ++filled;
    else {
      asm volatile("cp.async.wait_group %0;" ::"n"(DEPTH - 1) : "memory");
      const float4 v = ring[slot * 32 + lane];
      acc += v.x + v.y + v.z + v.w;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (acc == 123.456f) sink[0] = acc;
}

template <typename K>
float timeit(K k, int blocks, int threads, size_t smem, const char* tab, const int* idx, long m, float* sink) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<<<blocks, threads, smem>>>(tab, idx, m, sink);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k<<<blocks, threads, smem>>>(tab, idx, m, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1e9; }
  return ms / 5;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long m = 64l << 20;
  int* idx; cudaMalloc(&idx, m * 4);
  float* sink; cudaMalloc(&sink, 4);
  char* tab; cudaMalloc(&tab, size_t(1) << 30); cudaMemset(tab, 0, size_t(1) << 30);
  std::vector<int> h(m);
  for (long mb : {40l, 1024l}) {
    const long rows = (mb << 20) / 128;
    srand(1);
    for (long i = 0; i < m; ++i) h[i] = int(((long(rand()) << 16) ^ rand()) % rows);
    cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
    const double bytes = double(m) * 128;
    for (int wpb : {4}) {
      float t;
      t = timeit(k_bulk<128, 4>, sms * 4, 128, 4 * (4 * 32 * 128 + 32), tab, idx, m, sink);
      printf("table %5ld MB bulk  W=128 D=4 4w/cta x4: %8.1f GB/s\n", mb, bytes / t / 1e6);
      t = timeit(k_bulk<128, 6>, sms * 3, 128, 4 * (6 * 32 * 128 + 48), tab, idx, m, sink);
      printf("table %5ld MB bulk  W=128 D=6 4w/cta x3: %8.1f GB/s\n", mb, bytes / t / 1e6);
      t = timeit(k_bulk<128, 2>, sms * 8, 128, 4 * (2 * 32 * 128 + 16), tab, idx, m, sink);
      printf("table %5ld MB bulk  W=128 D=2 4w/cta x8: %8.1f GB/s\n", mb, bytes / t / 1e6);
      t = timeit(k_lgsts<128, 8>, sms * 6, 256, 8 * 8 * 32 * 16, tab, idx, m, sink);
      printf("table %5ld MB lgsts W=128 D=8: %8.1f GB/s\n", mb, bytes / t / 1e6);
      t = timeit(k_lgsts<128, 16>, sms * 4, 256, 8 * 16 * 32 * 16, tab, idx, m, sink);
      printf("table %5ld MB lgsts W=128 D=16: %8.1f GB/s\n", mb, bytes / t / 1e6);
    }
    fflush(stdout);
  }
  return 0;
}
