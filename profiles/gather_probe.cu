// gather_probe.cu — measures the random-row gather ceiling of one B200 (the
// floor under K4 SpMM on a power-law graph without locality).  Each "edge"
// gathers one W-byte row of a table of S bytes at a uniformly random index;
// G = W/16 lanes cooperate on a row (16-byte loads), a warp covers 32/G rows
// per load step and UNR steps are kept in flight.  Prints gathered GB/s.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_probe.cu -o gather_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

template <int G, int UNR>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ tab, int ld4,
                                                const int* __restrict__ idx, long m,
                                                float* __restrict__ sink) {
  const int lane = threadIdx.x & 31, sub = lane % G, grp = lane / G;
  constexpr int RPW = 32 / G;  // rows per warp step
  const long warp = (long(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const long nw = (long(gridDim.x) * blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long e0 = warp * RPW * UNR; e0 < m; e0 += nw * RPW * UNR) {
    int c[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const long e = e0 + u * RPW + grp;
      c[u] = e < m ? __ldg(idx + e) : -1;
    }
    float4 v[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u)
      v[u] = c[u] >= 0 ? __ldg(tab + long(c[u]) * ld4 + sub) : make_float4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      acc.x += v[u].x;
      acc.y += v[u].y;
      acc.z += v[u].z;
      acc.w += v[u].w;
    }
  }
  const float s = acc.x + acc.y + acc.z + acc.w;
  if (s == 123.456f) sink[0] = s;
}

template <int G, int UNR>
float run(const float4* tab, int ld4, const int* idx, long m, float* sink, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 2; ++i) k_gather<G, UNR><<<blocks, 256>>>(tab, ld4, idx, m, sink);
  cudaEventRecord(a);
  const int reps = 5;
  for (int i = 0; i < reps; ++i) k_gather<G, UNR><<<blocks, 256>>>(tab, ld4, idx, m, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long m = 64l << 20;  // gathers
  int* idx;
  cudaMalloc(&idx, m * 4);
  float* sink;
  cudaMalloc(&sink, 4);
  const size_t maxbytes = size_t(3) << 30;
  float4* tab;
  cudaMalloc(&tab, maxbytes);
  cudaMemset(tab, 0, maxbytes);
  std::vector<int> h(m);
  for (long sz_mb : {16l, 48l, 96l, 192l, 2048l}) {
    for (int w : {64, 128, 256, 512, 1024}) {
      const long rows = (sz_mb << 20) / w;
      srand(1);
      for (long i = 0; i < m; ++i) h[i] = int(((long(rand()) << 16) ^ rand()) % rows);
      cudaMemcpy(idx, h.data(), m * 4, cudaMemcpyHostToDevice);
      const int ld4 = w / 16;
      float best = 1e30f;
      int bestb = 0;
      for (int bpsm : {4, 8}) {
        const int blocks = sms * bpsm;
        float t;
        switch (w) {
          case 64: t = run<4, 8>(tab, ld4, idx, m, sink, blocks); break;
          case 128: t = run<8, 8>(tab, ld4, idx, m, sink, blocks); break;
          case 256: t = run<16, 8>(tab, ld4, idx, m, sink, blocks); break;
          case 512: t = run<32, 8>(tab, ld4, idx, m, sink, blocks); break;
          default: {  // 1024 B: two 512-byte halves per row, as two gathers
            t = run<32, 8>(tab, ld4, idx, m, sink, blocks);
          }
        }
        if (t < best) best = t, bestb = bpsm;
      }
      const double bytes = double(m) * (w == 1024 ? 512 : w);
      printf("table %5ld MB  row %4d B  %.3f ms  %8.1f GB/s gathered  (%d CTA/SM)\n", sz_mb, w,
             best, bytes / best / 1e6, bestb);
      fflush(stdout);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
