// dbuf.cuh — owning device buffer shared by the engine and the GPU setup.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace qgnn_b200 {

// ---------------------------------------------------------- device buffer ---
template <typename X>
struct DBuf {
  X* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    return *this;
  }
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void alloc(size_t count, bool zero = true) {
    if (count <= n && p) {
      if (zero) QGNN_CUDA(cudaMemset(p, 0, count * sizeof(X)));
      QGNN_CUDA(cudaDeviceSynchronize());
      return;
    }
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    QGNN_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(X)));
    if (zero) QGNN_CUDA(cudaMemset(p, 0, std::max<size_t>(1, count) * sizeof(X)));
    // legacy-stream memsets/copies do not order against our non-blocking streams
    QGNN_CUDA(cudaDeviceSynchronize());
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void upload(const std::vector<X>& v) {
    alloc(v.size(), false);
    if (!v.empty()) QGNN_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(X), cudaMemcpyHostToDevice));
    QGNN_CUDA(cudaDeviceSynchronize());
  }
};

}  // namespace qgnn_b200
