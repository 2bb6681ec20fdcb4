// setup.cu — GPU-side graph setup.  See setup.cuh.
//
// What runs where: every per-edge pass (consumer sets, the local/remote split
// of each row's adjacency with its coefficients, the transpose of the remote
// CSR, the distinct-source counts, the receivers' Σα² per message) runs on the
// device over a resident copy of the CSR; the host keeps the O(n) list work
// (ascending id lists, row maps, slot lists) and receives only pointer arrays
// and lists.  Summation and list orders are the reference's, so the outputs
// are identical to host_graph.cpp's builders (tests/test_gpu_setup.py).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <cstring>

#include "setup.cuh"

namespace qgnn_b200 {

namespace {

constexpr int kThreads = 256;  // 8 warps per block, a warp per node / row

inline unsigned grid_for_warps(int64_t warps) {
  return unsigned(std::min<int64_t>(std::max<int64_t>(1, ceil_div(warps * 32, kThreads)), 148 * 64));
}
inline unsigned grid_for(int64_t n) {
  return unsigned(std::min<int64_t>(std::max<int64_t>(1, ceil_div(n, kThreads)), 148 * 64));
}
__device__ __forceinline__ int64_t gwarp() {
  return (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
}
__device__ __forceinline__ int64_t nwarps() { return (int64_t(gridDim.x) * blockDim.x) >> 5; }
__device__ __forceinline__ int64_t gthread() { return int64_t(blockIdx.x) * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t nthreads() { return int64_t(gridDim.x) * blockDim.x; }

// coeffs.hpp:30-45, evaluated for the edge (row v, neighbour u): GCN
// 1/sqrt((d_u+1)(d_v+1)), SAGE-mean 1/(d_v+1).  Each operation correctly
// rounded, no contraction: bit-identical to the host's -ffp-contract=off build.
__device__ __forceinline__ double coeff(double du1, double dv1, bool sage) {
  return sage ? __ddiv_rn(1.0, dv1) : __ddiv_rn(1.0, __dsqrt_rn(__dmul_rn(du1, dv1)));
}
__device__ __forceinline__ double deg1(const int64_t* ptr, int64_t v) {
  return double(ptr[v + 1] - ptr[v]) + 1.0;
}

// partition.hpp:57-71: the consumers of v are the distinct owners of its
// neighbours other than owner[v].  Count pass (cons == nullptr) writes
// cnt[v + 1]; fill pass lists them ascending at cons[cptr[v]].
__global__ void k_consumers(const int64_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                            const uint32_t* __restrict__ owner, int64_t n, int W,
                            int64_t* __restrict__ cnt, const int64_t* __restrict__ cptr,
                            uint32_t* __restrict__ cons) {
  extern __shared__ uint32_t sm[];
  const int lane = threadIdx.x & 31;
  uint32_t* bm = sm + (threadIdx.x >> 5) * W;
  for (int64_t v = gwarp(); v < n; v += nwarps()) {
    for (int w = lane; w < W; w += 32) bm[w] = 0;
    __syncwarp();
    const uint32_t ov = owner[v];
    for (int64_t e = ptr[v] + lane; e < ptr[v + 1]; e += 32) {
      const uint32_t q = owner[adj[e]];
      if (q != ov) atomicOr(&bm[q >> 5], 1u << (q & 31));
    }
    __syncwarp();
    if (!cons) {
      int c = 0;
      for (int w = lane; w < W; w += 32) c += __popc(bm[w]);
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0) cnt[v + 1] = c;
    } else if (lane == 0) {
      int64_t k = cptr[v];
      for (int w = 0; w < W; ++w)
        for (uint32_t x = bm[w]; x; x &= x - 1) cons[k++] = uint32_t(w) * 32 + uint32_t(__ffs(x) - 1);
    }
    __syncwarp();
  }
}

__global__ void k_scatter_index(const uint32_t* __restrict__ idx, int64_t n, int32_t* __restrict__ map) {
  for (int64_t i = gthread(); i < n; i += nthreads()) map[idx[i]] = int32_t(i);
}

// Per view row: number of same-partition (local) and cross-partition (remote)
// neighbours -> lptr[g + 1], rptr[g + 1] (scanned afterwards).
__global__ void k_view_count(const int64_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                             const uint32_t* __restrict__ owner, uint32_t me,
                             const uint32_t* __restrict__ row_node, int64_t n_rows,
                             int64_t* __restrict__ lptr, int64_t* __restrict__ rptr) {
  const int lane = threadIdx.x & 31;
  for (int64_t g = gwarp(); g < n_rows; g += nwarps()) {
    const int64_t v = row_node[g];
    int l = 0, r = 0;
    for (int64_t e = ptr[v] + lane; e < ptr[v + 1]; e += 32) (owner[adj[e]] == me ? l : r) += 1;
    l = __reduce_add_sync(0xffffffffu, l);
    r = __reduce_add_sync(0xffffffffu, r);
    if (lane == 0) lptr[g + 1] = l, rptr[g + 1] = r;
  }
}

// aggregate.hpp:58-85: each row's adjacency split into local and remote
// entries in adjacency order (ballot prefix per 32-edge chunk), with the
// forward / backward coefficients and, for the remote transpose, each remote
// entry's row.
template <typename T>
__global__ void k_view_fill(const int64_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                            const uint32_t* __restrict__ owner, uint32_t me,
                            const uint32_t* __restrict__ row_node, int64_t n_rows,
                            const int32_t* __restrict__ row_of, const int32_t* __restrict__ slot_of,
                            bool sage, const int64_t* __restrict__ lptr,
                            const int64_t* __restrict__ rptr, T* __restrict__ self_alpha,
                            int32_t* __restrict__ lcol, T* __restrict__ lafwd,
                            T* __restrict__ labwd, int32_t* __restrict__ rslot,
                            T* __restrict__ ralpha, int32_t* __restrict__ erow) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  for (int64_t g = gwarp(); g < n_rows; g += nwarps()) {
    const int64_t v = row_node[g];
    const int64_t e0 = ptr[v], e1 = ptr[v + 1];
    const double dv1 = double(e1 - e0) + 1.0;
    if (lane == 0) self_alpha[g] = T(__ddiv_rn(1.0, dv1));
    int64_t lp = lptr[g], rp = rptr[g];
    for (int64_t base = e0; base < e1; base += 32) {
      const int64_t e = base + lane;
      const bool ok = e < e1;
      const int32_t u = ok ? adj[e] : 0;
      const uint32_t q = ok ? owner[u] : me;
      const bool isl = ok && q == me, isr = ok && q != me;
      const uint32_t bl = __ballot_sync(0xffffffffu, isl), br = __ballot_sync(0xffffffffu, isr);
      if (ok) {
        const double du1 = deg1(ptr, u);
        const double a = coeff(du1, dv1, sage);
        if (isl) {
          const int64_t i = lp + __popc(bl & lt);
          lcol[i] = row_of[u];
          lafwd[i] = T(a);
          labwd[i] = T(sage ? __ddiv_rn(1.0, du1) : a);  // coeffs.of(g, v, u)
        } else {
          const int64_t i = rp + __popc(br & lt);
          rslot[i] = slot_of[u];
          ralpha[i] = T(a);
          erow[i] = int32_t(g);
        }
      }
      lp += __popc(bl);
      rp += __popc(br);
    }
  }
}

__global__ void k_iota(int32_t* __restrict__ a, int64_t n) {
  for (int64_t i = gthread(); i < n; i += nthreads()) a[i] = int32_t(i);
}
__global__ void k_slot_hist(const int32_t* __restrict__ rslot, int64_t n, int64_t* __restrict__ sptr) {
  for (int64_t i = gthread(); i < n; i += nthreads())
    atomicAdd(reinterpret_cast<unsigned long long*>(sptr + rslot[i] + 1), 1ull);
}
// aggregate.hpp:156-163: slot -> contributing rows in ascending reference-row
// order.  Remote entries exist only on marginal rows, whose view order is
// ascending id (= reference order) in both row orders, so the stable sort by
// slot of the entries in CSR order is exactly that order.
template <typename T>
__global__ void k_transpose_gather(const int32_t* __restrict__ perm, int64_t n,
                                   const int32_t* __restrict__ erow, const T* __restrict__ ralpha,
                                   int32_t* __restrict__ srow, T* __restrict__ salpha) {
  for (int64_t i = gthread(); i < n; i += nthreads()) {
    const int32_t e = perm[i];
    srow[i] = erow[e];
    salpha[i] = ralpha[e];
  }
}

// Distinct source rows of a row range (self rows included; §8d operand bytes).
__global__ void k_mark_sources(const int64_t* __restrict__ lptr, const int32_t* __restrict__ lcol,
                               int64_t r0, int64_t r1, uint8_t* __restrict__ seen) {
  const int lane = threadIdx.x & 31;
  for (int64_t g = r0 + gwarp(); g < r1; g += nwarps()) {
    if (lane == 0) seen[g] = 1;
    for (int64_t e = lptr[g] + lane; e < lptr[g + 1]; e += 32) seen[lcol[e]] = 1;
  }
}
__global__ void k_count_set(const uint8_t* __restrict__ a, int64_t n, unsigned long long* out) {
  unsigned c = 0;
  for (int64_t i = gthread(); i < n; i += nthreads()) c += a[i] != 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, (unsigned long long)c);
}

// engine.hpp:262-273: Σ α² over the neighbours of message node u owned by the
// receiver q, in adjacency (ascending id) order; one thread per message.
__global__ void k_rx_asq(const int64_t* __restrict__ ptr, const int32_t* __restrict__ adj,
                         const uint32_t* __restrict__ owner, const uint32_t* __restrict__ ids,
                         const uint32_t* __restrict__ dst, int64_t m, bool sage,
                         double* __restrict__ out) {
  for (int64_t i = gthread(); i < m; i += nthreads()) {
    const int64_t u = ids[i];
    const uint32_t q = dst[i];
    const double du1 = deg1(ptr, u);
    double acc = 0.0;
    for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {
      const int32_t v = adj[e];
      if (owner[v] != q) continue;
      // alpha of the entry (row u, neighbour v), or self_alpha[v] for SAGE
      const double a = coeff(deg1(ptr, v), du1, false);
      const double w = sage ? __ddiv_rn(1.0, deg1(ptr, v)) : a;
      acc = __dadd_rn(acc, __dmul_rn(w, w));
    }
    out[i] = acc;
  }
}

// build_graph: both directions of every non-loop edge as (u << 32 | v) keys; loops
// become the all-ones key, sorted last and dropped
__global__ void k_edge_keys(const uint2* __restrict__ e, int64_t m, uint64_t* __restrict__ keys) {
  for (int64_t i = gthread(); i < m; i += nthreads()) {
    const uint2 uv = e[i];
    const bool loop = uv.x == uv.y;
    keys[2 * i] = loop ? ~0ull : (uint64_t(uv.x) << 32 | uv.y);
    keys[2 * i + 1] = loop ? ~0ull : (uint64_t(uv.y) << 32 | uv.x);
  }
}
__global__ void k_csr_from_keys(const uint64_t* __restrict__ keys, int64_t m,
                                int64_t* __restrict__ cnt, int32_t* __restrict__ adj) {
  for (int64_t i = gthread(); i < m; i += nthreads()) {
    const uint64_t k = keys[i];
    adj[i] = int32_t(uint32_t(k));
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (k >> 32) + 1), 1ull);
  }
}

// counts written at p[1..n] (p[0] = 0) -> inclusive scan in place
void scan_counts(int64_t* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  DBuf<int64_t> out;
  out.alloc(size_t(n), false);
  size_t bytes = 0;
  QGNN_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, p + 1, out.p, n, st));
  DBuf<uint8_t> tmp;
  tmp.alloc(std::max<size_t>(1, bytes), false);
  QGNN_CUDA(cub::DeviceScan::InclusiveSum(tmp.p, bytes, p + 1, out.p, n, st));
  QGNN_CUDA(cudaMemcpyAsync(p + 1, out.p, size_t(n) * sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
  QGNN_CUDA(cudaStreamSynchronize(st));
}

template <typename X>
std::vector<X> download(const X* p, int64_t n, cudaStream_t st) {
  std::vector<X> h(size_t(std::max<int64_t>(0, n)));
  if (n > 0) QGNN_CUDA(cudaMemcpyAsync(h.data(), p, size_t(n) * sizeof(X), cudaMemcpyDeviceToHost, st));
  QGNN_CUDA(cudaStreamSynchronize(st));
  return h;
}

}  // namespace

void build_graph_csr(int64_t n, const std::vector<std::pair<uint32_t, uint32_t>>& edges,
                     int device, std::vector<int64_t>& ptr, std::vector<int32_t>& adj) {
  const int64_t m = int64_t(edges.size());
  if (device < 0) {  // host: per-node sort + unique, like the reference
    std::vector<std::vector<int32_t>> lists(size_t(std::max<int64_t>(0, n)));
    for (const auto& e : edges) {
      if (e.first == e.second) continue;
      lists[e.first].push_back(int32_t(e.second));
      lists[e.second].push_back(int32_t(e.first));
    }
    ptr.assign(size_t(n + 1), 0);
    adj.clear();
    for (int64_t v = 0; v < n; ++v) {
      auto& l = lists[size_t(v)];
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
      ptr[size_t(v + 1)] = ptr[size_t(v)] + int64_t(l.size());
      adj.insert(adj.end(), l.begin(), l.end());
    }
    return;
  }
  QGNN_CUDA(cudaSetDevice(device));
  QGNN_REQUIRE(2 * m < (int64_t(1) << 31), QGNN_EINVAL, "dataset: more than 2^30 edges");
  cudaStream_t st = nullptr;
  QGNN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct Guard {
    cudaStream_t s;
    ~Guard() { cudaStreamDestroy(s); }
  } guard{st};
  DBuf<uint2> e;
  e.alloc(size_t(std::max<int64_t>(1, m)), false);
  if (m) QGNN_CUDA(cudaMemcpy(e.p, edges.data(), size_t(m) * sizeof(uint2), cudaMemcpyHostToDevice));
  DBuf<uint64_t> k0, k1;
  k0.alloc(size_t(std::max<int64_t>(1, 2 * m)), false);
  k1.alloc(size_t(std::max<int64_t>(1, 2 * m)), false);
  int64_t u = 0;
  if (m) {
    k_edge_keys<<<grid_for(m), kThreads, 0, st>>>(e.p, m, k0.p);
    check_launch("k_edge_keys");
    size_t bytes = 0;
    QGNN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k0.p, k1.p, int(2 * m), 0, 64, st));
    DBuf<uint8_t> tmp;
    tmp.alloc(std::max<size_t>(1, bytes), false);
    QGNN_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, k0.p, k1.p, int(2 * m), 0, 64, st));
    DBuf<int> nu;
    nu.alloc(1, true);
    size_t b2 = 0;
    QGNN_CUDA(cub::DeviceSelect::Unique(nullptr, b2, k1.p, k0.p, nu.p, int(2 * m), st));
    DBuf<uint8_t> tmp2;
    tmp2.alloc(std::max<size_t>(1, b2), false);
    QGNN_CUDA(cub::DeviceSelect::Unique(tmp2.p, b2, k1.p, k0.p, nu.p, int(2 * m), st));
    int nuh = 0;
    QGNN_CUDA(cudaMemcpyAsync(&nuh, nu.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    QGNN_CUDA(cudaStreamSynchronize(st));
    u = nuh;
    if (u > 0) {  // the loop sentinel sorts last
      uint64_t last = 0;
      QGNN_CUDA(cudaMemcpy(&last, k0.p + (u - 1), sizeof(uint64_t), cudaMemcpyDeviceToHost));
      if (last == ~0ull) --u;
    }
  }
  DBuf<int64_t> cnt;
  cnt.alloc(size_t(n + 1), true);
  DBuf<int32_t> a;
  a.alloc(size_t(std::max<int64_t>(1, u)), false);
  if (u) {
    k_csr_from_keys<<<grid_for(u), kThreads, 0, st>>>(k0.p, u, cnt.p, a.p);
    check_launch("k_csr_from_keys");
    scan_counts(cnt.p, n, st);
  }
  ptr = download(cnt.p, n + 1, st);
  adj = download(a.p, u, st);
}

GraphDev::GraphDev(const int64_t* ptr_h, const int32_t* adj_h, int64_t n_, const uint32_t* owner_h,
                   int64_t n_parts_, cudaStream_t s)
    : n(n_), nnz(ptr_h[n_]), n_parts(n_parts_), st(s) {
  QGNN_REQUIRE(n_parts >= 1, QGNN_EINVAL, "partitions: n_parts must be positive");
  for (int64_t v = 0; v < n; ++v)
    QGNN_REQUIRE(owner_h[v] < uint64_t(n_parts), QGNN_EINVAL, "owner id out of range");
  QGNN_REQUIRE(nnz < (int64_t(1) << 31), QGNN_EINVAL, "setup: more than 2^31 CSR entries");
  ptr.alloc(size_t(n + 1), false);
  adj.alloc(size_t(std::max<int64_t>(1, nnz)), false);
  owner.alloc(size_t(std::max<int64_t>(1, n)), false);
  row_of.alloc(size_t(std::max<int64_t>(1, n)), false);
  slot_of.alloc(size_t(std::max<int64_t>(1, n)), false);
  QGNN_CUDA(cudaMemcpy(ptr.p, ptr_h, size_t(n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  if (nnz) QGNN_CUDA(cudaMemcpy(adj.p, adj_h, size_t(nnz) * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (n) QGNN_CUDA(cudaMemcpy(owner.p, owner_h, size_t(n) * sizeof(uint32_t), cudaMemcpyHostToDevice));
}

std::vector<Part> partitions_from_owner_gpu(GraphDev& g, const uint32_t* owner) {
  const int64_t n = g.n, P = g.n_parts;
  const int W = int(ceil_div(P, 32));
  const size_t smem = size_t(kThreads / 32) * size_t(W) * sizeof(uint32_t);
  QGNN_REQUIRE(smem <= 48 * 1024, QGNN_EINVAL, "partitions: n_parts too large for the GPU setup");
  DBuf<int64_t> cptr;
  cptr.alloc(size_t(n + 1), true);
  if (n) {
    k_consumers<<<grid_for_warps(n), kThreads, smem, g.st>>>(g.ptr.p, g.adj.p, g.owner.p, n, W,
                                                             cptr.p, nullptr, nullptr);
    check_launch("k_consumers");
    scan_counts(cptr.p, n, g.st);
  }
  const std::vector<int64_t> cp = download(cptr.p, n + 1, g.st);
  DBuf<uint32_t> cons;
  cons.alloc(size_t(std::max<int64_t>(1, cp[n])), false);
  if (cp[n]) {
    k_consumers<<<grid_for_warps(n), kThreads, smem, g.st>>>(g.ptr.p, g.adj.p, g.owner.p, n, W,
                                                             nullptr, cptr.p, cons.p);
    check_launch("k_consumers");
  }
  const std::vector<uint32_t> cs = download(cons.p, cp[n], g.st);
  // partition.hpp:39-84 list assembly: ascending node ids throughout
  std::vector<Part> parts(static_cast<size_t>(P));
  std::vector<int64_t> n_owned(static_cast<size_t>(P), 0);
  for (int64_t v = 0; v < n; ++v) ++n_owned[owner[v]];
  for (int64_t p = 0; p < P; ++p) {
    parts[p].id = uint32_t(p);
    parts[p].remote_in.resize(size_t(P));
    parts[p].remote_out.resize(size_t(P));
    parts[p].owned.reserve(size_t(n_owned[p]));
  }
  for (int64_t v = 0; v < n; ++v) {
    Part& Pt = parts[owner[v]];
    Pt.owned.push_back(uint32_t(v));
    (cp[v + 1] > cp[v] ? Pt.marginal : Pt.central).push_back(uint32_t(v));
    for (int64_t k = cp[v]; k < cp[v + 1]; ++k) Pt.remote_out[cs[k]].push_back(uint32_t(v));
  }
  for (int64_t p = 0; p < P; ++p)
    for (int64_t q = 0; q < P; ++q)
      if (q != p) parts[p].remote_in[q] = parts[q].remote_out[p];
  return parts;
}

template <typename T>
void build_view_gpu(GraphDev& g, const Part& part, bool sage, bool gpu_order, View& v,
                    ViewDev<T>& d, bool host_arrays) {
  const int64_t P = g.n_parts;
  const uint32_t me = part.id;
  cudaStream_t st = g.st;
  // ---- host: row order, row maps, halo slots (aggregate.hpp:45-56) ----
  v = View{};
  v.num_owned = int64_t(part.owned.size());
  v.n_central = int64_t(part.central.size());
  v.n_marginal = int64_t(part.marginal.size());
  v.owned_sorted = part.owned;
  v.owned_gpu_row.assign(size_t(v.num_owned), -1);
  if (gpu_order) {
    v.row_node.reserve(size_t(v.num_owned));
    v.row_node.insert(v.row_node.end(), part.central.begin(), part.central.end());
    v.row_node.insert(v.row_node.end(), part.marginal.begin(), part.marginal.end());
  } else {
    v.row_node = part.owned;
  }
  v.ref_row.assign(size_t(v.num_owned), 0);
  v.gpu_row_of_ref.assign(size_t(v.num_owned), 0);
  {
    size_t ic = 0, im = 0;
    for (int64_t r = 0; r < v.num_owned; ++r) {
      const uint32_t node = part.owned[r];
      int32_t gr;
      if (!gpu_order)
        gr = int32_t(r);
      else if (ic < part.central.size() && part.central[ic] == node)
        gr = int32_t(ic++);
      else
        gr = int32_t(v.n_central + int64_t(im++));
      v.owned_gpu_row[r] = gr;
      v.ref_row[gr] = int32_t(r);
      v.gpu_row_of_ref[r] = gr;
    }
  }
  v.device_slot_offset.assign(size_t(P + 1), 0);
  for (int64_t q = 0; q < P; ++q) {
    v.device_slot_offset[q] = int64_t(v.slot_node.size());
    v.slot_node.insert(v.slot_node.end(), part.remote_in[q].begin(), part.remote_in[q].end());
  }
  v.device_slot_offset[P] = int64_t(v.slot_node.size());
  v.num_remote = int64_t(v.slot_node.size());
  const int64_t no = v.num_owned, nr = v.num_remote;

  // ---- device: row / slot maps, then the two CSR passes ----
  DBuf<uint32_t> rn, sn;
  rn.upload(v.row_node);
  sn.upload(v.slot_node);
  if (no) k_scatter_index<<<grid_for(no), kThreads, 0, st>>>(rn.p, no, g.row_of.p);
  if (nr) k_scatter_index<<<grid_for(nr), kThreads, 0, st>>>(sn.p, nr, g.slot_of.p);
  d.lptr.alloc(size_t(no + 1), true);
  d.rptr.alloc(size_t(no + 1), true);
  if (no) {
    k_view_count<<<grid_for_warps(no), kThreads, 0, st>>>(g.ptr.p, g.adj.p, g.owner.p, me, rn.p,
                                                          no, d.lptr.p, d.rptr.p);
    check_launch("k_view_count");
    scan_counts(d.lptr.p, no, st);
    scan_counts(d.rptr.p, no, st);
  }
  v.local_ptr = download(d.lptr.p, no + 1, st);
  v.remote_ptr = download(d.rptr.p, no + 1, st);
  const int64_t ln = v.local_ptr[no], rnz = v.remote_ptr[no];
  d.self_alpha.alloc(size_t(std::max<int64_t>(1, no)), false);
  d.lcol.alloc(size_t(std::max<int64_t>(1, ln)), false);
  d.lafwd.alloc(size_t(std::max<int64_t>(1, ln)), false);
  d.labwd.alloc(size_t(std::max<int64_t>(1, ln)), false);
  d.rslot.alloc(size_t(std::max<int64_t>(1, rnz)), false);
  d.ralpha.alloc(size_t(std::max<int64_t>(1, rnz)), false);
  DBuf<int32_t> erow;
  erow.alloc(size_t(std::max<int64_t>(1, rnz)), false);
  if (no) {
    k_view_fill<T><<<grid_for_warps(no), kThreads, 0, st>>>(
        g.ptr.p, g.adj.p, g.owner.p, me, rn.p, no, g.row_of.p, g.slot_of.p, sage, d.lptr.p,
        d.rptr.p, d.self_alpha.p, d.lcol.p, d.lafwd.p, d.labwd.p, d.rslot.p, d.ralpha.p, erow.p);
    check_launch("k_view_fill");
  }
  // ---- transpose of the remote CSR (stable radix sort of the entries by slot) ----
  d.sptr.alloc(size_t(nr + 1), true);
  d.srow.alloc(size_t(std::max<int64_t>(1, rnz)), false);
  d.salpha.alloc(size_t(std::max<int64_t>(1, rnz)), false);
  if (rnz) {
    k_slot_hist<<<grid_for(rnz), kThreads, 0, st>>>(d.rslot.p, rnz, d.sptr.p);
    scan_counts(d.sptr.p, nr, st);
    DBuf<int32_t> iota, perm, keys;
    iota.alloc(size_t(rnz), false);
    perm.alloc(size_t(rnz), false);
    keys.alloc(size_t(rnz), false);
    k_iota<<<grid_for(rnz), kThreads, 0, st>>>(iota.p, rnz);
    int end_bit = 1;
    while (end_bit < 32 && (int64_t(1) << end_bit) < nr) ++end_bit;
    auto* kin = reinterpret_cast<const uint32_t*>(d.rslot.p);
    auto* kout = reinterpret_cast<uint32_t*>(keys.p);
    size_t bytes = 0;
    QGNN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, iota.p, perm.p, int(rnz),
                                              0, end_bit, st));
    DBuf<uint8_t> tmp;
    tmp.alloc(std::max<size_t>(1, bytes), false);
    QGNN_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, kin, kout, iota.p, perm.p, int(rnz),
                                              0, end_bit, st));
    k_transpose_gather<T><<<grid_for(rnz), kThreads, 0, st>>>(perm.p, rnz, erow.p, d.ralpha.p,
                                                              d.srow.p, d.salpha.p);
    check_launch("k_transpose_gather");
  }
  v.slot_ptr = download(d.sptr.p, nr + 1, st);
  // ---- §8d distinct source rows per call site ----
  {
    DBuf<uint8_t> seen;
    seen.alloc(size_t(std::max<int64_t>(1, no)), false);
    DBuf<unsigned long long> cnt;
    cnt.alloc(1, false);
    auto count = [&](int64_t r0, int64_t r1) -> int64_t {
      QGNN_CUDA(cudaMemsetAsync(seen.p, 0, size_t(std::max<int64_t>(1, no)), st));
      QGNN_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
      if (r1 > r0)
        k_mark_sources<<<grid_for_warps(r1 - r0), kThreads, 0, st>>>(d.lptr.p, d.lcol.p, r0, r1,
                                                                    seen.p);
      if (no) k_count_set<<<grid_for(no), kThreads, 0, st>>>(seen.p, no, cnt.p);
      return int64_t(download(cnt.p, 1, st)[0]);
    };
    v.src_rows_central = count(0, v.n_central);
    v.src_rows_marginal = count(v.n_central, no);
    v.src_rows_all = count(0, no);
    int64_t used = 0;
    for (int64_t k = 0; k < nr; ++k) used += v.slot_ptr[k + 1] > v.slot_ptr[k];
    v.src_slots_marginal = used;
  }
  if (host_arrays) {
    auto dbl = [&](const DBuf<T>& b, int64_t m) {
      const std::vector<T> h = download(b.p, m, st);
      return std::vector<double>(h.begin(), h.end());
    };
    v.self_alpha = dbl(d.self_alpha, no);
    v.local_col = download(d.lcol.p, ln, st);
    v.local_afwd = dbl(d.lafwd, ln);
    v.local_abwd = dbl(d.labwd, ln);
    v.remote_slot = download(d.rslot.p, rnz, st);
    v.remote_alpha = dbl(d.ralpha, rnz);
    v.slot_row = download(d.srow.p, rnz, st);
    v.slot_alpha = dbl(d.salpha, rnz);
  }
  QGNN_CUDA(cudaStreamSynchronize(st));
}

template void build_view_gpu<float>(GraphDev&, const Part&, bool, bool, View&, ViewDev<float>&,
                                    bool);
template void build_view_gpu<double>(GraphDev&, const Part&, bool, bool, View&, ViewDev<double>&,
                                     bool);

std::vector<std::vector<std::vector<double>>> rx_alpha_sq_gpu(GraphDev& g,
                                                              const std::vector<Part>& parts,
                                                              bool sage) {
  const int64_t P = int64_t(parts.size());
  std::vector<uint32_t> ids, dst;
  for (int64_t p = 0; p < P; ++p)
    for (int64_t q = 0; q < P; ++q) {
      if (p == q) continue;
      const auto& l = parts[p].remote_out[q];
      ids.insert(ids.end(), l.begin(), l.end());
      dst.insert(dst.end(), l.size(), uint32_t(q));
    }
  const int64_t m = int64_t(ids.size());
  std::vector<double> acc;
  if (m) {
    DBuf<uint32_t> di, dd;
    DBuf<double> out;
    di.upload(ids);
    dd.upload(dst);
    out.alloc(size_t(m), false);
    k_rx_asq<<<grid_for(m), kThreads, 0, g.st>>>(g.ptr.p, g.adj.p, g.owner.p, di.p, dd.p, m, sage,
                                                 out.p);
    check_launch("k_rx_asq");
    acc = download(out.p, m, g.st);
  }
  std::vector<std::vector<std::vector<double>>> r(static_cast<size_t>(P));
  for (auto& x : r) x.resize(static_cast<size_t>(P));
  int64_t k = 0;
  for (int64_t p = 0; p < P; ++p)
    for (int64_t q = 0; q < P; ++q) {
      if (p == q) continue;
      const size_t c = parts[p].remote_out[q].size();
      r[p][q].assign(acc.begin() + k, acc.begin() + k + int64_t(c));
      k += int64_t(c);
    }
  return r;
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

namespace {
struct SetupStream {  // private non-blocking stream on the caller's device
  cudaStream_t s = nullptr;
  explicit SetupStream(int device) {
    QGNN_CUDA(cudaSetDevice(device));
    QGNN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~SetupStream() {
    if (s) cudaStreamDestroy(s);
  }
};
}  // namespace

extern "C" {

int qgnn_partitions_from_owner_gpu(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                                   const uint32_t* owner, int64_t n_parts, int device,
                                   qgnn_partition** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(adj_ptr && owner && out, QGNN_EINVAL, "partitions: null argument");
  SetupStream ss(device);
  GraphDev g(adj_ptr, adj, n, owner, n_parts, ss.s);
  std::vector<Part> parts = partitions_from_owner_gpu(g, owner);
  for (int64_t p = 0; p < n_parts; ++p) {
    out[p] = new qgnn_partition;
    out[p]->part = std::move(parts[p]);
  }
  QGNN_API_END
}

int qgnn_agg_view_build_gpu(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                            const uint32_t* owner, const qgnn_partition* part, int sage,
                            int device, qgnn_agg_view** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(adj_ptr && part && out && owner, QGNN_EINVAL, "agg_view: null argument");
  const Part& P = part->part;
  const int64_t n_parts = int64_t(P.remote_in.size());
  SetupStream ss(device);
  GraphDev g(adj_ptr, adj, n, owner, n_parts, ss.s);
  View v;
  ViewDev<double> d;
  build_view_gpu<double>(g, P, sage != 0, false, v, d, true);
  auto* V = new qgnn_agg_view;
  V->num_owned = v.num_owned;
  V->num_remote = v.num_remote;
  V->self_alpha = std::move(v.self_alpha);
  V->local_ptr = std::move(v.local_ptr);
  V->local_row.assign(v.local_col.begin(), v.local_col.end());
  V->local_alpha_fwd = std::move(v.local_afwd);
  V->local_alpha_bwd = std::move(v.local_abwd);
  V->remote_ptr = std::move(v.remote_ptr);
  V->remote_slot.assign(v.remote_slot.begin(), v.remote_slot.end());
  V->remote_alpha = std::move(v.remote_alpha);
  V->slot_node = std::move(v.slot_node);
  V->device_slot_offset = std::move(v.device_slot_offset);
  for (int64_t q = 0; q < n_parts; ++q)
    V->slot_owner.insert(V->slot_owner.end(),
                         size_t(V->device_slot_offset[q + 1] - V->device_slot_offset[q]), uint32_t(q));
  for (int64_t i = 0; i < V->num_owned; ++i)
    (V->remote_ptr[i + 1] > V->remote_ptr[i] ? V->marginal_rows : V->central_rows).push_back(uint32_t(i));
  *out = V;
  QGNN_API_END
}

}  // extern "C"
