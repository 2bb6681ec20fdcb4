// setup.cuh — GPU-side graph setup: the reference's
// partitions_from_owner (graphcore/partition.hpp:39-84), compute_coeffs
// (graphcore/coeffs.hpp:30-45), DeviceAggView::build (tensorops/aggregate.hpp:41-89)
// and the receivers' squared consumption weights (trainer/engine.hpp:262-273),
// computed from a device-resident copy of the graph.  Outputs are identical to
// the host builders in host_graph.cpp (same lists, same fp64 coefficient
// arithmetic: mul, sqrt and div each correctly rounded, no contraction).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "dbuf.cuh"
#include "host.hpp"

namespace qgnn_b200 {

// The CSR graph and owner map resident on the device for the duration of setup.
struct GraphDev {
  int64_t n = 0, nnz = 0, n_parts = 0;
  DBuf<int64_t> ptr;
  DBuf<int32_t> adj;
  DBuf<uint32_t> owner;
  DBuf<int32_t> row_of, slot_of;  // per node: row in its view / halo slot (scratch)
  cudaStream_t st = nullptr;
  GraphDev(const int64_t* ptr, const int32_t* adj, int64_t n, const uint32_t* owner,
           int64_t n_parts, cudaStream_t st);
};

// partitions_from_owner: consumer sets per node on the device (warp per node,
// shared-memory bitmap over the P partitions), lists assembled on the host in
// one pass over the node ids.
std::vector<Part> partitions_from_owner_gpu(GraphDev& g, const uint32_t* owner_host);

// Device arrays of one view, in the engine's dtype (fp64 for the C-ABI view).
template <typename T>
struct ViewDev {
  DBuf<T> self_alpha, lafwd, labwd, ralpha, salpha;
  DBuf<int64_t> lptr, rptr, sptr;
  DBuf<int32_t> lcol, rslot, srow;
};

// DeviceAggView::build for `part` with rows in GPU order (central then
// marginal, gpu_order) or the reference's order (owned ascending).  Host side:
// v's row maps, slot lists, local/remote/slot pointers and the §8d source-row
// counts; device side: every per-edge array in d.  host_arrays also downloads
// the per-edge arrays into v (C-ABI view, tests).
template <typename T>
void build_view_gpu(GraphDev& g, const Part& part, bool sage, bool gpu_order, View& v,
                    ViewDev<T>& d, bool host_arrays);

// engine.hpp:262-273 for every ordered pair (p, q): out[p][q][i] = Σ α² over the
// neighbours owned by q of remote_out[p][q][i], ascending neighbour order.
std::vector<std::vector<std::vector<double>>> rx_alpha_sq_gpu(GraphDev& g,
                                                              const std::vector<Part>& parts,
                                                              bool sage);

}  // namespace qgnn_b200
