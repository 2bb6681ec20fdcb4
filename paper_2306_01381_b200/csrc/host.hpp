// host.hpp — C++ host runtime shared by the C-ABI and the GPU engine:
// partitioning, halo layout, aggregation views, plans and the bit-width
// solver.  All of it is setup / control-plane work that runs once per run or
// once per plan version; the per-epoch data path lives on the GPU.
#pragma once

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

namespace qgnn_b200 {

// ---- graphcore/partition.hpp:16-23 -----------------------------------------
struct Part {
  uint32_t id = 0;
  std::vector<uint32_t> owned, central, marginal;  // ascending node ids
  std::vector<std::vector<uint32_t>> remote_in;    // [q] nodes owned by q consumed here
  std::vector<std::vector<uint32_t>> remote_out;   // [q] owned nodes consumed by q
};

// partition.hpp:90-135 (seeded BFS region growing) -> owner map
std::vector<uint32_t> partition_owner_bfs(const int64_t* ptr, const int32_t* adj, int64_t n,
                                          int64_t n_parts, uint64_t seed);
// partition.hpp:39-84
std::vector<Part> partitions_from_owner(const int64_t* ptr, const int32_t* adj, int64_t n,
                                        const uint32_t* owner, int64_t n_parts);
// coeffs.hpp:30-45
void compute_coeffs(const int64_t* ptr, const int32_t* adj, int64_t n, bool sage,
                    std::vector<double>& alpha, std::vector<double>& self_alpha);

// ---- tensorops/aggregate.hpp:17-90, re-laid out for the GPU -----------------
// GPU row order: central rows (ascending id) then marginal rows (ascending id),
// so the central/marginal subsets are contiguous row ranges.  ref_row[g] is
// the reference's owned-row index of GPU row g (ascending id order).
struct View {
  int64_t num_owned = 0, num_remote = 0, n_central = 0, n_marginal = 0;
  std::vector<uint32_t> row_node;     // GPU row -> node id
  std::vector<int32_t> ref_row;       // GPU row -> reference owned-row index
  std::vector<int32_t> gpu_row_of_ref;  // reference row -> GPU row
  std::vector<double> self_alpha;     // per GPU row
  std::vector<int64_t> local_ptr;     // CSR over GPU rows (neighbour order = adjacency order)
  std::vector<int32_t> local_col;     // GPU row of the neighbour
  std::vector<double> local_afwd, local_abwd;
  std::vector<int64_t> remote_ptr;
  std::vector<int32_t> remote_slot;
  std::vector<double> remote_alpha;
  // transpose of the remote CSR: slot -> contributing marginal GPU rows in
  // ascending reference-row order (backward_remote_partials, aggregate.hpp:156-163)
  std::vector<int64_t> slot_ptr;
  std::vector<int32_t> slot_row;
  std::vector<double> slot_alpha;
  std::vector<int64_t> device_slot_offset;  // n_parts + 1
  std::vector<uint32_t> slot_node;
  std::vector<std::vector<double>> rx_alpha_sq;  // [src][i] engine.hpp:262-273
  // gpu row of owned node id (sorted owned ids + rows for lookup)
  int32_t gpu_row(uint32_t node) const;
  std::vector<uint32_t> owned_sorted;   // == Part::owned
  std::vector<int32_t> owned_gpu_row;   // GPU row of owned_sorted[i]
  // distinct source rows per SpMM call site (self rows included; §8d bytes)
  int64_t src_rows_central = 0, src_rows_marginal = 0, src_rows_all = 0, src_slots_marginal = 0;
  // (the GPU setup keeps the edge arrays on the device only: counts from the pointers)
  int64_t local_nnz() const { return local_ptr.empty() ? 0 : local_ptr.back(); }
  int64_t remote_nnz() const { return remote_ptr.empty() ? 0 : remote_ptr.back(); }
};

// build_graph (graph.hpp:59-78): symmetrize, drop self loops, sort and deduplicate
// every adjacency list.  device >= 0: radix sort of the directed pairs on that GPU
// (setup.cu); device < 0: on the host.
void build_graph_csr(int64_t n, const std::vector<std::pair<uint32_t, uint32_t>>& edges,
                     int device, std::vector<int64_t>& ptr, std::vector<int32_t>& adj);

View build_view(const int64_t* ptr, const int32_t* adj, int64_t n, const Part& part,
                int64_t n_parts, const std::vector<double>& alpha,
                const std::vector<double>& self_alpha, bool sage);

// ---- assigner (trace.hpp / plan.hpp / solve.hpp) ----------------------------
struct MsgStat {
  uint32_t id = 0;
  uint64_t dim = 0;
  double lo = 0, hi = 0, asq = 0;
  uint32_t pos = 0;  // caller's index of the message (carried into Group::pos)
};
struct PairStat {
  uint32_t src = 0, dst = 0;
  std::vector<MsgStat> msgs;  // ascending id
};
struct Group {
  std::vector<uint32_t> ids;
  std::vector<uint32_t> pos;  // MsgStat::pos of each id
  std::vector<uint64_t> dims;
  double beta = 0;
  int bits = 8;
  uint64_t dim_sum() const;
};
struct PlanPairG {
  uint32_t src = 0, dst = 0;
  std::vector<Group> groups;
};
struct SolveResult {
  std::vector<PlanPairG> pairs;
  double objective = 0, variance = 0, z = 0;
};
struct Cost {
  int64_t n = 0;
  std::vector<double> theta, gamma;  // src * n + dst
  double seconds(int64_t s, int64_t d, double bits) const {
    const int64_t i = s * n + d;
    return theta[i] * bits + gamma[i];
  }
};

double compute_beta(const MsgStat& m);  // trace.hpp:71-74
SolveResult group_and_order(const std::vector<PairStat>& pairs, int64_t group_size);
void solve_exact(SolveResult& plan, const Cost& cm, double lambda);   // solve.hpp:264-309
void solve_brute(SolveResult& plan, const Cost& cm, double lambda);   // solve.hpp:220-258
double uniform_expected_variance(const std::vector<PairStat>& pairs);  // solve.hpp:313-326

}  // namespace qgnn_b200

// C-ABI handles (include/qgnn_b200.h): a partition and a reference-order view
struct qgnn_partition {
  qgnn_b200::Part part;
};
struct qgnn_agg_view {
  std::vector<double> self_alpha, local_alpha_fwd, local_alpha_bwd, remote_alpha;
  std::vector<int64_t> local_ptr, remote_ptr, device_slot_offset;
  std::vector<uint32_t> local_row, remote_slot, slot_node, slot_owner, central_rows, marginal_rows;
  int64_t num_owned = 0, num_remote = 0;
};
