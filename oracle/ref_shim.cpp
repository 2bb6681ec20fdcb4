// ref_shim.cpp — extern "C" adapter over the UNMODIFIED reference headers
// (/root/reference/proj/include/qgnn/...), compiled by oracle/Makefile into
// oracle/_ref/libqgnn_ref.so.
//
// TEST INFRASTRUCTURE ONLY: this is the checker that pins oracle/qgnn_oracle.c
// and generates tests/golden/ fixtures; it is also bench.py's CPU baseline
// ("kind": "reference").  The product never links it.  No reference source is
// copied here: the reference headers are #included from where they lie.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "qgnn/assigner/plan.hpp"
#include "qgnn/assigner/solve.hpp"
#include "qgnn/cli/synth.hpp"
#include "qgnn/graphcore/coeffs.hpp"
#include "qgnn/graphcore/partition.hpp"
#include "qgnn/quantcodec/codec.hpp"
#include "qgnn/quantcodec/quant.hpp"
#include "qgnn/quantcodec/rng.hpp"
#include "qgnn/tensorops/aggregate.hpp"
#include "qgnn/tensorops/model.hpp"

// Partitioner interposition for the Engine (engine.hpp:212 calls
// partition_graph).  When ref_engine_run is given an owner map, the Engine
// partitions with the reference's own partitions_from_owner
// (partition.hpp:39-84, the halo-layout API SURVEY.md §8e names for the
// planted-block configs) instead of the BFS partition_graph; with no owner
// map it calls partition_graph unchanged.  Only the one call token is
// redirected; the header text is untouched.
namespace qgnn::shim_hook {
inline const std::vector<uint32_t>* g_owner = nullptr;
inline std::vector<Partition> partition_graph(const Graph& g, std::size_t n_parts,
                                              uint64_t seed) {
  if (g_owner) return qgnn::partitions_from_owner(g, *g_owner, n_parts);
  return qgnn::partition_graph(g, n_parts, seed);
}
}  // namespace qgnn::shim_hook
#define partition_graph shim_hook::partition_graph
#include "qgnn/trainer/engine.hpp"
#undef partition_graph

using namespace qgnn;

namespace {
thread_local std::string g_err;

int map_exc() {
  try {
    throw;
  } catch (const DecodeError& e) {
    g_err = e.what();
    return 2;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 3;
  } catch (const ResourceLimitError& e) {
    g_err = e.what();
    return 4;
  } catch (const DivergedError& e) {
    g_err = e.what();
    return 5;
  } catch (const IoError& e) {
    g_err = e.what();
    return 6;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

#define GUARD(...)     \
  try {                \
    __VA_ARGS__;       \
    return 0;          \
  } catch (...) {      \
    return map_exc();  \
  }

// Rebuilds a reference Graph from CSR arrays.
Graph graph_from_csr(const int64_t* adj_ptr, const int32_t* adj, uint64_t n) {
  Graph g;
  g.num_nodes = n;
  g.adj_ptr.assign(adj_ptr, adj_ptr + n + 1);
  g.adj.assign(adj, adj + adj_ptr[n]);
  return g;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- rng ----------------------------------------------------------------
// Draws `n` u64 values from RngStream(seed).fork(coords...) (rng.hpp:13-61).
int ref_rng_draws(uint64_t seed, const uint64_t* coords, int n_coords, uint64_t n, uint64_t* out) {
  GUARD({
    RngStream r(seed);
    for (int i = 0; i < n_coords; ++i) r = r.fork(coords[i]);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
  })
}

int ref_rng_gaussians(uint64_t seed, const uint64_t* coords, int n_coords, uint64_t n, double* out) {
  GUARD({
    RngStream r(seed);
    for (int i = 0; i < n_coords; ++i) r = r.fork(coords[i]);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_gaussian();
  })
}

// ---- quant ----------------------------------------------------------------
// quantize(h, b, RngStream(seed).fork(coords...)) -> scale, zero, payload
int ref_quantize(const double* h, uint64_t n, int b, uint64_t seed, const uint64_t* coords,
                 int n_coords, double* scale, double* zero, uint8_t* payload) {
  GUARD({
    RngStream r(seed);
    for (int i = 0; i < n_coords; ++i) r = r.fork(coords[i]);
    const QuantizedChunk c = quantize(std::span<const double>(h, n), b, r);
    *scale = c.scale;
    *zero = c.zero_point;
    std::memcpy(payload, c.payload.data(), c.payload.size());
  })
}

int ref_pack(const uint32_t* codes, uint64_t n, int b, uint8_t* out) {
  GUARD({
    const auto v = pack(std::span<const uint32_t>(codes, n), b);
    std::memcpy(out, v.data(), v.size());
  })
}

// encode_message_set over rows of `values` (stride ld): message i = row rows[i], id ids[i],
// width bits[i]; stream RngStream(seed).fork(coords...).  Outputs wire bytes and the
// retrieval index (entry k: id, bits, offset, dim).
int ref_encode_message_set(const double* values, uint64_t ld, const int64_t* rows,
                           const uint32_t* ids, const int32_t* bits, uint64_t n, uint64_t dim,
                           uint64_t seed, const uint64_t* coords, int n_coords, uint8_t* out,
                           uint64_t* out_bytes, uint32_t* e_id, int32_t* e_bits, uint64_t* e_off,
                           uint64_t* e_dim) {
  GUARD({
    RngStream r(seed);
    for (int i = 0; i < n_coords; ++i) r = r.fork(coords[i]);
    std::vector<MessageView> msgs(n);
    std::map<uint32_t, int> bit_of;
    for (uint64_t i = 0; i < n; ++i) {
      msgs[i] = {ids[i], std::span<const double>(values + rows[i] * ld, dim)};
      bit_of[ids[i]] = bits[i];
    }
    const EncodedSet set =
        encode_message_set(msgs, [&](uint32_t id) { return bit_of.at(id); }, r);
    std::memcpy(out, set.bytes.data(), set.bytes.size());
    *out_bytes = set.bytes.size();
    for (std::size_t k = 0; k < set.index.entries.size(); ++k) {
      e_id[k] = set.index.entries[k].id;
      e_bits[k] = set.index.entries[k].bit_width;
      e_off[k] = set.index.entries[k].offset;
      e_dim[k] = set.index.entries[k].dim;
    }
  })
}

int ref_decode_message_set(const uint8_t* bytes, uint64_t nbytes, const uint32_t* e_id,
                           const int32_t* e_bits, const uint64_t* e_off, const uint64_t* e_dim,
                           uint64_t n, uint64_t total_bytes, double* out, uint64_t ld) {
  GUARD({
    RetrievalIndex idx;
    idx.total_bytes = total_bytes;
    for (uint64_t k = 0; k < n; ++k)
      idx.entries.push_back({e_id[k], static_cast<uint8_t>(e_bits[k]), e_off[k], e_dim[k]});
    const auto dec = decode_message_set(std::span<const uint8_t>(bytes, nbytes), idx);
    for (std::size_t k = 0; k < dec.size(); ++k)
      std::memcpy(out + k * ld, dec[k].values.data(), dec[k].values.size() * sizeof(double));
  })
}

// ---- graph / partition / coeffs / view --------------------------------------
struct RefDataset {
  Graph g;
};

// generate_dataset (cli/synth.hpp:55-149).  kind 0 = sbm, 1 = cite.
void* ref_generate_dataset(int kind, uint64_t nodes, uint64_t classes, uint64_t feature_dim,
                           double p_intra, double p_inter, uint64_t attach_edges,
                           double same_class_bias, double sep, uint64_t seed) {
  try {
    DatasetSpec s;
    s.kind = kind ? SynthKind::kCite : SynthKind::kSbm;
    s.nodes = nodes;
    s.classes = classes;
    s.feature_dim = feature_dim;
    s.p_intra = p_intra;
    s.p_inter = p_inter;
    s.attach_edges = attach_edges;
    s.same_class_bias = same_class_bias;
    s.sep = sep;
    s.seed = seed;
    auto* d = new RefDataset{generate_dataset(s)};
    return d;
  } catch (...) {
    map_exc();
    return nullptr;
  }
}

void ref_dataset_free(void* d) { delete static_cast<RefDataset*>(d); }

// save_dataset / load_dataset (cli/synth.hpp:153-205)
int ref_dataset_save(void* d, const char* dir) {
  try {
    save_dataset(static_cast<RefDataset*>(d)->g, dir);
    return 0;
  } catch (...) {
    return map_exc();
  }
}
void* ref_dataset_load(const char* dir) {
  try {
    return new RefDataset{load_dataset(dir)};
  } catch (...) {
    map_exc();
    return nullptr;
  }
}

// sizes: nodes, nnz, feature cols
void ref_dataset_sizes(void* d, uint64_t* nodes, uint64_t* nnz, uint64_t* fdim) {
  const Graph& g = static_cast<RefDataset*>(d)->g;
  *nodes = g.num_nodes;
  *nnz = g.adj.size();
  *fdim = g.features.cols;
}

void ref_dataset_export(void* d, int64_t* adj_ptr, int32_t* adj, double* features,
                        int32_t* labels, uint8_t* train, uint8_t* val, uint8_t* test) {
  const Graph& g = static_cast<RefDataset*>(d)->g;
  for (std::size_t i = 0; i <= g.num_nodes; ++i) adj_ptr[i] = static_cast<int64_t>(g.adj_ptr[i]);
  for (std::size_t i = 0; i < g.adj.size(); ++i) adj[i] = static_cast<int32_t>(g.adj[i]);
  std::memcpy(features, g.features.data.data(), g.features.data.size() * sizeof(double));
  for (std::size_t i = 0; i < g.num_nodes; ++i) {
    labels[i] = g.labels[i];
    train[i] = g.train_mask[i];
    val[i] = g.val_mask[i];
    test[i] = g.test_mask[i];
  }
}

// partition_graph (partition.hpp:90-135) -> owner per node
int ref_partition_owner(const int64_t* adj_ptr, const int32_t* adj, uint64_t n, uint64_t n_parts,
                        uint64_t seed, uint32_t* owner) {
  GUARD({
    const Graph g = graph_from_csr(adj_ptr, adj, n);
    const auto parts = partition_graph(g, n_parts, seed);
    for (const Partition& p : parts)
      for (NodeId v : p.owned) owner[v] = p.device_id;
  })
}

// compute_coeffs (coeffs.hpp:30-45)
int ref_compute_coeffs(const int64_t* adj_ptr, const int32_t* adj, uint64_t n, int sage,
                       double* alpha, double* self_alpha) {
  GUARD({
    const Graph g = graph_from_csr(adj_ptr, adj, n);
    const AggCoeffs c = compute_coeffs(g, sage ? AggMode::kSageMean : AggMode::kGcn);
    std::memcpy(alpha, c.alpha.data(), c.alpha.size() * sizeof(double));
    std::memcpy(self_alpha, c.self_alpha.data(), c.self_alpha.size() * sizeof(double));
  })
}

// Partition + DeviceAggView for device `dev` under an owner map, exported flat.
struct RefView {
  Partition part;
  DeviceAggView view;
};

void* ref_view_build(const int64_t* adj_ptr, const int32_t* adj, uint64_t n,
                     const uint32_t* owner, uint64_t n_parts, uint32_t dev, int sage) {
  try {
    const Graph g = graph_from_csr(adj_ptr, adj, n);
    const auto parts = partitions_from_owner(g, std::vector<uint32_t>(owner, owner + n), n_parts);
    const AggCoeffs c = compute_coeffs(g, sage ? AggMode::kSageMean : AggMode::kGcn);
    auto* v = new RefView{parts[dev], DeviceAggView::build(g, parts[dev], c)};
    return v;
  } catch (...) {
    map_exc();
    return nullptr;
  }
}

void ref_view_free(void* v) { delete static_cast<RefView*>(v); }

// counts: [num_owned, num_remote, local_nnz, remote_nnz, n_central, n_marginal]
void ref_view_counts(void* pv, uint64_t* c) {
  const auto& v = static_cast<RefView*>(pv)->view;
  c[0] = v.num_owned;
  c[1] = v.num_remote;
  c[2] = v.local_row.size();
  c[3] = v.remote_slot.size();
  c[4] = v.central_rows.size();
  c[5] = v.marginal_rows.size();
}

void ref_view_export(void* pv, double* self_alpha, int64_t* local_ptr, int32_t* local_row,
                     double* local_alpha_fwd, double* local_alpha_bwd, int64_t* remote_ptr,
                     int32_t* remote_slot, double* remote_alpha, uint32_t* slot_node,
                     uint32_t* slot_owner, int64_t* device_slot_offset, int32_t* central,
                     int32_t* marginal, uint32_t* owned) {
  const auto& rv = *static_cast<RefView*>(pv);
  const auto& v = rv.view;
  for (std::size_t i = 0; i < v.num_owned; ++i) self_alpha[i] = v.self_alpha[i];
  for (std::size_t i = 0; i <= v.num_owned; ++i) {
    local_ptr[i] = static_cast<int64_t>(v.local_ptr[i]);
    remote_ptr[i] = static_cast<int64_t>(v.remote_ptr[i]);
  }
  for (std::size_t i = 0; i < v.local_row.size(); ++i) {
    local_row[i] = static_cast<int32_t>(v.local_row[i]);
    local_alpha_fwd[i] = v.local_alpha_fwd[i];
    local_alpha_bwd[i] = v.local_alpha_bwd[i];
  }
  for (std::size_t i = 0; i < v.remote_slot.size(); ++i) {
    remote_slot[i] = static_cast<int32_t>(v.remote_slot[i]);
    remote_alpha[i] = v.remote_alpha[i];
  }
  for (std::size_t i = 0; i < v.num_remote; ++i) {
    slot_node[i] = v.slot_node[i];
    slot_owner[i] = v.slot_owner[i];
  }
  for (std::size_t i = 0; i < v.device_slot_offset.size(); ++i)
    device_slot_offset[i] = static_cast<int64_t>(v.device_slot_offset[i]);
  for (std::size_t i = 0; i < v.central_rows.size(); ++i) central[i] = v.central_rows[i];
  for (std::size_t i = 0; i < v.marginal_rows.size(); ++i) marginal[i] = v.marginal_rows[i];
  for (std::size_t i = 0; i < rv.part.owned.size(); ++i) owned[i] = rv.part.owned[i];
}

// remote_in / remote_out list sizes and contents for device `dev`: flattened by q.
void ref_view_remote_lists(void* pv, uint64_t n_parts, uint64_t* in_sizes, uint64_t* out_sizes,
                           uint32_t* in_ids, uint32_t* out_ids) {
  const auto& p = static_cast<RefView*>(pv)->part;
  uint64_t a = 0, b = 0;
  for (uint64_t q = 0; q < n_parts; ++q) {
    in_sizes[q] = p.remote_in[q].size();
    out_sizes[q] = p.remote_out[q].size();
    if (in_ids)
      for (auto id : p.remote_in[q]) in_ids[a++] = id;
    if (out_ids)
      for (auto id : p.remote_out[q]) out_ids[b++] = id;
  }
}

// aggregate_rows / aggregate_backward_local / backward_remote_partials on a view
int ref_view_aggregate_rows(void* pv, const double* h, const double* h_remote, uint64_t d,
                            const uint32_t* rows, uint64_t n_rows, double* out) {
  GUARD({
    const auto& v = static_cast<RefView*>(pv)->view;
    Matrix H(v.num_owned, d), R(v.num_remote, d), O(v.num_owned, d);
    std::memcpy(H.data.data(), h, H.data.size() * sizeof(double));
    if (v.num_remote) std::memcpy(R.data.data(), h_remote, R.data.size() * sizeof(double));
    std::memcpy(O.data.data(), out, O.data.size() * sizeof(double));
    aggregate_rows(v, H, R, std::span<const uint32_t>(rows, n_rows), O);
    std::memcpy(out, O.data.data(), O.data.size() * sizeof(double));
  })
}

int ref_view_aggregate_backward_local(void* pv, const double* gbar, uint64_t d,
                                      const uint32_t* rows, uint64_t n_rows, double* out) {
  GUARD({
    const auto& v = static_cast<RefView*>(pv)->view;
    Matrix G(v.num_owned, d), O(v.num_owned, d);
    std::memcpy(G.data.data(), gbar, G.data.size() * sizeof(double));
    std::memcpy(O.data.data(), out, O.data.size() * sizeof(double));
    aggregate_backward_local(v, G, std::span<const uint32_t>(rows, n_rows), O);
    std::memcpy(out, O.data.data(), O.data.size() * sizeof(double));
  })
}

int ref_view_backward_remote_partials(void* pv, const double* gbar, uint64_t d, double* out) {
  GUARD({
    const auto& v = static_cast<RefView*>(pv)->view;
    Matrix G(v.num_owned, d);
    std::memcpy(G.data.data(), gbar, G.data.size() * sizeof(double));
    const Matrix P = backward_remote_partials(v, G);
    std::memcpy(out, P.data.data(), P.data.size() * sizeof(double));
  })
}

// ---- dense ------------------------------------------------------------------
int ref_layer_forward_rows(const double* h_agg, uint64_t n, const double* w, uint64_t din,
                           uint64_t dout, int relu, const uint32_t* rows, uint64_t n_rows,
                           double* out) {
  GUARD({
    GnnLayer layer;
    layer.weight = Matrix(din, dout);
    std::memcpy(layer.weight.data.data(), w, din * dout * sizeof(double));
    layer.act = relu ? Activation::kRelu : Activation::kNone;
    GnnModel model;
    LayerCache cache;
    cache.h_agg = Matrix(n, din);
    std::memcpy(cache.h_agg.data.data(), h_agg, n * din * sizeof(double));
    cache.pre_act = Matrix(n, dout);
    Matrix O(n, dout);
    std::memcpy(O.data.data(), out, n * dout * sizeof(double));
    layer_forward_rows(layer, model, cache, std::span<const uint32_t>(rows, n_rows), O,
                       RngStream(0));
    std::memcpy(out, O.data.data(), n * dout * sizeof(double));
  })
}

int ref_input_grad_rows(const double* dz, uint64_t n, const double* w, uint64_t din,
                        uint64_t dout, const uint32_t* rows, uint64_t n_rows, double* out) {
  GUARD({
    GnnLayer layer;
    layer.weight = Matrix(din, dout);
    std::memcpy(layer.weight.data.data(), w, din * dout * sizeof(double));
    Matrix DZ(n, dout), O(n, din);
    std::memcpy(DZ.data.data(), dz, n * dout * sizeof(double));
    std::memcpy(O.data.data(), out, n * din * sizeof(double));
    input_grad_rows(layer, DZ, std::span<const uint32_t>(rows, n_rows), O);
    std::memcpy(out, O.data.data(), n * din * sizeof(double));
  })
}

int ref_matmul_transa(const double* a, const double* b, uint64_t k, uint64_t m, uint64_t n,
                      double* out) {
  GUARD({
    Matrix A(k, m), B(k, n);
    std::memcpy(A.data.data(), a, k * m * sizeof(double));
    std::memcpy(B.data.data(), b, k * n * sizeof(double));
    const Matrix O = matmul_transa(A, B);
    std::memcpy(out, O.data.data(), m * n * sizeof(double));
  })
}

// GnnModel::init weights (model.hpp:27-41), concatenated layer by layer
int ref_model_init(const uint64_t* dims, int n_dims, uint64_t seed, double* out) {
  GUARD({
    const auto m = GnnModel::init(AggMode::kGcn, std::vector<std::size_t>(dims, dims + n_dims), seed);
    std::size_t o = 0;
    for (const auto& l : m.layers) {
      std::memcpy(out + o, l.weight.data.data(), l.weight.data.size() * sizeof(double));
      o += l.weight.data.size();
    }
  })
}

// ---- assigner ---------------------------------------------------------------
// Instance encoding (flat): pairs (src, dst, n_msgs) with messages (id, dim, lo, hi, sum_alpha_sq).
static InstanceStats decode_instance(uint64_t n_pairs, const uint32_t* pair_src,
                                     const uint32_t* pair_dst, const uint64_t* pair_count,
                                     const uint32_t* m_id, const uint64_t* m_dim,
                                     const double* m_lo, const double* m_hi,
                                     const double* m_asq) {
  InstanceStats inst;
  uint64_t o = 0;
  for (uint64_t p = 0; p < n_pairs; ++p) {
    PairStats ps;
    ps.src = pair_src[p];
    ps.dst = pair_dst[p];
    for (uint64_t i = 0; i < pair_count[p]; ++i, ++o)
      ps.messages.push_back({m_id[o], m_dim[o], m_lo[o], m_hi[o], m_asq[o]});
    inst.pairs.push_back(std::move(ps));
  }
  return inst;
}

// group_and_order + solve_assignment (or brute force): per message bits in the
// same flat order as the input; returns objective/variance/z.
int ref_solve_instance(uint64_t n_pairs, const uint32_t* pair_src, const uint32_t* pair_dst,
                       const uint64_t* pair_count, const uint32_t* m_id, const uint64_t* m_dim,
                       const double* m_lo, const double* m_hi, const double* m_asq,
                       uint64_t n_devices, const double* theta, const double* gamma,
                       double lambda, uint64_t group_size, int brute, int32_t* out_bits,
                       double* out_eval) {
  GUARD({
    const InstanceStats inst =
        decode_instance(n_pairs, pair_src, pair_dst, pair_count, m_id, m_dim, m_lo, m_hi, m_asq);
    CostModel cm;
    cm.num_devices = n_devices;
    cm.theta.assign(theta, theta + n_devices * n_devices);
    cm.gamma.assign(gamma, gamma + n_devices * n_devices);
    InstancePlan plan = group_and_order(inst, group_size);
    const SolveEval ev = brute ? brute_force_assignment(plan, cm, lambda)
                               : solve_assignment(plan, cm, lambda);
    out_eval[0] = ev.objective;
    out_eval[1] = ev.variance_term;
    out_eval[2] = ev.z_seconds;
    std::map<std::pair<uint32_t, uint32_t>, std::map<uint32_t, int>> bits;
    for (const PlanPair& pp : plan.pairs)
      for (const PlanGroup& g : pp.groups)
        for (uint32_t id : g.ids) bits[{pp.src, pp.dst}][id] = g.bits;
    uint64_t o = 0;
    for (uint64_t p = 0; p < n_pairs; ++p)
      for (uint64_t i = 0; i < pair_count[p]; ++i, ++o)
        out_bits[o] = bits[{pair_src[p], pair_dst[p]}][m_id[o]];
  })
}

// ---- engine -----------------------------------------------------------------
// Runs the reference Engine (trainer/engine.hpp) on a generated dataset and
// reports per-epoch (loss, val_acc, test_acc, bytes_total, msgs_b2, msgs_b4,
// msgs_b8, msgs_fp, plan_version, wall_seconds) and final weights.
// bit_mode: 0 fp, 1 fixed, 2 uniform, 3 adaptive.  threads != 0 -> kThreads.
// owner != NULL: partitions_from_owner(g, owner) instead of partition_graph
// (see shim_hook above).  times_out (optional, 2 doubles): Engine
// construction seconds and run() seconds (epoch_out[.., 9] = run() / epochs,
// setup excluded).  layer_norm / dropout: TrainSettings::layer_norm / dropout.
int ref_engine_run(void* dataset, const uint64_t* dims, int n_dims, int sage, int bit_mode,
                   int fixed_bits, double lambda, uint64_t group_size, uint64_t period,
                   uint64_t epochs, uint64_t seed, uint64_t n_parts, int threads, double theta,
                   double gamma, double lr, double* epoch_out, double* final_weights,
                   const uint32_t* owner, double* times_out, int layer_norm, double dropout) {
  GUARD({
    const Graph& g = static_cast<RefDataset*>(dataset)->g;
    TrainSettings s;
    s.agg = sage ? AggMode::kSageMean : AggMode::kGcn;
    s.dims.assign(dims, dims + n_dims);
    s.opt = OptKind::kAdam;
    s.lr = lr;
    s.bit_mode = static_cast<BitMode>(bit_mode);
    s.fixed_bits = fixed_bits;
    s.lambda = lambda;
    s.group_size = group_size;
    s.period = period;
    s.epochs = epochs;
    s.seed = seed;
    s.n_parts = n_parts;
    s.exec = threads ? ExecMode::kThreads : ExecMode::kRoundRobin;
    s.cost = CostModel::uniform(n_parts, theta, gamma);
    s.layer_norm = layer_norm != 0;  // TrainSettings (engine.hpp:42-43)
    s.dropout = dropout;
    std::vector<uint32_t> own;
    if (owner) own.assign(owner, owner + g.num_nodes);
    const auto ts = std::chrono::steady_clock::now();
    shim_hook::g_owner = owner ? &own : nullptr;
    struct Reset {
      ~Reset() { shim_hook::g_owner = nullptr; }
    } reset;
    Engine eng(g, s);  // setup(): partition, coefficients, views, model init
    shim_hook::g_owner = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const TrainResult res = eng.run();
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (times_out) {
      times_out[0] = std::chrono::duration<double>(t0 - ts).count();  // Engine construction
      times_out[1] = wall;                                             // run(): all epochs
    }
    for (std::size_t e = 0; e < res.epochs.size(); ++e) {
      const EpochMetrics& m = res.epochs[e];
      double* o = epoch_out + e * 10;
      o[0] = m.train_loss;
      o[1] = m.val_acc;
      o[2] = m.test_acc;
      o[3] = static_cast<double>(m.bytes_total);
      o[4] = static_cast<double>(m.msgs_b2);
      o[5] = static_cast<double>(m.msgs_b4);
      o[6] = static_cast<double>(m.msgs_b8);
      o[7] = static_cast<double>(m.msgs_fp);
      o[8] = static_cast<double>(m.plan_version);
      o[9] = wall / static_cast<double>(res.epochs.size());
    }
    if (final_weights) {
      std::size_t o = 0;
      for (const Matrix& w : res.final_weights) {
        std::memcpy(final_weights + o, w.data.data(), w.data.size() * sizeof(double));
        o += w.data.size();
      }
    }
  })
}

// Engine on an explicit graph given as CSR + features/labels/masks (used for
// the bench's CPU baseline on the planted-block sample).
void* ref_dataset_from_arrays(const int64_t* adj_ptr, const int32_t* adj, uint64_t n,
                              const double* features, uint64_t fdim, const int32_t* labels,
                              const uint8_t* train, const uint8_t* val, const uint8_t* test) {
  try {
    auto* d = new RefDataset{graph_from_csr(adj_ptr, adj, n)};
    d->g.features = Matrix(n, fdim);
    std::memcpy(d->g.features.data.data(), features, n * fdim * sizeof(double));
    d->g.labels.assign(labels, labels + n);
    d->g.train_mask.assign(train, train + n);
    d->g.val_mask.assign(val, val + n);
    d->g.test_mask.assign(test, test + n);
    return d;
  } catch (...) {
    map_exc();
    return nullptr;
  }
}

}  // extern "C"
