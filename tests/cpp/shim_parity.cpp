// shim_parity.cpp — the reference-side C++ binding (include/qgnn_b200_shim.hpp)
// compiled against the UNMODIFIED reference headers and checked, function by
// function, against the reference's own implementation on the same inputs.
//
//   shim_parity --host   host-side operators only (no GPU needed)
//   shim_parity --all    plus the device operators (K1/K3/K4/K5 through the C-ABI)
//
// Inputs: the reference's cite generator (cli/synth.hpp:55-149) partitioned by
// its BFS partition_graph (partition.hpp:90-135).  Integer/byte results and the
// fp64 operators must match bit for bit.  Exit status 0 iff every check passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "qgnn/assigner/plan.hpp"
#include "qgnn/cli/synth.hpp"
#include "qgnn/tensorops/model.hpp"
#include "qgnn_b200_shim.hpp"

namespace {
int g_checks = 0, g_fails = 0;
void expect(bool ok, const char* what, int line) {
  ++g_checks;
  if (!ok) {
    ++g_fails;
    std::fprintf(stderr, "FAIL line %d: %s\n", line, what);
  }
}
#define EXPECT(c) expect((c), #c, __LINE__)

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 8) == 0);
}

template <typename F>
std::string thrown(F&& f) {  // exception class of f(), or "" if none
  try {
    f();
  } catch (const qgnn::DecodeError&) {
    return "DecodeError";
  } catch (const qgnn::ProtocolError&) {
    return "ProtocolError";
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::exception&) {
    return "other";
  }
  return "";
}

qgnn::Matrix random_matrix(std::size_t r, std::size_t c, uint64_t seed) {
  qgnn::Matrix m(r, c);
  qgnn::RngStream rng(seed);
  for (double& x : m.data) x = rng.next_gaussian();
  return m;
}

void host_checks(const qgnn::Graph& g, std::size_t n_parts) {
  const auto ref_parts = qgnn::partition_graph(g, n_parts, 7);
  std::vector<uint32_t> owner(g.num_nodes);
  for (const auto& p : ref_parts)
    for (qgnn::NodeId v : p.owned) owner[v] = p.device_id;
  const auto ref_from_owner = qgnn::partitions_from_owner(g, owner, n_parts);
  const auto parts = qgnn::b200::partitions_from_owner(g, owner, n_parts);
  EXPECT(parts.size() == n_parts);
  for (std::size_t p = 0; p < n_parts; ++p) {
    const auto& a = parts[p];
    const auto& b = ref_from_owner[p];
    EXPECT(a.device_id == b.device_id && a.owned == b.owned && a.central == b.central &&
           a.marginal == b.marginal && a.remote_in == b.remote_in && a.remote_out == b.remote_out);
    for (auto mode : {qgnn::AggMode::kGcn, qgnn::AggMode::kSageMean}) {
      const auto rv = qgnn::DeviceAggView::build(g, b, qgnn::compute_coeffs(g, mode));
      const auto v = qgnn::b200::build_view(g, owner, n_parts, static_cast<uint32_t>(p), mode);
      EXPECT(v.num_owned == rv.num_owned && v.num_remote == rv.num_remote);
      EXPECT(same_bits(v.self_alpha, rv.self_alpha));
      EXPECT(v.local_ptr == rv.local_ptr && v.local_row == rv.local_row);
      EXPECT(same_bits(v.local_alpha_fwd, rv.local_alpha_fwd));
      EXPECT(same_bits(v.local_alpha_bwd, rv.local_alpha_bwd));
      EXPECT(v.remote_ptr == rv.remote_ptr && v.remote_slot == rv.remote_slot);
      EXPECT(same_bits(v.remote_alpha, rv.remote_alpha));
      EXPECT(v.slot_node == rv.slot_node && v.slot_owner == rv.slot_owner);
      EXPECT(v.device_slot_offset == rv.device_slot_offset);
      EXPECT(v.central_rows == rv.central_rows && v.marginal_rows == rv.marginal_rows);
      EXPECT(v.row_of_node == rv.row_of_node);
    }
  }
  // Lookup::bits_for over a plan's (key, src, dst) entries (plan.hpp:60-72)
  qgnn::BitWidthPlan plan;
  qgnn::InstancePlan inst;
  qgnn::PlanPair pp{0, 1, {}};
  pp.groups.push_back({{5, 17, 40}, {8, 8, 8}, 0.0, 2});
  pp.groups.push_back({{3, 9}, {8, 8}, 0.0, 8});
  inst.pairs.push_back(pp);
  const qgnn::TensorKey key{1, qgnn::Direction::kForward};
  plan.instances[key] = inst;
  const auto lk = plan.make_lookup();
  const auto& entries = lk.by_pair.at(key).at({0u, 1u});
  for (uint32_t id : {3u, 5u, 9u, 17u, 40u})
    EXPECT(qgnn::b200::bits_for(entries, id) == lk.bits_for(key, 0, 1, id));
  EXPECT(thrown([&] { (void)lk.bits_for(key, 0, 1, 4); }) == "invalid_argument");
  EXPECT(thrown([&] { (void)qgnn::b200::bits_for(entries, 4); }) == "invalid_argument");
}

void device_checks(const qgnn::Graph& g, std::size_t n_parts) {
  const auto ref_parts = qgnn::partition_graph(g, n_parts, 7);
  std::vector<uint32_t> owner(g.num_nodes);
  for (const auto& p : ref_parts)
    for (qgnn::NodeId v : p.owned) owner[v] = p.device_id;
  // ---- encode / decode: one device pair's forward message set (engine.hpp:483-497)
  const auto& part = ref_parts[0];
  const std::size_t dim = g.features.cols;
  std::vector<qgnn::MessageView> msgs;
  for (qgnn::NodeId v : part.remote_out[1]) msgs.push_back({v, g.features.row(v)});
  auto bits_of = [](uint32_t id) { return id % 3 == 0 ? 2 : id % 3 == 1 ? 4 : 8; };
  const qgnn::RngStream rng = qgnn::RngStream(7).fork({0x2, 1, 2, 0, 1});
  const auto ref_set = qgnn::encode_message_set(msgs, bits_of, rng);
  const auto set = qgnn::b200::encode_message_set(msgs, bits_of, rng);
  EXPECT(!msgs.empty());
  EXPECT(set.bytes == ref_set.bytes);
  EXPECT(set.index.total_bytes == ref_set.index.total_bytes);
  EXPECT(set.index.entries.size() == ref_set.index.entries.size());
  for (std::size_t k = 0; k < set.index.entries.size() && k < ref_set.index.entries.size(); ++k) {
    const auto& a = set.index.entries[k];
    const auto& b = ref_set.index.entries[k];
    EXPECT(a.id == b.id && a.bit_width == b.bit_width && a.offset == b.offset && a.dim == b.dim);
  }
  const auto ref_dec = qgnn::decode_message_set(ref_set.bytes, ref_set.index);
  const auto dec = qgnn::b200::decode_message_set(set.bytes, set.index);
  EXPECT(dec.size() == ref_dec.size());
  for (std::size_t k = 0; k < dec.size() && k < ref_dec.size(); ++k)
    EXPECT(dec[k].id == ref_dec[k].id && same_bits(dec[k].values, ref_dec[k].values));
  // error taxonomy (codec.hpp:82-95, quant.hpp:61-68)
  auto bad = set;
  bad.bytes.pop_back();
  EXPECT(thrown([&] { qgnn::decode_message_set(bad.bytes, bad.index); }) == "DecodeError");
  EXPECT(thrown([&] { qgnn::b200::decode_message_set(bad.bytes, bad.index); }) == "DecodeError");
  auto skew = set;
  skew.index.entries[0].bit_width = skew.index.entries[0].bit_width == 8 ? 4 : 8;
  EXPECT(thrown([&] { qgnn::decode_message_set(skew.bytes, skew.index); }) == "DecodeError");
  EXPECT(thrown([&] { qgnn::b200::decode_message_set(skew.bytes, skew.index); }) == "DecodeError");
  std::vector<double> nan_row(dim, 1.0);
  nan_row[dim / 2] = std::nan("");
  const std::vector<qgnn::MessageView> nan_msg{{1, nan_row}};
  auto eight = [](uint32_t) { return 8; };
  EXPECT(thrown([&] { qgnn::encode_message_set(nan_msg, eight, rng); }) == "invalid_argument");
  EXPECT(thrown([&] { qgnn::b200::encode_message_set(nan_msg, eight, rng); }) ==
         "invalid_argument");
  // ---- aggregation (aggregate.hpp:94-165), every device of the partition
  for (std::size_t p = 0; p < n_parts; ++p) {
    const auto coeffs = qgnn::compute_coeffs(g, qgnn::AggMode::kGcn);
    const auto rv = qgnn::DeviceAggView::build(g, ref_parts[p], coeffs);
    const auto v = qgnn::b200::build_view(g, owner, n_parts, static_cast<uint32_t>(p),
                                          qgnn::AggMode::kGcn);
    const std::size_t d = 24;
    const auto h = random_matrix(rv.num_owned, d, 11 + p);
    const auto hr = random_matrix(std::max<std::size_t>(1, rv.num_remote), d, 23 + p);
    for (const auto* rows : {&rv.central_rows, &rv.marginal_rows}) {
      qgnn::Matrix a(rv.num_owned, d), b(rv.num_owned, d);
      qgnn::aggregate_rows(rv, h, hr, *rows, a);
      qgnn::b200::aggregate_rows(v, h, hr, *rows, b);
      EXPECT(same_bits(a.data, b.data));
    }
    std::vector<uint32_t> all(rv.num_owned);
    for (std::size_t i = 0; i < all.size(); ++i) all[i] = static_cast<uint32_t>(i);
    qgnn::Matrix a(rv.num_owned, d), b(rv.num_owned, d);
    qgnn::aggregate_backward_local(rv, h, all, a);
    qgnn::b200::aggregate_backward_local(v, h, all, b);
    EXPECT(same_bits(a.data, b.data));
    EXPECT(same_bits(qgnn::backward_remote_partials(rv, h).data,
                     qgnn::b200::backward_remote_partials(v, h).data));
  }
  // ---- dense transform (model.hpp:90-170, matrix.hpp:51-65)
  const std::size_t n = 300, din = 40, dout = 24;
  const auto hagg = random_matrix(n, din, 5);
  const auto w = random_matrix(din, dout, 6);
  std::vector<uint32_t> rows;
  for (uint32_t r = 0; r < n; r += 2) rows.push_back(r);
  for (bool relu : {true, false}) {
    qgnn::GnnLayer layer;
    layer.weight = w;
    layer.act = relu ? qgnn::Activation::kRelu : qgnn::Activation::kNone;
    qgnn::GnnModel model;
    qgnn::LayerCache cache;
    cache.h_agg = hagg;
    cache.pre_act = qgnn::Matrix(n, dout);
    qgnn::Matrix a(n, dout), b(n, dout);
    qgnn::layer_forward_rows(layer, model, cache, rows, a, qgnn::RngStream(1));
    qgnn::b200::layer_forward_rows(hagg, w, relu, rows, b);
    EXPECT(same_bits(a.data, b.data));
  }
  qgnn::GnnLayer layer;
  layer.weight = w;
  const auto dz = random_matrix(n, dout, 8);
  qgnn::Matrix a(n, din), b(n, din);
  qgnn::input_grad_rows(layer, dz, rows, a);
  qgnn::b200::input_grad_rows(dz, w, rows, b);
  EXPECT(same_bits(a.data, b.data));
  EXPECT(same_bits(qgnn::matmul_transa(hagg, dz).data, qgnn::b200::matmul_transa(hagg, dz).data));
}
}  // namespace

int main(int argc, char** argv) {
  const bool all = argc > 1 && std::string(argv[1]) == "--all";
  qgnn::DatasetSpec spec;
  spec.kind = qgnn::SynthKind::kCite;
  spec.nodes = 3000;
  spec.classes = 8;
  spec.feature_dim = 48;
  spec.attach_edges = 6;
  spec.seed = 3;
  const qgnn::Graph g = qgnn::generate_dataset(spec);
  for (std::size_t parts : {2u, 5u}) {
    host_checks(g, parts);
    if (all) device_checks(g, parts);
  }
  std::printf("shim_parity %s: %d checks, %d failed\n", all ? "--all" : "--host", g_checks,
              g_fails);
  return g_fails == 0 ? 0 : 1;
}
