// qgnn_b200_shim.hpp — reference-side binding of libqgnn_b200 (C++20).
//
// A maintainer drops this header into the reference tree (it includes the
// reference's own headers, proj/include/qgnn/...) and links
// -lqgnn_b200 -lcudart.  Every function keeps the reference operator's name,
// signature, ownership (value types returned, caller's `out` written) and
// exception types, while the work runs on the GPU through the C-ABI in
// qgnn_b200.h:
//
//   encode_message_set / decode_message_set   codec.hpp:41-96   (K1 / K3, fp64, 25-byte wire)
//   partitions_from_owner                     partition.hpp:39-84
//   build_view  (DeviceAggView::build)        aggregate.hpp:41-89
//   aggregate_rows / aggregate_backward_local / backward_remote_partials   aggregate.hpp:94-165
//   layer_forward_rows (ReLU / linear) / input_grad_rows / matmul_transa   model.hpp:90-170,
//                                                                          matrix.hpp:51-65
//   Lookup::bits_for                          plan.hpp:60-72
//
// tests/cpp/shim_parity.cpp compiles this header against the unmodified
// reference headers and checks every function against the reference itself.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "qgnn/common/errors.hpp"
#include "qgnn/graphcore/coeffs.hpp"
#include "qgnn/graphcore/partition.hpp"
#include "qgnn/quantcodec/codec.hpp"
#include "qgnn/quantcodec/rng.hpp"
#include "qgnn/tensorops/aggregate.hpp"
#include "qgnn/tensorops/matrix.hpp"
#include "qgnn_b200.h"

namespace qgnn::b200 {

// status -> the reference's exception taxonomy (common/errors.hpp:8-36)
inline void check(int st) {
  if (st == QGNN_OK) return;
  const std::string m = qgnn_last_error();
  switch (st) {
    case QGNN_EDECODE: throw DecodeError(m);
    case QGNN_EPROTOCOL: throw ProtocolError(m);
    case QGNN_ERESOURCE: throw ResourceLimitError(m);
    case QGNN_EDIVERGED: throw DivergedError(m);
    case QGNN_EIO: throw IoError(m);
    case QGNN_EINVAL: throw std::invalid_argument(m);
    default: throw std::runtime_error(m);
  }
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) throw std::runtime_error(cudaGetErrorString(e));
}

// One context (error word + scratch) per thread, on the current device.
inline qgnn_ctx* ctx() {
  struct Holder {
    qgnn_ctx* h = nullptr;
    Holder() {
      int dev = 0;
      cuda_check(cudaGetDevice(&dev));
      check(qgnn_ctx_create(dev, &h));
    }
    ~Holder() { qgnn_ctx_destroy(h); }
  };
  thread_local Holder holder;
  return holder.h;
}

// Device copy of a host vector; freed on scope exit.
template <typename T>
struct Dev {
  T* p = nullptr;
  std::size_t n = 0;
  explicit Dev(std::size_t count) : n(count) {
    cuda_check(cudaMalloc(&p, std::max<std::size_t>(1, n) * sizeof(T)));
    cuda_check(cudaMemset(p, 0, std::max<std::size_t>(1, n) * sizeof(T)));
  }
  template <typename U>
  explicit Dev(const std::vector<U>& v) : Dev(v.size()) {
    static_assert(sizeof(U) == sizeof(T));
    if (n) cuda_check(cudaMemcpy(p, v.data(), n * sizeof(T), cudaMemcpyHostToDevice));
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() { cudaFree(p); }
  template <typename U>
  std::vector<U> host() const {
    std::vector<U> v(n * sizeof(T) / sizeof(U));
    if (n) cuda_check(cudaMemcpy(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
    return v;
  }
};

// ---- RngStream -> C-ABI key --------------------------------------------------
// RngStream keeps its key private; its first draw is mix(key + phi) (rng.hpp:30)
// and mix (rng.hpp:52-57) is a bijection, so the key is recovered by inverting
// the finalizer: key = unmix(draw) - phi.  The C-ABI forks from that key
// exactly like RngStream::fork (rng.hpp:17-22).
namespace detail {
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;
constexpr uint64_t inv_odd(uint64_t a) {  // a^-1 mod 2^64 (Newton)
  uint64_t x = a;
  for (int i = 0; i < 6; ++i) x *= 2 - a * x;
  return x;
}
constexpr uint64_t unxorshift(uint64_t y, int s) {
  uint64_t x = y;
  for (int k = s; k < 64; k += s) x = y ^ (x >> s);
  return x;
}
constexpr uint64_t unmix(uint64_t z) {
  z = unxorshift(z, 31);
  z *= inv_odd(0x94d049bb133111ebull);
  z = unxorshift(z, 27);
  z *= inv_odd(0xbf58476d1ce4e5b9ull);
  z = unxorshift(z, 30);
  return z - kPhi;  // mix adds phi first
}
}  // namespace detail

// Key of a stream whose counter is 0 (every RngStream returned by fork()).
inline uint64_t stream_key(const RngStream& rng) {
  RngStream copy = rng;
  return detail::unmix(copy.next_u64()) - detail::kPhi;
}

// ---- codec.hpp:41-72 ----------------------------------------------------------
inline EncodedSet encode_message_set(std::span<const MessageView> messages,
                                     const std::function<int(uint32_t)>& bits_of,
                                     const RngStream& rng) {
  const std::size_t n = messages.size();
  const std::size_t dim = n ? messages[0].values.size() : 0;
  std::vector<int32_t> bits(n), rows(n);
  std::vector<uint32_t> ids(n);
  std::vector<double> vals(n * dim);
  for (std::size_t i = 0; i < n; ++i) {
    bits[i] = bits_of(messages[i].id);
    if (bits[i] != 2 && bits[i] != 4 && bits[i] != 8)
      throw std::invalid_argument("encode_message_set: bit width must be 2, 4, or 8");
    if (messages[i].values.size() != dim)
      throw std::invalid_argument("encode_message_set: messages must share one dimension");
    ids[i] = messages[i].id;
    rows[i] = static_cast<int32_t>(i);
    std::memcpy(vals.data() + i * dim, messages[i].values.data(), dim * sizeof(double));
  }
  std::vector<uint32_t> sorted = ids;
  std::sort(sorted.begin(), sorted.end());
  if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
    throw std::invalid_argument("encode_message_set: duplicate message ids");
  EncodedSet set;
  if (n == 0) return set;
  std::vector<int64_t> pos(n);
  std::vector<uint64_t> off(n);
  uint64_t total = 0;
  check(qgnn_wire_layout(bits.data(), static_cast<int64_t>(n), static_cast<int64_t>(dim),
                         QGNN_WIRE_REF, QGNN_F64, pos.data(), off.data(), &total));
  std::vector<uint8_t> bits8(bits.begin(), bits.end());
  const std::vector<uint64_t> key{stream_key(rng)};
  Dev<double> d_vals(vals);
  Dev<int32_t> d_rows(rows);
  Dev<uint32_t> d_ids(ids);
  Dev<uint8_t> d_bits(bits8);
  Dev<uint64_t> d_off(off), d_key(key);
  Dev<uint8_t> d_out(total);
  check(qgnn_quantize_pack(ctx(), d_vals.p, QGNN_F64, static_cast<int64_t>(dim),
                           static_cast<int64_t>(dim), static_cast<int64_t>(n), d_rows.p, d_ids.p,
                           d_bits.p, d_off.p, nullptr, d_key.p, QGNN_WIRE_REF, d_out.p, nullptr,
                           nullptr, 0, nullptr));
  check(qgnn_ctx_check(ctx(), nullptr));  // non-finite input -> std::invalid_argument
  set.bytes = d_out.host<uint8_t>();
  set.index.total_bytes = total;
  for (std::size_t k = 0; k < n; ++k) {
    const std::size_t i = static_cast<std::size_t>(pos[k]);
    set.index.entries.push_back({ids[i], static_cast<uint8_t>(bits[i]), off[i], dim});
  }
  return set;
}

// ---- codec.hpp:80-96 ----------------------------------------------------------
inline std::vector<DecodedMessage> decode_message_set(std::span<const uint8_t> bytes,
                                                      const RetrievalIndex& index) {
  const std::size_t n = index.entries.size();
  std::vector<uint8_t> bits(n);
  std::vector<uint64_t> off(n), dims(n);
  for (std::size_t k = 0; k < n; ++k) {
    bits[k] = index.entries[k].bit_width;
    off[k] = index.entries[k].offset;
    dims[k] = index.entries[k].dim;
  }
  check(qgnn_decode_validate(bits.data(), off.data(), dims.data(), static_cast<int64_t>(n),
                             QGNN_WIRE_REF, QGNN_F64, index.total_bytes, bytes.size()));
  std::vector<DecodedMessage> out;
  out.reserve(n);
  if (n == 0) return out;
  // the kernel decodes one dimension per launch: group entries by dim
  std::vector<std::vector<double>> vals(n);
  std::vector<uint64_t> seen;
  for (std::size_t k = 0; k < n; ++k)
    if (std::find(seen.begin(), seen.end(), dims[k]) == seen.end()) seen.push_back(dims[k]);
  Dev<uint8_t> d_in(std::vector<uint8_t>(bytes.begin(), bytes.end()));
  for (uint64_t d : seen) {
    std::vector<uint8_t> b;
    std::vector<uint64_t> o;
    std::vector<std::size_t> which;
    for (std::size_t k = 0; k < n; ++k)
      if (dims[k] == d) {
        b.push_back(bits[k]);
        o.push_back(off[k]);
        which.push_back(k);
      }
    Dev<uint8_t> d_b(b);
    Dev<uint64_t> d_o(o);
    Dev<double> d_out(which.size() * d);
    check(qgnn_dequant_scatter(ctx(), d_in.p, static_cast<int64_t>(which.size()),
                               static_cast<int64_t>(d), d_b.p, d_o.p, QGNN_WIRE_REF, nullptr, 0,
                               d_out.p, QGNN_F64, static_cast<int64_t>(d), nullptr, nullptr));
    check(qgnn_ctx_check(ctx(), nullptr));  // chunk vs index -> DecodeError
    const std::vector<double> h = d_out.host<double>();
    for (std::size_t i = 0; i < which.size(); ++i)
      vals[which[i]].assign(h.begin() + i * d, h.begin() + (i + 1) * d);
  }
  for (std::size_t k = 0; k < n; ++k) out.push_back({index.entries[k].id, std::move(vals[k])});
  return out;
}

// ---- partition.hpp:39-84 -------------------------------------------------------
inline std::vector<int64_t> ptr64(const Graph& g) {
  return std::vector<int64_t>(g.adj_ptr.begin(), g.adj_ptr.end());
}
inline std::vector<int32_t> adj32(const Graph& g) {
  return std::vector<int32_t>(g.adj.begin(), g.adj.end());
}

inline std::vector<Partition> partitions_from_owner(const Graph& g,
                                                    const std::vector<uint32_t>& owner,
                                                    std::size_t n_parts) {
  if (owner.size() != g.num_nodes) throw std::invalid_argument("owner size mismatch");
  const auto ptr = ptr64(g);
  const auto adj = adj32(g);
  std::vector<qgnn_partition*> hs(n_parts, nullptr);
  check(qgnn_partitions_from_owner(ptr.data(), adj.data(), static_cast<int64_t>(g.num_nodes),
                                   owner.data(), static_cast<int64_t>(n_parts), hs.data()));
  auto list = [](const qgnn_partition* h, int which, int64_t q) {
    const uint32_t* ids = nullptr;
    int64_t len = 0;
    check(qgnn_partition_list(h, which, q, &ids, &len));
    return std::vector<NodeId>(ids, ids + len);
  };
  std::vector<Partition> parts(n_parts);
  for (std::size_t p = 0; p < n_parts; ++p) {
    parts[p].device_id = static_cast<uint32_t>(p);
    parts[p].owned = list(hs[p], QGNN_PART_OWNED, 0);
    parts[p].central = list(hs[p], QGNN_PART_CENTRAL, 0);
    parts[p].marginal = list(hs[p], QGNN_PART_MARGINAL, 0);
    for (std::size_t q = 0; q < n_parts; ++q) {
      parts[p].remote_in.push_back(list(hs[p], QGNN_PART_REMOTE_IN, static_cast<int64_t>(q)));
      parts[p].remote_out.push_back(list(hs[p], QGNN_PART_REMOTE_OUT, static_cast<int64_t>(q)));
    }
  }
  for (auto* h : hs) qgnn_partition_destroy(h);
  return parts;
}

// ---- aggregate.hpp:41-89 -------------------------------------------------------
inline DeviceAggView build_view(const Graph& g, const std::vector<uint32_t>& owner,
                                std::size_t n_parts, uint32_t device, AggMode mode) {
  const auto ptr = ptr64(g);
  const auto adj = adj32(g);
  std::vector<qgnn_partition*> hs(n_parts, nullptr);
  check(qgnn_partitions_from_owner(ptr.data(), adj.data(), static_cast<int64_t>(g.num_nodes),
                                   owner.data(), static_cast<int64_t>(n_parts), hs.data()));
  qgnn_agg_view* vh = nullptr;
  const int st = qgnn_agg_view_build(ptr.data(), adj.data(), static_cast<int64_t>(g.num_nodes),
                                     owner.data(), hs[device], mode == AggMode::kSageMean, &vh);
  for (auto* h : hs) qgnn_partition_destroy(h);
  check(st);
  qgnn_agg_view_arrays a{};
  check(qgnn_agg_view_arrays_get(vh, &a));
  DeviceAggView v;
  v.num_owned = static_cast<std::size_t>(a.num_owned);
  v.num_remote = static_cast<std::size_t>(a.num_remote);
  v.self_alpha.assign(a.self_alpha, a.self_alpha + a.num_owned);
  v.local_ptr.assign(a.local_ptr, a.local_ptr + a.num_owned + 1);
  v.local_row.assign(a.local_row, a.local_row + a.local_nnz);
  v.local_alpha_fwd.assign(a.local_alpha_fwd, a.local_alpha_fwd + a.local_nnz);
  v.local_alpha_bwd.assign(a.local_alpha_bwd, a.local_alpha_bwd + a.local_nnz);
  v.remote_ptr.assign(a.remote_ptr, a.remote_ptr + a.num_owned + 1);
  v.remote_slot.assign(a.remote_slot, a.remote_slot + a.remote_nnz);
  v.remote_alpha.assign(a.remote_alpha, a.remote_alpha + a.remote_nnz);
  v.slot_node.assign(a.slot_node, a.slot_node + a.num_remote);
  v.slot_owner.assign(a.slot_owner, a.slot_owner + a.num_remote);
  v.device_slot_offset.assign(a.device_slot_offset, a.device_slot_offset + a.n_parts + 1);
  v.central_rows.assign(a.central_rows, a.central_rows + a.n_central);
  v.marginal_rows.assign(a.marginal_rows, a.marginal_rows + a.n_marginal);
  qgnn_agg_view_destroy(vh);
  std::vector<NodeId> owned;
  for (NodeId u = 0; u < g.num_nodes; ++u)
    if (owner[u] == device) owned.push_back(u);
  for (std::size_t i = 0; i < owned.size(); ++i) v.row_of_node[owned[i]] = static_cast<uint32_t>(i);
  return v;
}

// ---- aggregate.hpp:94-165 (fp64: the reference's summation order, bit for bit) -----------
namespace detail {
inline void csr_rows(const DeviceAggView& v, const Matrix& x, const Matrix* y, bool self,
                     const std::vector<int64_t>& pa, const std::vector<int32_t>& ca,
                     const std::vector<double>& aa, const std::vector<int64_t>* pb,
                     const std::vector<int32_t>* cb, const std::vector<double>* ab,
                     std::span<const uint32_t> rows, Matrix& out) {
  Dev<double> d_x(x.data), d_sa(self ? v.self_alpha : std::vector<double>{});
  Dev<int64_t> d_pa(pa);
  Dev<int32_t> d_ca(ca);
  Dev<double> d_aa(aa);
  Dev<double> d_y(y ? y->data : std::vector<double>{});
  Dev<int64_t> d_pb(pb ? *pb : std::vector<int64_t>{});
  Dev<int32_t> d_cb(cb ? *cb : std::vector<int32_t>{});
  Dev<double> d_ab(ab ? *ab : std::vector<double>{});
  std::vector<int32_t> r32(rows.begin(), rows.end());
  Dev<int32_t> d_rows(r32);
  Dev<double> d_out(out.data);
  check(qgnn_csr_aggregate(ctx(), QGNN_F64, static_cast<int64_t>(x.cols), d_x.p,
                           static_cast<int64_t>(x.cols), y ? d_y.p : nullptr,
                           static_cast<int64_t>(y ? y->cols : 0), self ? d_sa.p : nullptr,
                           d_pa.p, d_ca.p, d_aa.p, pb ? d_pb.p : nullptr, cb ? d_cb.p : nullptr,
                           ab ? d_ab.p : nullptr, d_rows.p, 0, static_cast<int64_t>(r32.size()),
                           d_out.p, static_cast<int64_t>(out.cols), nullptr));
  out.data = d_out.host<double>();
}
inline std::vector<int64_t> to64(const std::vector<std::size_t>& v) {
  return std::vector<int64_t>(v.begin(), v.end());
}
inline std::vector<int32_t> to32(const std::vector<uint32_t>& v) {
  return std::vector<int32_t>(v.begin(), v.end());
}
}  // namespace detail

inline void aggregate_rows(const DeviceAggView& v, const Matrix& h_owned, const Matrix& h_remote,
                           std::span<const uint32_t> rows, Matrix& out) {
  check_shape(h_owned.rows == v.num_owned && out.rows == v.num_owned &&
                  out.cols == h_owned.cols && (v.num_remote == 0 || h_remote.cols == h_owned.cols),
              "aggregate_rows");
  const auto rp = detail::to64(v.remote_ptr);
  const auto rs = detail::to32(v.remote_slot);
  detail::csr_rows(v, h_owned, v.num_remote ? &h_remote : nullptr, true, detail::to64(v.local_ptr),
                   detail::to32(v.local_row), v.local_alpha_fwd, &rp, &rs, &v.remote_alpha, rows,
                   out);
}

inline void aggregate_backward_local(const DeviceAggView& v, const Matrix& gbar,
                                     std::span<const uint32_t> rows, Matrix& out) {
  check_shape(gbar.rows == v.num_owned && out.rows == v.num_owned && out.cols == gbar.cols,
              "aggregate_backward_local");
  detail::csr_rows(v, gbar, nullptr, true, detail::to64(v.local_ptr), detail::to32(v.local_row),
                   v.local_alpha_bwd, nullptr, nullptr, nullptr, rows, out);
}

// partials[slot] += alpha * gbar[r] over marginal rows ascending (aggregate.hpp:152-165):
// gathered per slot through the transpose of the remote CSR, same order.
inline Matrix backward_remote_partials(const DeviceAggView& v, const Matrix& gbar) {
  check_shape(gbar.rows == v.num_owned, "backward_remote_partials");
  std::vector<int64_t> tp(v.num_remote + 1, 0);
  for (uint32_t s : v.remote_slot) ++tp[s + 1];
  for (std::size_t s = 0; s < v.num_remote; ++s) tp[s + 1] += tp[s];
  std::vector<int32_t> tr(v.remote_slot.size());
  std::vector<double> ta(v.remote_slot.size());
  std::vector<int64_t> fill(tp.begin(), tp.end() - 1);
  for (uint32_t r : v.marginal_rows)
    for (std::size_t e = v.remote_ptr[r]; e < v.remote_ptr[r + 1]; ++e) {
      const int64_t k = fill[v.remote_slot[e]]++;
      tr[k] = static_cast<int32_t>(r);
      ta[k] = v.remote_alpha[e];
    }
  Matrix out(v.num_remote, gbar.cols);
  if (v.num_remote == 0) return out;
  std::vector<uint32_t> slots(v.num_remote);
  for (std::size_t s = 0; s < v.num_remote; ++s) slots[s] = static_cast<uint32_t>(s);
  detail::csr_rows(v, gbar, nullptr, false, tp, tr, ta, nullptr, nullptr, nullptr, slots, out);
  return out;
}

// ---- model.hpp:90-170, matrix.hpp:51-65 (no layer norm / dropout) --------------
inline void layer_forward_rows(const Matrix& h_agg, const Matrix& w, bool relu,
                               std::span<const uint32_t> rows, Matrix& out) {
  check_shape(h_agg.cols == w.rows && out.cols == w.cols && out.rows == h_agg.rows,
              "layer_forward");
  std::vector<int32_t> r32(rows.begin(), rows.end());
  Dev<double> d_a(h_agg.data), d_w(w.data), d_out(out.data);
  Dev<int32_t> d_rows(r32);
  check(qgnn_dense_forward(ctx(), QGNN_F64, d_a.p, static_cast<int64_t>(h_agg.cols), d_w.p,
                           static_cast<int64_t>(w.rows), static_cast<int64_t>(w.cols), d_rows.p, 0,
                           static_cast<int64_t>(r32.size()), relu ? 1 : 0, d_out.p,
                           static_cast<int64_t>(out.cols), nullptr));
  out.data = d_out.host<double>();
}

inline void input_grad_rows(const Matrix& dz, const Matrix& w, std::span<const uint32_t> rows,
                            Matrix& dh_agg) {
  check_shape(dz.cols == w.cols && dh_agg.cols == w.rows, "input_grad");
  std::vector<int32_t> r32(rows.begin(), rows.end());
  Dev<double> d_dz(dz.data), d_w(w.data), d_out(dh_agg.data);
  Dev<int32_t> d_rows(r32);
  check(qgnn_dense_input_grad(ctx(), QGNN_F64, d_dz.p, static_cast<int64_t>(dz.cols), d_w.p,
                              static_cast<int64_t>(w.rows), static_cast<int64_t>(w.cols), d_rows.p,
                              0, static_cast<int64_t>(r32.size()), d_out.p,
                              static_cast<int64_t>(dh_agg.cols), nullptr));
  dh_agg.data = d_out.host<double>();
}

inline Matrix matmul_transa(const Matrix& a, const Matrix& b) {
  check_shape(a.rows == b.rows, "matmul_transa");
  Matrix out(a.cols, b.cols);
  Dev<double> d_a(a.data), d_b(b.data), d_out(out.data);
  check(qgnn_dense_weight_grad(ctx(), QGNN_F64, d_a.p, static_cast<int64_t>(a.cols), d_b.p,
                               static_cast<int64_t>(b.cols), static_cast<int64_t>(a.cols),
                               static_cast<int64_t>(b.cols), nullptr, 0,
                               static_cast<int64_t>(a.rows), 0, d_out.p, nullptr));
  out.data = d_out.host<double>();
  return out;
}

// ---- plan.hpp:60-72: one (key, src, dst) list of a Lookup, ids ascending ----------
inline int bits_for(const std::vector<std::tuple<uint32_t, int, uint64_t>>& entries, uint32_t id) {
  std::vector<uint32_t> ids;
  std::vector<int32_t> bits;
  for (const auto& t : entries) {
    ids.push_back(std::get<0>(t));
    bits.push_back(std::get<1>(t));
  }
  int32_t out = 0;
  check(qgnn_plan_bits_for(ids.data(), bits.data(), static_cast<int64_t>(ids.size()), &id, 1, &out));
  return out;
}

}  // namespace qgnn::b200
