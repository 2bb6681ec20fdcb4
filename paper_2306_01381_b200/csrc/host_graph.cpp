// host_graph.cpp — partitioning, coefficients, GPU aggregation views and the
// synthetic planted-block graph generator (host setup for the GPU engine).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <numeric>
#include <thread>

#include "host.hpp"
#include "qgnn_b200.h"
#include "rng.cuh"
#include "status.hpp"

namespace qgnn_b200 {

namespace {
template <typename F>
void parallel_for(int64_t n, F&& f, int max_threads = 0) {
  int64_t t = std::max(1u, std::thread::hardware_concurrency());
  if (max_threads > 0) t = std::min<int64_t>(t, max_threads);
  t = std::min<int64_t>(t, std::max<int64_t>(1, n));
  if (t <= 1) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  const int64_t chunk = (n + t - 1) / t;
  for (int64_t w = 0; w < t; ++w)
    th.emplace_back([&, w] {
      for (int64_t i = w * chunk; i < std::min(n, (w + 1) * chunk); ++i) f(i);
    });
  for (auto& x : th) x.join();
}
}  // namespace

// partition.hpp:90-135 — identical claim order, quotas and RNG draws.
std::vector<uint32_t> partition_owner_bfs(const int64_t* ptr, const int32_t* adj, int64_t n,
                                          int64_t n_parts, uint64_t seed) {
  QGNN_REQUIRE(n_parts >= 1 && n_parts <= n, QGNN_EINVAL,
               "partition_graph: n_parts must be in [1, num_nodes]");
  std::vector<uint32_t> owner(n, UINT32_MAX);
  std::vector<int64_t> quota(n_parts, n / n_parts);
  for (int64_t p = 0; p < n % n_parts; ++p) ++quota[p];
  const uint64_t key = rng_fork(rng_seed_key(seed), 0x9a27);
  uint64_t ctr = 0;
  std::vector<std::deque<uint32_t>> frontier(n_parts);
  std::vector<char> rooted(n, 0);
  for (int64_t p = 0; p < n_parts; ++p) {
    uint32_t r = static_cast<uint32_t>(rng_next_below(key, ctr, n));
    while (rooted[r]) r = static_cast<uint32_t>(rng_next_below(key, ctr, n));
    rooted[r] = 1;
    frontier[p].push_back(r);
  }
  std::vector<int64_t> owned(n_parts, 0);
  uint32_t next_unclaimed = 0;
  int64_t assigned = 0;
  while (assigned < n) {
    for (int64_t p = 0; p < n_parts && assigned < n; ++p) {
      if (owned[p] >= quota[p]) continue;
      uint32_t v = UINT32_MAX;
      while (!frontier[p].empty()) {
        const uint32_t c = frontier[p].front();
        frontier[p].pop_front();
        if (owner[c] == UINT32_MAX) {
          v = c;
          break;
        }
      }
      if (v == UINT32_MAX) {
        while (next_unclaimed < n && owner[next_unclaimed] != UINT32_MAX) ++next_unclaimed;
        v = next_unclaimed;
      }
      owner[v] = static_cast<uint32_t>(p);
      ++owned[p];
      ++assigned;
      for (int64_t e = ptr[v]; e < ptr[v + 1]; ++e)
        if (owner[adj[e]] == UINT32_MAX) frontier[p].push_back(static_cast<uint32_t>(adj[e]));
    }
  }
  return owner;
}

// partition.hpp:39-84.  Each node's consumer set (the other partitions owning
// one of its neighbours) is a short ascending list in a CSR, so any P works;
// remote_out[q] of p is filled in ascending node order and remote_in[q] of p
// is q's remote_out[p] (the nodes q owns that p consumes).
std::vector<Part> partitions_from_owner(const int64_t* ptr, const int32_t* adj, int64_t n,
                                        const uint32_t* owner, int64_t n_parts) {
  QGNN_REQUIRE(n_parts >= 1, QGNN_EINVAL, "partitions: n_parts must be positive");
  std::vector<Part> parts(n_parts);
  for (int64_t p = 0; p < n_parts; ++p) {
    parts[p].id = static_cast<uint32_t>(p);
    parts[p].remote_in.resize(n_parts);
    parts[p].remote_out.resize(n_parts);
  }
  for (int64_t v = 0; v < n; ++v) {
    QGNN_REQUIRE(owner[v] < n_parts, QGNN_EINVAL, "owner id out of range");
    parts[owner[v]].owned.push_back(static_cast<uint32_t>(v));
  }
  // consumers of v: distinct owner[u] != owner[v] over v's neighbours
  std::vector<int64_t> cptr(n + 1, 0);
  std::vector<std::vector<uint32_t>> cbuf(std::max<int64_t>(1, std::min<int64_t>(
      n, std::max(1u, std::thread::hardware_concurrency()))));
  const int64_t nb = static_cast<int64_t>(cbuf.size()), chunk = (n + nb - 1) / std::max<int64_t>(1, nb);
  parallel_for(nb, [&](int64_t w) {
    std::vector<uint32_t> tmp;
    for (int64_t v = w * chunk; v < std::min(n, (w + 1) * chunk); ++v) {
      tmp.clear();
      for (int64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
        const uint32_t q = owner[adj[e]];
        if (q != owner[v]) tmp.push_back(q);
      }
      std::sort(tmp.begin(), tmp.end());
      tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
      cptr[v + 1] = static_cast<int64_t>(tmp.size());
      cbuf[w].insert(cbuf[w].end(), tmp.begin(), tmp.end());
    }
  });
  for (int64_t v = 0; v < n; ++v) cptr[v + 1] += cptr[v];
  std::vector<uint32_t> cons(cptr[n]);
  parallel_for(nb, [&](int64_t w) {
    const int64_t v0 = std::min(n, w * chunk);
    if (!cbuf[w].empty()) std::copy(cbuf[w].begin(), cbuf[w].end(), cons.begin() + cptr[v0]);
  });
  parallel_for(n_parts, [&](int64_t p) {
    Part& P = parts[p];
    for (uint32_t v : P.owned) {
      (cptr[v + 1] > cptr[v] ? P.marginal : P.central).push_back(v);
      for (int64_t k = cptr[v]; k < cptr[v + 1]; ++k) P.remote_out[cons[k]].push_back(v);
    }
  });
  parallel_for(n_parts, [&](int64_t p) {
    for (int64_t q = 0; q < n_parts; ++q)
      if (q != p) parts[p].remote_in[q] = parts[q].remote_out[p];
  });
  return parts;
}

// coeffs.hpp:30-45
void compute_coeffs(const int64_t* ptr, const int32_t* adj, int64_t n, bool sage,
                    std::vector<double>& alpha, std::vector<double>& self_alpha) {
  alpha.assign(ptr[n], 0.0);
  self_alpha.assign(n, 0.0);
  parallel_for(n, [&](int64_t v) {
    const double dv1 = static_cast<double>(ptr[v + 1] - ptr[v]) + 1.0;
    self_alpha[v] = 1.0 / dv1;
    for (int64_t e = ptr[v]; e < ptr[v + 1]; ++e) {
      const int64_t u = adj[e];
      const double du1 = static_cast<double>(ptr[u + 1] - ptr[u]) + 1.0;
      alpha[e] = sage ? 1.0 / dv1 : 1.0 / std::sqrt(du1 * dv1);
    }
  });
}

int32_t View::gpu_row(uint32_t node) const {
  auto it = std::lower_bound(owned_sorted.begin(), owned_sorted.end(), node);
  if (it == owned_sorted.end() || *it != node) return -1;
  return owned_gpu_row[it - owned_sorted.begin()];
}

// aggregate.hpp:41-89 in GPU row order (central block then marginal block).
View build_view(const int64_t* ptr, const int32_t* adj, int64_t n, const Part& part,
                int64_t n_parts, const std::vector<double>& alpha,
                const std::vector<double>& self_alpha, bool sage) {
  (void)n;
  View v;
  v.num_owned = static_cast<int64_t>(part.owned.size());
  v.n_central = static_cast<int64_t>(part.central.size());
  v.n_marginal = static_cast<int64_t>(part.marginal.size());
  v.owned_sorted = part.owned;
  v.owned_gpu_row.assign(v.num_owned, -1);
  v.row_node.reserve(v.num_owned);
  for (uint32_t x : part.central) v.row_node.push_back(x);
  for (uint32_t x : part.marginal) v.row_node.push_back(x);
  v.ref_row.assign(v.num_owned, 0);
  v.gpu_row_of_ref.assign(v.num_owned, 0);
  // owned ids ascending == reference row order; central/marginal are sorted subsets
  {
    size_t ic = 0, im = 0;
    for (int64_t r = 0; r < v.num_owned; ++r) {
      const uint32_t node = part.owned[r];
      int32_t g;
      if (ic < part.central.size() && part.central[ic] == node)
        g = static_cast<int32_t>(ic++);
      else
        g = static_cast<int32_t>(v.n_central + static_cast<int64_t>(im++));
      v.owned_gpu_row[r] = g;
      v.ref_row[g] = static_cast<int32_t>(r);
      v.gpu_row_of_ref[r] = g;
    }
  }
  // halo slots: remote_in lists by ascending source (aggregate.hpp:45-56)
  v.device_slot_offset.assign(n_parts + 1, 0);
  for (int64_t q = 0; q < n_parts; ++q) {
    v.device_slot_offset[q] = static_cast<int64_t>(v.slot_node.size());
    for (uint32_t k : part.remote_in[q]) v.slot_node.push_back(k);
  }
  v.device_slot_offset[n_parts] = static_cast<int64_t>(v.slot_node.size());
  v.num_remote = static_cast<int64_t>(v.slot_node.size());
  // slot lookup: (owner q, index in remote_in[q]) via binary search per source list
  auto slot_of = [&](uint32_t node, uint32_t q) -> int32_t {
    const auto& lst = part.remote_in[q];
    auto it = std::lower_bound(lst.begin(), lst.end(), node);
    return static_cast<int32_t>(v.device_slot_offset[q] + (it - lst.begin()));
  };
  // owner lookup for remote neighbours: a node not owned here is in exactly one remote_in list
  std::vector<std::pair<uint32_t, uint32_t>> remote_owner;  // (node, q) sorted by node
  for (int64_t q = 0; q < n_parts; ++q)
    for (uint32_t k : part.remote_in[q]) remote_owner.emplace_back(k, static_cast<uint32_t>(q));
  std::sort(remote_owner.begin(), remote_owner.end());

  v.self_alpha.assign(v.num_owned, 0.0);
  v.local_ptr.assign(v.num_owned + 1, 0);
  v.remote_ptr.assign(v.num_owned + 1, 0);
  for (int64_t g = 0; g < v.num_owned; ++g) {
    const uint32_t node = v.row_node[g];
    v.self_alpha[g] = self_alpha[node];
    for (int64_t e = ptr[node]; e < ptr[node + 1]; ++e) {
      const uint32_t u = static_cast<uint32_t>(adj[e]);
      const int32_t lr = v.gpu_row(u);
      if (lr >= 0) {
        v.local_col.push_back(lr);
        v.local_afwd.push_back(alpha[e]);
        v.local_abwd.push_back(sage ? self_alpha[u] : alpha[e]);  // coeffs.of(g, v, u)
      } else {
        auto it = std::lower_bound(remote_owner.begin(), remote_owner.end(),
                                   std::make_pair(u, uint32_t{0}));
        QGNN_REQUIRE(it != remote_owner.end() && it->first == u, QGNN_EINVAL,
                     "view: remote neighbour missing from remote_in");
        v.remote_slot.push_back(slot_of(u, it->second));
        v.remote_alpha.push_back(alpha[e]);
      }
    }
    v.local_ptr[g + 1] = static_cast<int64_t>(v.local_col.size());
    v.remote_ptr[g + 1] = static_cast<int64_t>(v.remote_slot.size());
  }
  // transpose of the remote CSR, contributions in ascending reference-row order
  v.slot_ptr.assign(v.num_remote + 1, 0);
  for (int32_t s : v.remote_slot) ++v.slot_ptr[s + 1];
  for (int64_t k = 0; k < v.num_remote; ++k) v.slot_ptr[k + 1] += v.slot_ptr[k];
  v.slot_row.assign(v.remote_slot.size(), 0);
  v.slot_alpha.assign(v.remote_slot.size(), 0.0);
  {
    std::vector<int64_t> fill(v.slot_ptr.begin(), v.slot_ptr.end() - 1);
    for (int64_t r = 0; r < v.num_owned; ++r) {  // reference row order
      const int32_t g = v.gpu_row_of_ref[r];
      for (int64_t e = v.remote_ptr[g]; e < v.remote_ptr[g + 1]; ++e) {
        const int32_t s = v.remote_slot[e];
        v.slot_row[fill[s]] = g;
        v.slot_alpha[fill[s]] = v.remote_alpha[e];
        ++fill[s];
      }
    }
  }
  // engine.hpp:262-273: squared consumption weights of incoming messages
  v.rx_alpha_sq.assign(n_parts, {});
  for (int64_t p = 0; p < n_parts; ++p) v.rx_alpha_sq[p].assign(part.remote_in[p].size(), 0.0);
  {
    std::vector<uint32_t> slot_src(v.num_remote);
    for (int64_t q = 0; q < n_parts; ++q)
      for (int64_t k = v.device_slot_offset[q]; k < v.device_slot_offset[q + 1]; ++k)
        slot_src[k] = static_cast<uint32_t>(q);
    for (int64_t r = 0; r < v.num_owned; ++r) {
      const int32_t g = v.gpu_row_of_ref[r];
      for (int64_t e = v.remote_ptr[g]; e < v.remote_ptr[g + 1]; ++e) {
        const int32_t s = v.remote_slot[e];
        const uint32_t src = slot_src[s];
        const double a = v.remote_alpha[e];
        v.rx_alpha_sq[src][s - v.device_slot_offset[src]] += a * a;
      }
    }
  }
  // compulsory source rows of each SpMM call site (SURVEY.md §8d operand-size
  // model): distinct owned rows read by a row range (self rows included) and
  // distinct halo slots read by the marginal rows
  {
    std::vector<uint8_t> seen(v.num_owned, 0);
    auto count = [&](int64_t r0, int64_t r1) {
      std::fill(seen.begin(), seen.end(), 0);
      int64_t c = 0;
      for (int64_t r = r0; r < r1; ++r) {
        if (!seen[r]) seen[r] = 1, ++c;
        for (int64_t e = v.local_ptr[r]; e < v.local_ptr[r + 1]; ++e)
          if (!seen[v.local_col[e]]) seen[v.local_col[e]] = 1, ++c;
      }
      return c;
    };
    v.src_rows_central = count(0, v.n_central);
    v.src_rows_marginal = count(v.n_central, v.num_owned);
    v.src_rows_all = count(0, v.num_owned);
    int64_t used = 0;
    for (int64_t k = 0; k < v.num_remote; ++k) used += v.slot_ptr[k + 1] > v.slot_ptr[k];
    v.src_slots_marginal = used;
  }
  return v;
}


}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" {

int qgnn_partition_graph(const int64_t* adj_ptr, const int32_t* adj, int64_t n, int64_t n_parts,
                         uint64_t seed, uint32_t* owner) {
  QGNN_API_BEGIN
  const auto o = partition_owner_bfs(adj_ptr, adj, n, n_parts, seed);
  std::memcpy(owner, o.data(), o.size() * sizeof(uint32_t));
  QGNN_API_END
}

int qgnn_compute_coeffs(const int64_t* adj_ptr, const int32_t* adj, int64_t n, int sage,
                        double* alpha, double* self_alpha) {
  QGNN_API_BEGIN
  std::vector<double> a, sa;
  compute_coeffs(adj_ptr, adj, n, sage != 0, a, sa);
  std::memcpy(alpha, a.data(), a.size() * sizeof(double));
  std::memcpy(self_alpha, sa.data(), sa.size() * sizeof(double));
  QGNN_API_END
}

// Exchange schedule of one tensor for one rank (plan.hpp:90-154 pair_wire_bytes /
// negotiate_buffers, engine.hpp:460-505 routing).  Sender and receiver derive
// each pair's bytes from their own Part (remote_out vs remote_in), so the
// GPU engine needs no size handshake; tests check the two sides agree.
int qgnn_exchange_plan(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                       const uint32_t* owner, int64_t n_parts, int world, int rank, int64_t dim,
                       int bits, int bwd, int layout, int dtype, uint64_t* send_bytes,
                       uint64_t* recv_bytes) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(world >= 1 && rank >= 0 && rank < world && n_parts % world == 0, QGNN_EINVAL,
               "exchange_plan: n_parts must divide by world, 0 <= rank < world");
  QGNN_REQUIRE(bits == 0 || bits == 2 || bits == 4 || bits == 8, QGNN_EINVAL,
               "exchange_plan: bit width must be 0, 2, 4 or 8");
  const auto parts = partitions_from_owner(adj_ptr, adj, n, owner, n_parts);
  const int64_t ppr = n_parts / world;
  const uint64_t chunk = qgnn_chunk_wire_bytes(uint64_t(dim), bits, layout, dtype);
  for (int r = 0; r < world; ++r) send_bytes[r] = recv_bytes[r] = 0;
  for (int64_t p = rank * ppr; p < (rank + 1) * ppr; ++p)
    for (int64_t q = 0; q < n_parts; ++q) {
      if (q / ppr == rank) continue;  // same GPU: zero copy
      // forward p -> q: rows of p's owned nodes q consumes; backward: partials of
      // the halo slots p holds for q's nodes (engine.hpp:566-588, 661-688)
      const auto& out_ids = bwd ? parts[p].remote_in[q] : parts[p].remote_out[q];
      const auto& in_ids = bwd ? parts[p].remote_out[q] : parts[p].remote_in[q];
      send_bytes[q / ppr] += chunk * out_ids.size();
      recv_bytes[q / ppr] += chunk * in_ids.size();
    }
  QGNN_API_END
}

// Partition statistics for an owner map: per part [owned, central, marginal,
// halo (num_remote), sum_q |remote_out[q]|].  out has 5 * n_parts entries.
int qgnn_partition_stats(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                         const uint32_t* owner, int64_t n_parts, int64_t* out) {
  QGNN_API_BEGIN
  const auto parts = partitions_from_owner(adj_ptr, adj, n, owner, n_parts);
  for (int64_t p = 0; p < n_parts; ++p) {
    int64_t halo = 0, outm = 0;
    for (int64_t q = 0; q < n_parts; ++q) {
      halo += static_cast<int64_t>(parts[p].remote_in[q].size());
      outm += static_cast<int64_t>(parts[p].remote_out[q].size());
    }
    out[5 * p + 0] = static_cast<int64_t>(parts[p].owned.size());
    out[5 * p + 1] = static_cast<int64_t>(parts[p].central.size());
    out[5 * p + 2] = static_cast<int64_t>(parts[p].marginal.size());
    out[5 * p + 3] = halo;
    out[5 * p + 4] = outm;
  }
  QGNN_API_END
}


// ---- partitions_from_owner / DeviceAggView::build / Lookup::bits_for ---------
}  // extern "C"

extern "C" {

int qgnn_partitions_from_owner(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                               const uint32_t* owner, int64_t n_parts, qgnn_partition** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(out, QGNN_EINVAL, "partitions: null output");
  auto parts = partitions_from_owner(adj_ptr, adj, n, owner, n_parts);
  for (int64_t p = 0; p < n_parts; ++p) out[p] = new qgnn_partition{std::move(parts[p])};
  QGNN_API_END
}

int qgnn_partition_destroy(qgnn_partition* part) {
  delete part;
  return QGNN_OK;
}

int qgnn_partition_list(const qgnn_partition* part, int which, int64_t q, const uint32_t** ids,
                        int64_t* len) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(part && ids && len, QGNN_EINVAL, "partition_list: null argument");
  const Part& P = part->part;
  const std::vector<uint32_t>* v = nullptr;
  switch (which) {
    case QGNN_PART_OWNED: v = &P.owned; break;
    case QGNN_PART_CENTRAL: v = &P.central; break;
    case QGNN_PART_MARGINAL: v = &P.marginal; break;
    case QGNN_PART_REMOTE_IN:
    case QGNN_PART_REMOTE_OUT:
      QGNN_REQUIRE(q >= 0 && q < static_cast<int64_t>(P.remote_in.size()), QGNN_EINVAL,
                   "partition_list: device out of range");
      v = which == QGNN_PART_REMOTE_IN ? &P.remote_in[q] : &P.remote_out[q];
      break;
    default:
      QGNN_REQUIRE(false, QGNN_EINVAL, "partition_list: unknown list");
  }
  *ids = v->data();
  *len = static_cast<int64_t>(v->size());
  QGNN_API_END
}

// DeviceAggView::build (aggregate.hpp:41-89) in the reference's row order (owned
// ascending): slots concatenate remote_in by ascending source; per owned row the
// adjacency is split into same-device (local) and cross-device (remote) entries
// in adjacency order; rows with a remote entry are marginal.
int qgnn_agg_view_build(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                        const uint32_t* owner, const qgnn_partition* part, int sage,
                        qgnn_agg_view** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(part && out && owner, QGNN_EINVAL, "agg_view: null argument");
  const Part& P = part->part;
  const uint32_t me = P.id;
  const int64_t n_parts = static_cast<int64_t>(P.remote_in.size());
  std::vector<double> alpha, self_alpha;
  compute_coeffs(adj_ptr, adj, n, sage != 0, alpha, self_alpha);
  auto* V = new qgnn_agg_view;
  V->num_owned = static_cast<int64_t>(P.owned.size());
  V->device_slot_offset.assign(n_parts + 1, 0);
  for (int64_t q = 0; q < n_parts; ++q) {
    V->device_slot_offset[q] = static_cast<int64_t>(V->slot_node.size());
    for (uint32_t k : P.remote_in[q]) {
      V->slot_node.push_back(k);
      V->slot_owner.push_back(static_cast<uint32_t>(q));
    }
  }
  V->device_slot_offset[n_parts] = static_cast<int64_t>(V->slot_node.size());
  V->num_remote = static_cast<int64_t>(V->slot_node.size());
  auto row_of = [&](uint32_t v) {  // owned ascending: binary search
    return static_cast<uint32_t>(std::lower_bound(P.owned.begin(), P.owned.end(), v) - P.owned.begin());
  };
  auto slot_of = [&](uint32_t u) {  // slots of source q are ascending ids
    const uint32_t q = owner[u];
    const auto& in = P.remote_in[q];
    return static_cast<uint32_t>(V->device_slot_offset[q] +
                                 (std::lower_bound(in.begin(), in.end(), u) - in.begin()));
  };
  V->local_ptr.assign(V->num_owned + 1, 0);
  V->remote_ptr.assign(V->num_owned + 1, 0);
  V->self_alpha.resize(V->num_owned);
  for (int64_t i = 0; i < V->num_owned; ++i) {
    const uint32_t v = P.owned[i];
    V->self_alpha[i] = self_alpha[v];
    bool has_remote = false;
    for (int64_t e = adj_ptr[v]; e < adj_ptr[v + 1]; ++e) {
      const uint32_t u = static_cast<uint32_t>(adj[e]);
      if (owner[u] == me) {
        V->local_row.push_back(row_of(u));
        V->local_alpha_fwd.push_back(alpha[e]);
        // coeffs.of(g, v, u): u's adjacency entry for v (graph.hpp sorted lists)
        const int32_t* b = adj + adj_ptr[u];
        const int32_t* f = std::lower_bound(b, adj + adj_ptr[u + 1], static_cast<int32_t>(v));
        V->local_alpha_bwd.push_back(alpha[adj_ptr[u] + (f - b)]);
      } else {
        V->remote_slot.push_back(slot_of(u));
        V->remote_alpha.push_back(alpha[e]);
        has_remote = true;
      }
    }
    V->local_ptr[i + 1] = static_cast<int64_t>(V->local_row.size());
    V->remote_ptr[i + 1] = static_cast<int64_t>(V->remote_slot.size());
    (has_remote ? V->marginal_rows : V->central_rows).push_back(static_cast<uint32_t>(i));
  }
  *out = V;
  QGNN_API_END
}

int qgnn_agg_view_destroy(qgnn_agg_view* view) {
  delete view;
  return QGNN_OK;
}

int qgnn_agg_view_arrays_get(const qgnn_agg_view* v, qgnn_agg_view_arrays* a) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(v && a, QGNN_EINVAL, "agg_view: null argument");
  a->num_owned = v->num_owned;
  a->num_remote = v->num_remote;
  a->local_nnz = static_cast<int64_t>(v->local_row.size());
  a->remote_nnz = static_cast<int64_t>(v->remote_slot.size());
  a->n_parts = static_cast<int64_t>(v->device_slot_offset.size()) - 1;
  a->n_central = static_cast<int64_t>(v->central_rows.size());
  a->n_marginal = static_cast<int64_t>(v->marginal_rows.size());
  a->self_alpha = v->self_alpha.data();
  a->local_ptr = v->local_ptr.data();
  a->local_row = v->local_row.data();
  a->local_alpha_fwd = v->local_alpha_fwd.data();
  a->local_alpha_bwd = v->local_alpha_bwd.data();
  a->remote_ptr = v->remote_ptr.data();
  a->remote_slot = v->remote_slot.data();
  a->remote_alpha = v->remote_alpha.data();
  a->slot_node = v->slot_node.data();
  a->slot_owner = v->slot_owner.data();
  a->device_slot_offset = v->device_slot_offset.data();
  a->central_rows = v->central_rows.data();
  a->marginal_rows = v->marginal_rows.data();
  QGNN_API_END
}

// BitWidthPlan::Lookup::bits_for (plan.hpp:60-72) for one (key, src, dst)
// entry list: ids ascending, bits parallel.  Unknown ids fail like the reference.
int qgnn_plan_bits_for(const uint32_t* ids, const int32_t* bits, int64_t n,
                       const uint32_t* query, int64_t n_query, int32_t* out) {
  QGNN_API_BEGIN
  for (int64_t k = 0; k < n_query; ++k) {
    const uint32_t* it = std::lower_bound(ids, ids + n, query[k]);
    QGNN_REQUIRE(it != ids + n && *it == query[k], QGNN_EINVAL, "plan: unknown message id");
    out[k] = bits[it - ids];
  }
  QGNN_API_END
}

}  // extern "C"
