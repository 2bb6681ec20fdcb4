// planted.cpp — synthetic planted-block power-law graphs for the benchmark
// configurations.  Input generation only: it is
// shared by both bench arms (the GPU engine and the reference CPU engine) so
// that they see byte-identical graphs, and it is neither product kernel code
// nor oracle code.  Built into synth/_build/libqgnn_synth.so by synth/Makefile.
//
// The RNG is the reference's splitmix chain (quantcodec/rng.hpp:13-61), so
// every draw is a pure function of (key, counter) and the graph does not
// depend on the thread count.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

namespace {
constexpr uint64_t kPhi = 0x9e3779b97f4a7c15ull;
inline uint64_t rng_mix(uint64_t z) {
  z += kPhi;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
inline uint64_t rng_seed_key(uint64_t seed) { return rng_mix(seed ^ 0x6a09e667f3bcc909ull); }
inline uint64_t rng_fork(uint64_t key, uint64_t coord) { return rng_mix(key ^ rng_mix(coord + kPhi)); }
inline uint64_t rng_u64(uint64_t key, uint64_t ctr) { return rng_mix(key + ctr * kPhi); }
inline uint64_t rng_u53(uint64_t key, uint64_t ctr) { return rng_u64(key, ctr) >> 11; }

template <typename F>
void parallel_for(int64_t n, F&& f) {
  int64_t t = std::max(1u, std::thread::hardware_concurrency());
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

// ---------------------------------------------------------------------------
// Planted-block power-law generator.
//
// Nodes are split into `blocks` contiguous id ranges (the planted partition:
// owner = block).  Node u emits k_u undirected edges with k_u drawn from a
// discrete Pareto law (mean avg_degree/2, exponent `gamma`).  A fraction
// `cross_frac` of them lands in another block on a node picked with
// probability proportional to its own Pareto weight (hubs attract cut edges,
// as in real co-purchase/social graphs); the rest stay in the block at a
// log-uniform id distance (community locality as left by a locality-
// preserving node order such as METIS/RCM).  Pairs are de-duplicated, self
// loops dropped and the count is trimmed/topped up to exactly n_edges.
// Labels follow 256-node communities; features are sep*mu_class + N(0,1)
// (synth.hpp:112-124 recipe) drawn from per-node RngStream forks.
// ---------------------------------------------------------------------------
struct PlantedSpec {
  int64_t nodes, n_edges, feat, classes, blocks;
  double cross_frac, gamma, sep;
  uint64_t seed;
};

static double u01(uint64_t key, uint64_t ctr) {
  return static_cast<double>(rng_u53(key, ctr)) * 0x1.0p-53;
}

static void gen_planted(const PlantedSpec& s, int64_t* adj_ptr, int32_t* adj, float* features,
                        int32_t* labels, uint8_t* train, uint8_t* val, uint8_t* test) {
  const int64_t n = s.nodes;
  const int64_t bsz = (n + s.blocks - 1) / s.blocks;
  const uint64_t root = rng_seed_key(s.seed);
  // Pareto weights w_u >= 1, tail exponent gamma; k_u ~ w_u * scale
  std::vector<double> w(n);
  const uint64_t kw = rng_fork(root, 0x61);
  parallel_for(n, [&](int64_t u) {
    const double x = u01(kw, static_cast<uint64_t>(u) + 1);
    w[u] = std::pow(1.0 - x, -1.0 / (s.gamma - 1.0));
  });
  // cumulative weights per block for preferential cross targets
  std::vector<double> cum(n + 1, 0.0);
  for (int64_t u = 0; u < n; ++u) cum[u + 1] = cum[u] + w[u];
  const double wsum = cum[n];
  const double target_pairs = static_cast<double>(s.n_edges) * 1.03;
  const double scale = target_pairs / wsum;

  const int nt = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
  std::vector<std::vector<uint64_t>> buckets(nt);
  const uint64_t ke = rng_fork(root, 0x62);
  {
    std::vector<std::thread> th;
    const int64_t chunk = (n + nt - 1) / nt;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        auto& out = buckets[t];
        for (int64_t u = t * chunk; u < std::min(n, (t + 1) * chunk); ++u) {
          const uint64_t k = rng_fork(ke, static_cast<uint64_t>(u));
          uint64_t c = 0;
          const double lam = w[u] * scale;
          int64_t ku = static_cast<int64_t>(lam);
          if (u01(k, ++c) < lam - static_cast<double>(ku)) ++ku;
          const int64_t b = u / bsz;
          const int64_t b0 = b * bsz, b1 = std::min(n, b0 + bsz);
          for (int64_t e = 0; e < ku; ++e) {
            int64_t v;
            if (s.blocks > 1 && u01(k, ++c) < s.cross_frac) {
              // other block, preferential by weight
              int64_t ob = static_cast<int64_t>(u01(k, ++c) * (s.blocks - 1));
              if (ob >= b) ++ob;
              const int64_t o0 = ob * bsz, o1 = std::min(n, o0 + bsz);
              const double t2 = cum[o0] + u01(k, ++c) * (cum[o1] - cum[o0]);
              v = std::upper_bound(cum.begin() + o0, cum.begin() + o1 + 1, t2) - cum.begin() - 1;
              v = std::clamp<int64_t>(v, o0, o1 - 1);
            } else {
              const double span = static_cast<double>(b1 - b0);
              const double dist = std::floor(std::exp(u01(k, ++c) * std::log(span)));
              const int64_t d = static_cast<int64_t>(dist);
              v = u01(k, ++c) < 0.5 ? u + d : u - d;
              const int64_t len = b1 - b0;
              v = b0 + (((v - b0) % len) + len) % len;
            }
            if (v == u) continue;
            const uint64_t a = static_cast<uint64_t>(std::min(u, v)),
                           bb = static_cast<uint64_t>(std::max(u, v));
            out.push_back(a << 32 | bb);
          }
        }
      });
    for (auto& x : th) x.join();
  }
  // global radix by high node id range, sort + unique per range
  std::vector<std::vector<uint64_t>> ranges(nt);
  const int64_t rchunk = (n + nt - 1) / nt;
  {
    std::vector<std::vector<size_t>> counts(nt, std::vector<size_t>(nt, 0));
    for (int t = 0; t < nt; ++t)
      for (uint64_t x : buckets[t]) ++counts[t][static_cast<int64_t>(x >> 32) / rchunk];
    for (int r = 0; r < nt; ++r) {
      size_t tot = 0;
      for (int t = 0; t < nt; ++t) tot += counts[t][r];
      ranges[r].reserve(tot);
    }
    for (int t = 0; t < nt; ++t) {
      for (uint64_t x : buckets[t]) ranges[static_cast<int64_t>(x >> 32) / rchunk].push_back(x);
      std::vector<uint64_t>().swap(buckets[t]);
    }
  }
  parallel_for(nt, [&](int64_t r) {
    auto& v = ranges[r];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  });
  std::vector<uint64_t> pairs;
  {
    size_t tot = 0;
    for (auto& r : ranges) tot += r.size();
    pairs.reserve(tot);
    for (auto& r : ranges) {
      pairs.insert(pairs.end(), r.begin(), r.end());
      std::vector<uint64_t>().swap(r);
    }
  }
  // exact edge count: drop a deterministic random subset, or top up with
  // extra local edges (rare; the 3% overshoot normally covers duplicates)
  const int64_t want = s.n_edges;
  if (static_cast<int64_t>(pairs.size()) > want) {
    const uint64_t kd = rng_fork(root, 0x63);
    std::vector<std::pair<uint64_t, uint64_t>> keyed(pairs.size());
    parallel_for(static_cast<int64_t>(pairs.size()), [&](int64_t i) {
      keyed[i] = {rng_u64(kd, pairs[i]), pairs[i]};
    });
    std::nth_element(keyed.begin(), keyed.begin() + want, keyed.end());
    keyed.resize(want);
    pairs.resize(want);
    for (int64_t i = 0; i < want; ++i) pairs[i] = keyed[i].second;
    std::vector<std::pair<uint64_t, uint64_t>>().swap(keyed);
    std::sort(pairs.begin(), pairs.end());
  } else {
    uint64_t c = 0;
    const uint64_t kt = rng_fork(root, 0x64);
    std::vector<uint64_t> extra;
    while (static_cast<int64_t>(pairs.size() + extra.size()) < want) {
      const int64_t u = static_cast<int64_t>(rng_u64(kt, ++c) % static_cast<uint64_t>(n));
      const int64_t b0 = (u / bsz) * bsz, b1 = std::min(n, b0 + bsz);
      const int64_t v = b0 + static_cast<int64_t>(rng_u64(kt, ++c) % static_cast<uint64_t>(b1 - b0));
      if (u == v) continue;
      const uint64_t key = static_cast<uint64_t>(std::min(u, v)) << 32 |
                           static_cast<uint64_t>(std::max(u, v));
      if (std::binary_search(pairs.begin(), pairs.end(), key)) continue;
      extra.push_back(key);
      if (static_cast<int64_t>(pairs.size() + extra.size()) == want) {
        std::sort(extra.begin(), extra.end());
        extra.erase(std::unique(extra.begin(), extra.end()), extra.end());
      }
    }
    pairs.insert(pairs.end(), extra.begin(), extra.end());
    std::sort(pairs.begin(), pairs.end());
  }
  // symmetric CSR
  std::vector<int64_t> deg(n + 1, 0);
  for (uint64_t x : pairs) {
    ++deg[(x >> 32) + 1];
    ++deg[(x & 0xffffffffu) + 1];
  }
  adj_ptr[0] = 0;
  for (int64_t v = 0; v < n; ++v) adj_ptr[v + 1] = adj_ptr[v] + deg[v + 1];
  {
    std::vector<int64_t> fill(adj_ptr, adj_ptr + n);
    for (uint64_t x : pairs) {
      const int64_t a = static_cast<int64_t>(x >> 32), b = static_cast<int64_t>(x & 0xffffffffu);
      adj[fill[a]++] = static_cast<int32_t>(b);
      adj[fill[b]++] = static_cast<int32_t>(a);
    }
  }
  std::vector<uint64_t>().swap(pairs);
  parallel_for(n, [&](int64_t v) { std::sort(adj + adj_ptr[v], adj + adj_ptr[v + 1]); });
  // labels: 256-node communities mapped to classes by a hash
  const uint64_t kl = rng_fork(root, 0x51);
  parallel_for(n, [&](int64_t v) {
    labels[v] = static_cast<int32_t>(rng_u64(kl, static_cast<uint64_t>(v / 256)) %
                                     static_cast<uint64_t>(s.classes));
  });
  // class means (synth.hpp:127-131) then per-node noise (:132-137)
  std::vector<double> means(s.classes * s.feat);
  {
    const uint64_t km = rng_fork(root, 0x54);
    uint64_t c = 0;
    for (auto& x : means) {
      double a = u01(km, ++c);
      while (a <= 0.0) a = u01(km, ++c);
      const double b = u01(km, ++c);
      x = std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586476925286766559 * b);
    }
  }
  const uint64_t kf = rng_fork(root, 0x55);
  parallel_for(n, [&](int64_t v) {
    const uint64_t k = rng_fork(kf, static_cast<uint64_t>(v));
    uint64_t c = 0;
    for (int64_t j = 0; j < s.feat; ++j) {
      double a = u01(k, ++c);
      while (a <= 0.0) a = u01(k, ++c);
      const double b = u01(k, ++c);
      const double gz = std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586476925286766559 * b);
      features[v * s.feat + j] = static_cast<float>(s.sep * means[labels[v] * s.feat + j] + gz);
    }
  });
  // 60/20/20 split by a per-node draw
  const uint64_t ks = rng_fork(root, 0x56);
  parallel_for(n, [&](int64_t v) {
    const double x = u01(ks, static_cast<uint64_t>(v) + 1);
    train[v] = x < 0.6;
    val[v] = x >= 0.6 && x < 0.8;
    test[v] = x >= 0.8;
  });
}
}  // namespace

extern "C" {
// adj must hold 2 * n_edges entries; returns 0, or 1 on bad arguments.
int qgnn_synth_planted(int64_t nodes, int64_t n_edges, int64_t feat, int64_t classes,
                       int64_t blocks, double cross_frac, double gamma, double sep,
                       uint64_t seed, int64_t* adj_ptr, int32_t* adj, float* features,
                       int32_t* labels, uint8_t* train, uint8_t* val, uint8_t* test) {
  if (nodes < 2 || n_edges < 1 || blocks < 1 || blocks > nodes || classes < 1 || feat < 1 ||
      gamma <= 1.0 || nodes > 0x7fffffff || n_edges >= nodes * (nodes - 1) / 4)
    return 1;
  try {
    gen_planted(PlantedSpec{nodes, n_edges, feat, classes, blocks, cross_frac, gamma, sep, seed},
                adj_ptr, adj, features, labels, train, val, test);
  } catch (...) {
    return 2;
  }
  return 0;
}
}
