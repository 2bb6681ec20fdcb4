// host_solve.cpp — the adaptive bit-width assigner kept on the host
// (north star (6)): variance weights, grouping, the canonical bi-objective,
// the exact per-pair knapsack solver and the brute-force oracle
// (assigner/trace.hpp:71-74, assigner/solve.hpp:24-363), and the affine
// cost-model fit (commsim/cost_model.hpp:78-109).
//
// Floating-point expressions are evaluated in the reference's order and the
// TU is built with -ffp-contract=off, so plans, objectives and tie-breaks are
// identical to the reference's solve_assignment.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <optional>
#include <string>
#include <thread>

#include "host.hpp"
#include "qgnn_b200.h"
#include "status.hpp"

namespace qgnn_b200 {

namespace {
constexpr int kBits[3] = {2, 4, 8};
constexpr size_t kBruteLimit = 16;  // solve.hpp:20

double variance_at(double beta, int bits) {  // solve.hpp:60-63
  const double levels = static_cast<double>((1u << bits) - 1);
  return beta / (levels * levels);
}

struct Eval {
  double objective = 0, variance = 0, z = 0;
};

Eval evaluate(const SolveResult& plan, const Cost& cm, double lambda) {  // solve.hpp:68-81
  Eval ev;
  for (const PlanPairG& pp : plan.pairs) {
    uint64_t pair_bits = 0;
    for (const Group& g : pp.groups) {
      ev.variance += variance_at(g.beta, g.bits);
      pair_bits += g.dim_sum() * static_cast<uint64_t>(g.bits);
    }
    ev.z = std::max(ev.z, cm.seconds(pp.src, pp.dst, static_cast<double>(pair_bits)));
  }
  ev.objective = lambda * ev.variance + (1.0 - lambda) * ev.z;
  return ev;
}

void validate(const SolveResult& plan, const Cost& cm, double lambda) {  // solve.hpp:85-101
  QGNN_REQUIRE(lambda >= 0.0 && lambda <= 1.0, QGNN_EINVAL, "solve: lambda must be in [0, 1]");
  QGNN_REQUIRE(!plan.pairs.empty(), QGNN_EINVAL, "solve: no device pairs");
  for (const PlanPairG& pp : plan.pairs) {
    QGNN_REQUIRE(pp.src < cm.n && pp.dst < cm.n, QGNN_EINVAL, "solve: pair outside cost model");
    QGNN_REQUIRE(!pp.groups.empty(), QGNN_EINVAL, "solve: empty groups");
    for (const Group& g : pp.groups) {
      QGNN_REQUIRE(!g.ids.empty() && g.ids.size() == g.dims.size(), QGNN_EINVAL,
                   "solve: malformed group");
      QGNN_REQUIRE(g.dim_sum() != 0, QGNN_EINVAL, "solve: zero-dim group");
      QGNN_REQUIRE(g.beta >= 0.0 && std::isfinite(g.beta), QGNN_EINVAL,
                   "solve: beta must be finite and >= 0");
    }
  }
}

std::vector<int> flat_bits(const SolveResult& p) {
  std::vector<int> b;
  for (const auto& pp : p.pairs)
    for (const auto& g : pp.groups) b.push_back(g.bits);
  return b;
}
void set_bits(SolveResult& p, const std::vector<int>& b) {
  size_t i = 0;
  for (auto& pp : p.pairs)
    for (auto& g : pp.groups) g.bits = b[i++];
}
// objective, then variance, then lexicographically larger bit vector (solve.hpp:116-121)
bool better(const Eval& a, const std::vector<int>& ba, const Eval& b, const std::vector<int>& bb) {
  if (a.objective != b.objective) return a.objective < b.objective;
  if (a.variance != b.variance) return a.variance < b.variance;
  return ba > bb;
}

// Per-pair knapsack over scaled bit totals (solve.hpp:125-194).  The
// reference fills a dense (groups + 1) x (smax + 1) table of least variances
// (148 MB over the 56 pairs of the bench's re-solve); each row is a step
// function of the capacity c whose steps sit at achievable bit totals, so row
// j is kept as its frontier: ascending totals with strictly decreasing
// variance, mv(j, c) = the value of the last entry <= c.  Every entry's value
// is var(bits) + value of a row-(j+1) entry, added in the reference's order,
// and rounding is monotone, so min over the entries <= c equals the dense
// cell bit for bit.
struct Table {
  double theta = 0, gamma = 0;
  uint64_t unit = 1, smax = 0;
  size_t n = 0;
  std::vector<uint64_t> w;  // [j*3 + bi]
  std::vector<std::vector<uint64_t>> fw;  // frontier totals of row j, j in [0, n]
  std::vector<std::vector<double>> fv;    // their least variances (strictly decreasing)
  std::vector<uint64_t> reach;            // every achievable total, ascending
  double mv(size_t j, uint64_t c) const {
    const auto& r = fw[j];
    const auto it = std::upper_bound(r.begin(), r.end(), c);
    return it == r.begin() ? std::numeric_limits<double>::infinity()
                           : fv[j][size_t(it - r.begin()) - 1];
  }
  double time_at(uint64_t s) const { return theta * static_cast<double>(s * unit) + gamma; }
  std::optional<uint64_t> cap_for(double z) const {  // solve.hpp:137-148
    if (time_at(0) > z) return std::nullopt;
    uint64_t lo = 0, hi = smax;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo + 1) / 2;
      if (time_at(mid) <= z)
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  }
  // largest achievable total <= c, or -1
  int64_t reach_below(uint64_t c) const {
    const auto it = std::upper_bound(reach.begin(), reach.end(), c);
    return it == reach.begin() ? -1 : int64_t(*(it - 1));
  }
};

Table build_table(const PlanPairG& pp, const Cost& cm) {
  Table t;
  t.theta = cm.theta[pp.src * cm.n + pp.dst];
  t.gamma = cm.gamma[pp.src * cm.n + pp.dst];
  uint64_t base = 0;
  for (const Group& g : pp.groups) base = std::gcd(base, g.dim_sum());
  t.unit = 2 * base;
  t.n = pp.groups.size();
  t.w.resize(t.n * 3);
  for (size_t j = 0; j < t.n; ++j) {
    for (int bi = 0; bi < 3; ++bi) t.w[j * 3 + bi] = pp.groups[j].dim_sum() * kBits[bi] / t.unit;
    t.smax += t.w[j * 3 + 2];
  }
  t.fw.resize(t.n + 1);
  t.fv.resize(t.n + 1);
  t.fw[t.n] = {0};  // no groups left: variance 0 at every capacity
  t.fv[t.n] = {0.0};
  std::vector<std::pair<uint64_t, double>> e;
  for (size_t j = t.n; j-- > 0;) {
    const auto& bw = t.fw[j + 1];
    const auto& bv = t.fv[j + 1];
    e.clear();
    for (int bi = 0; bi < 3; ++bi) {
      const double var = variance_at(pp.groups[j].beta, kBits[bi]);
      for (size_t k = 0; k < bw.size(); ++k) e.emplace_back(bw[k] + t.w[j * 3 + bi], var + bv[k]);
    }
    std::sort(e.begin(), e.end());
    double best = std::numeric_limits<double>::infinity();
    for (const auto& [wt, v] : e)
      if (v < best) {  // first entry of a total is its least value
        t.fw[j].push_back(wt);
        t.fv[j].push_back(v);
        best = v;
      }
  }
  t.reach = {0};
  std::vector<uint64_t> next;
  for (size_t j = 0; j < t.n; ++j) {
    next.clear();
    for (int bi = 0; bi < 3; ++bi)
      for (uint64_t s : t.reach) next.push_back(s + t.w[j * 3 + bi]);
    std::sort(next.begin(), next.end());
    next.erase(std::unique(next.begin(), next.end()), next.end());
    t.reach.swap(next);
  }
  return t;
}

// greedy largest-bits walk consistent with the minima (solve.hpp:197-214)
void reconstruct(const Table& t, const PlanPairG& pp, uint64_t cap, int* out) {
  uint64_t c = cap;
  const double inf = std::numeric_limits<double>::infinity();
  for (size_t j = 0; j < pp.groups.size(); ++j) {
    int pick = 0;
    for (int bi = 2; bi >= 0; --bi) {
      const uint64_t wt = t.w[j * 3 + bi];
      if (wt > c) continue;
      const double b = t.mv(j + 1, c - wt);
      if (b == inf) continue;
      if (variance_at(pp.groups[j].beta, kBits[bi]) + b == t.mv(j, c)) {
        pick = kBits[bi];
        c -= wt;
        break;
      }
    }
    out[j] = pick;
  }
}
}  // namespace

uint64_t Group::dim_sum() const { return std::accumulate(dims.begin(), dims.end(), uint64_t{0}); }

double compute_beta(const MsgStat& m) {  // trace.hpp:71-74
  const double range = m.hi - m.lo;
  return m.asq * static_cast<double>(m.dim) * range * range / 6.0;
}

namespace {
// Stable LSD radix sort by descending value of non-negative doubles (11-bit
// digits over the IEEE pattern, constant digits skipped).
template <typename K>
void radix_sort_desc(std::vector<K>& v) {
  const size_t n = v.size();
  if (n < 2) return;
  std::vector<K> tmp(n);
  std::vector<uint64_t> key(n), ktmp(n);
  for (size_t i = 0; i < n; ++i) {
    uint64_t b;
    std::memcpy(&b, &v[i].beta, 8);
    key[i] = ~b;
  }
  constexpr int kDig = 11, kB = 1 << kDig;
  std::vector<uint32_t> cnt(kB);
  for (int sh = 0; sh < 64; sh += kDig) {
    std::fill(cnt.begin(), cnt.end(), 0u);
    for (size_t i = 0; i < n; ++i) ++cnt[(key[i] >> sh) & (kB - 1)];
    if (cnt[(key[0] >> sh) & (kB - 1)] == n) continue;  // one digit value: order unchanged
    uint32_t s = 0;
    for (auto& c : cnt) {
      const uint32_t t = c;
      c = s;
      s += t;
    }
    for (size_t i = 0; i < n; ++i) {
      const uint32_t d = cnt[(key[i] >> sh) & (kB - 1)]++;
      tmp[d] = v[i];
      ktmp[d] = key[i];
    }
    v.swap(tmp);
    key.swap(ktmp);
  }
}
}  // namespace

SolveResult group_and_order(const std::vector<PairStat>& pairs, int64_t group_size) {
  QGNN_REQUIRE(group_size > 0, QGNN_EINVAL, "group_and_order: group_size must be > 0");
  for (const PairStat& p : pairs) {  // trace.hpp:58-67
    QGNN_REQUIRE(p.src != p.dst, QGNN_EINVAL, "stats: src == dst");
    for (const MsgStat& m : p.msgs) {
      QGNN_REQUIRE(m.dim != 0, QGNN_EINVAL, "stats: zero dim");
      QGNN_REQUIRE(!(m.hi < m.lo), QGNN_EINVAL, "stats: hi < lo");
      QGNN_REQUIRE(m.asq > 0.0, QGNN_EINVAL, "stats: sum_alpha_sq must be > 0");
    }
  }
  // pairs are independent: grouped on worker threads, kept in input order
  // (beta desc, id asc) as in the reference's stable_sort.  Messages arrive in
  // ascending id (the engine's send order), so a stable LSD radix sort on the
  // descending-beta bit pattern gives that order directly (beta >= 0: the IEEE
  // pattern is monotone); any other input — unsorted ids, a NaN or -0 beta —
  // keeps the reference's stable_sort call.
  struct Key {
    double beta;
    uint32_t id, idx;
  };
  std::vector<PlanPairG> out(pairs.size());
  auto one = [&](size_t pi) {
    const PairStat& p = pairs[pi];
    const size_t n = p.msgs.size();
    std::vector<Key> order(n);
    bool radix = true;
    for (size_t i = 0; i < n; ++i) {
      order[i] = {compute_beta(p.msgs[i]), p.msgs[i].id, uint32_t(i)};
      radix &= !std::signbit(order[i].beta) && !std::isnan(order[i].beta) &&
               (i == 0 || p.msgs[i - 1].id < p.msgs[i].id);
    }
    if (radix) {
      radix_sort_desc(order);
    } else {
      std::stable_sort(order.begin(), order.end(), [](const Key& a, const Key& b) {
        if (a.beta != b.beta) return a.beta > b.beta;
        return a.id < b.id;
      });
    }
    PlanPairG pp;
    pp.src = p.src;
    pp.dst = p.dst;
    const size_t gs = static_cast<size_t>(group_size);
    pp.groups.reserve((n + gs - 1) / gs);
    for (size_t i = 0; i < n; i += gs) {
      const size_t e = std::min(n, i + gs);
      Group g;
      g.ids.reserve(e - i);
      g.pos.reserve(e - i);
      g.dims.reserve(e - i);
      for (size_t j = i; j < e; ++j) {
        const MsgStat& m = p.msgs[order[j].idx];
        g.ids.push_back(m.id);
        g.pos.push_back(m.pos);
        g.dims.push_back(m.dim);
        g.beta += order[j].beta;
      }
      pp.groups.push_back(std::move(g));
    }
    out[pi] = std::move(pp);
  };
  size_t nthr = std::max<size_t>(1, std::min<size_t>(pairs.size(),
                                                      std::thread::hardware_concurrency() / 2));
  if (const char* e = std::getenv("QGNN_SOLVE_THREADS"))
    nthr = std::max<size_t>(1, std::min<size_t>(pairs.size(), size_t(std::atoi(e))));
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t i; (i = next.fetch_add(1)) < pairs.size();)
      if (!pairs[i].msgs.empty()) one(i);
  };
  std::vector<std::thread> th;
  for (size_t t = 1; t < nthr; ++t) th.emplace_back(worker);
  worker();
  for (auto& t : th) t.join();
  SolveResult plan;
  for (size_t i = 0; i < pairs.size(); ++i)
    if (!pairs[i].msgs.empty()) plan.pairs.push_back(std::move(out[i]));
  return plan;
}

// Exact solve (solve.hpp:264-309): every candidate makespan z (each pair's
// reachable transfer times) gives each pair its min-variance assignment under
// cap(z); the best (objective, variance, larger bits) wins.  Same caps, same
// reconstruction, same evaluation order as the reference, but:
//  * knapsack rows are frontiers (Table), and a pair's cap is tracked as the
//    largest achievable total under it; with theta >= 0 that index only
//    advances (a pointer instead of a binary search per candidate);
//  * a pair is reconstructed only when that total moves, and a candidate is
//    evaluated only when some pair's bits actually changed (identical bits give
//    an identical evaluation, which never beats the earlier candidate);
//  * per-group variances for the three widths are tabulated once;
//  * the candidate range is split over worker threads (each starts with binary
//    searched caps) and merged in range order with the reference's tie-break.
namespace {
struct EvalCtx {
  const SolveResult* plan;
  const Cost* cm;
  double lambda;
  std::vector<double> var3;        // [group * 3 + bi] = variance_at(beta, 2/4/8)
  std::vector<uint64_t> dimsum;    // per group (flat)
  std::vector<size_t> pair_first;  // first flat group of each pair
};

Eval eval_bits(const EvalCtx& C, const std::vector<int>& bits) {  // == evaluate()
  Eval ev;
  const SolveResult& plan = *C.plan;
  for (size_t i = 0; i < plan.pairs.size(); ++i) {
    uint64_t pair_bits = 0;
    for (size_t g = C.pair_first[i]; g < C.pair_first[i + 1]; ++g) {
      const int b = bits[g];
      ev.variance += C.var3[g * 3 + (b == 2 ? 0 : b == 4 ? 1 : 2)];
      pair_bits += C.dimsum[g] * static_cast<uint64_t>(b);
    }
    const PlanPairG& pp = plan.pairs[i];
    ev.z = std::max(ev.z, C.cm->seconds(pp.src, pp.dst, static_cast<double>(pair_bits)));
  }
  ev.objective = C.lambda * ev.variance + (1.0 - C.lambda) * ev.z;
  return ev;
}

struct ScanBest {
  bool have = false;
  Eval best;
  std::vector<int> bits;
};

// k[i] indexes the largest achievable total of pair i that fits the budget
// (reach_below(cap_for(z))), -1 if none (then mv(0, cap) is infinite: the
// candidate is infeasible).  Every step of every row sits at an achievable
// total, so the greedy walk gives the same bits anywhere between two
// consecutive totals: a pair is rebuilt only when its k moves.
void scan(const EvalCtx& C, const std::vector<Table>& tables, const std::vector<double>& cand,
          size_t c0, size_t c1, bool monotone, ScanBest& out) {
  if (c0 >= c1) return;
  const SolveResult& plan = *C.plan;
  const size_t P = tables.size();
  auto locate = [&](const Table& t, double z) -> int64_t {
    const auto c = t.cap_for(z);
    if (!c) return -1;
    return int64_t(std::upper_bound(t.reach.begin(), t.reach.end(), *c) - t.reach.begin()) - 1;
  };
  std::vector<int64_t> k(P, -1), done(P, -2);
  std::vector<int> bits(C.dimsum.size(), 0), nb;
  bool dirty = true;
  for (size_t i = 0; i < P; ++i) k[i] = locate(tables[i], cand[c0]);
  for (size_t ci = c0; ci < c1; ++ci) {
    const double z = cand[ci];
    bool feasible = true;
    for (size_t i = 0; i < P; ++i) {
      const Table& t = tables[i];
      if (!monotone)
        k[i] = locate(t, z);
      else  // time_at non-decreasing: the index only advances
        while (k[i] + 1 < int64_t(t.reach.size()) && t.time_at(t.reach[size_t(k[i] + 1)]) <= z)
          ++k[i];
      if (k[i] < 0) {
        feasible = false;
        continue;  // keep advancing the other pairs
      }
      if (done[i] != k[i]) {
        const size_t ng = plan.pairs[i].groups.size();
        nb.resize(ng);
        reconstruct(t, plan.pairs[i], t.reach[size_t(k[i])], nb.data());
        done[i] = k[i];
        if (!std::equal(nb.begin(), nb.end(), bits.begin() + C.pair_first[i])) {
          std::copy(nb.begin(), nb.end(), bits.begin() + C.pair_first[i]);
          dirty = true;
        }
      }
    }
    if (!feasible || !dirty) continue;
    dirty = false;
    const Eval ev = eval_bits(C, bits);
    if (!out.have || better(ev, bits, out.best, out.bits)) {
      out.best = ev;
      out.bits = bits;
      out.have = true;
    }
  }
}
}  // namespace

void solve_exact(SolveResult& plan, const Cost& cm, double lambda) {
  validate(plan, cm, lambda);
  // per-pair knapsack tables are independent: build them on worker threads
  const size_t P = plan.pairs.size();
  std::vector<Table> tables(P);
  {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t W = std::min<size_t>(P, std::max(1u, std::min(16u, hw / 2)));
    std::atomic<size_t> next{0};
    std::vector<std::string> errs(W);
    auto work = [&](size_t w) {
      try {
        for (size_t i = next++; i < P; i = next++) tables[i] = build_table(plan.pairs[i], cm);
      } catch (const std::exception& e) {
        errs[w] = e.what();
      }
    };
    std::vector<std::thread> th;
    for (size_t w = 1; w < W; ++w) th.emplace_back(work, w);
    work(0);
    for (auto& x : th) x.join();
    for (const auto& e : errs)
      QGNN_REQUIRE(e.empty(), QGNN_ERESOURCE, e);
  }
  std::vector<double> cand;
  bool monotone = true;
  for (const Table& t : tables) {
    monotone &= t.theta >= 0.0 && std::isfinite(t.theta) && std::isfinite(t.gamma);
    for (uint64_t s : t.reach) cand.push_back(t.time_at(s));
  }
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());

  EvalCtx C;
  C.plan = &plan;
  C.cm = &cm;
  C.lambda = lambda;
  C.pair_first.push_back(0);
  for (const PlanPairG& pp : plan.pairs) {
    for (const Group& g : pp.groups) {
      for (int bi = 0; bi < 3; ++bi) C.var3.push_back(variance_at(g.beta, kBits[bi]));
      C.dimsum.push_back(g.dim_sum());
    }
    C.pair_first.push_back(C.dimsum.size());
  }

  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  size_t T = std::min<size_t>(std::max<size_t>(1, cand.size() / 65536),
                              std::max(1u, std::min(8u, hw / 4)));
  if (const char* e = std::getenv("QGNN_SOLVE_THREADS"))  // tests: force the split
    T = std::max<size_t>(1, std::min<size_t>(cand.size(), size_t(std::atoi(e))));
  std::vector<ScanBest> part(T);
  auto run = [&](size_t t) {
    scan(C, tables, cand, cand.size() * t / T, cand.size() * (t + 1) / T, monotone, part[t]);
  };
  if (T == 1) {
    run(0);
  } else {
    std::vector<std::thread> th;
    for (size_t t = 0; t < T; ++t) th.emplace_back(run, t);
    for (auto& x : th) x.join();
  }
  ScanBest best;
  for (size_t t = 0; t < T; ++t)  // range order: earlier ranges win exact ties
    if (part[t].have && (!best.have || better(part[t].best, part[t].bits, best.best, best.bits)))
      best = std::move(part[t]);
  QGNN_REQUIRE(best.have, QGNN_EINVAL, "solve_assignment: no feasible assignment");
  set_bits(plan, best.bits);
  plan.objective = best.best.objective;
  plan.variance = best.best.variance;
  plan.z = best.best.z;
}

void solve_brute(SolveResult& plan, const Cost& cm, double lambda) {
  validate(plan, cm, lambda);
  size_t n = 0;
  for (const auto& pp : plan.pairs) n += pp.groups.size();
  QGNN_REQUIRE(n <= kBruteLimit, QGNN_ERESOURCE, "brute_force_assignment: too many groups");
  std::vector<int> idx(n, 0), bits(n, 2), best_bits;
  Eval best;
  bool have = false;
  SolveResult work = plan;
  for (;;) {
    set_bits(work, bits);
    const Eval ev = evaluate(work, cm, lambda);
    if (!have || better(ev, bits, best, best_bits)) {
      best = ev;
      best_bits = bits;
      have = true;
    }
    size_t j = 0;
    while (j < n) {
      if (++idx[j] < 3) {
        bits[j] = kBits[idx[j]];
        break;
      }
      idx[j] = 0;
      bits[j] = 2;
      ++j;
    }
    if (j == n) break;
  }
  set_bits(plan, best_bits);
  plan.objective = best.objective;
  plan.variance = best.variance;
  plan.z = best.z;
}

double uniform_expected_variance(const std::vector<PairStat>& pairs) {  // solve.hpp:313-326
  double mean_inv = 0.0;
  for (int b : kBits) {
    const double levels = static_cast<double>((1u << b) - 1);
    mean_inv += 1.0 / (levels * levels);
  }
  mean_inv /= 3.0;
  double total = 0.0;
  for (const auto& p : pairs)
    for (const auto& m : p.msgs) total += compute_beta(m) * mean_inv;
  return total;
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

extern "C" {

int qgnn_solve_instance(int64_t n_pairs, const uint32_t* pair_src, const uint32_t* pair_dst,
                        const uint64_t* pair_count, const uint32_t* m_id, const uint64_t* m_dim,
                        const double* m_lo, const double* m_hi, const double* m_asq,
                        int64_t n_devices, const double* theta, const double* gamma,
                        double lambda, int64_t group_size, int brute, int32_t* out_bits,
                        double* eval) {
  QGNN_API_BEGIN
  std::vector<PairStat> pairs(n_pairs);
  uint64_t o = 0;
  for (int64_t p = 0; p < n_pairs; ++p) {
    pairs[p].src = pair_src[p];
    pairs[p].dst = pair_dst[p];
    for (uint64_t i = 0; i < pair_count[p]; ++i, ++o)
      pairs[p].msgs.push_back({m_id[o], m_dim[o], m_lo[o], m_hi[o], m_asq[o]});
  }
  Cost cm;
  cm.n = n_devices;
  cm.theta.assign(theta, theta + n_devices * n_devices);
  cm.gamma.assign(gamma, gamma + n_devices * n_devices);
  SolveResult plan = group_and_order(pairs, group_size);
  if (brute)
    solve_brute(plan, cm, lambda);
  else
    solve_exact(plan, cm, lambda);
  eval[0] = plan.objective;
  eval[1] = plan.variance;
  eval[2] = plan.z;
  // map back to input order
  std::map<std::pair<uint32_t, uint32_t>, std::map<uint32_t, int>> bits;
  for (const auto& pp : plan.pairs)
    for (const auto& g : pp.groups)
      for (uint32_t id : g.ids) bits[{pp.src, pp.dst}][id] = g.bits;
  o = 0;
  for (int64_t p = 0; p < n_pairs; ++p)
    for (uint64_t i = 0; i < pair_count[p]; ++i, ++o)
      out_bits[o] = bits[{pair_src[p], pair_dst[p]}][m_id[o]];
  QGNN_API_END
}

// cost_model.hpp:78-109, one pair
int qgnn_fit_affine(const double* x, const double* y, int64_t n, double* theta, double* gamma) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(n >= 2, QGNN_EINVAL, "fit_cost_model: need at least 2 samples per pair");
  double mx = 0, my = 0;
  for (int64_t i = 0; i < n; ++i) {
    mx += x[i];
    my += y[i];
  }
  mx /= static_cast<double>(n);
  my /= static_cast<double>(n);
  double sxx = 0, sxy = 0;
  for (int64_t i = 0; i < n; ++i) {
    sxx += (x[i] - mx) * (x[i] - mx);
    sxy += (x[i] - mx) * (y[i] - my);
  }
  QGNN_REQUIRE(sxx != 0.0, QGNN_EINVAL, "fit_cost_model: need at least 2 distinct sizes per pair");
  const double th = sxy / sxx;
  const double ga = my - th * mx;
  *theta = std::max(0.0, th);
  *gamma = std::max(0.0, ga);
  QGNN_API_END
}

}  // extern "C"
