// dataset.cpp — the reference's on-disk dataset (SURVEY.md §8f rank 3 loader):
// load_dataset (cli/synth.hpp:184-205) over the formats of graph.hpp:80-200 —
// edges.txt ("u v" per line, '#' comments), features.bin (u64 rows, u64 cols,
// row-major f64), labels.txt (one label per non-empty line), {train,val,test}_mask.txt
// (node ids), meta.json ("nodes").  The edge list is parsed on host threads and the
// symmetric, deduplicated, sorted CSR (build_graph, graph.hpp:59-78) is built on the
// GPU (radix sort of the 2E directed pairs, setup.cu); the features are delivered
// both as stored (f64) and rounded to fp32 for the production engine.  Errors carry
// the reference's IoError / invalid_argument messages.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <future>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "qgnn_b200.h"
#include "status.hpp"

namespace qgnn_b200 {
namespace {

std::string read_file(const std::string& path, const std::string& what) {
  std::ifstream in(path, std::ios::binary);
  QGNN_REQUIRE(in, QGNN_EIO, "cannot open " + what + ": " + path);
  in.seekg(0, std::ios::end);
  const std::streamoff n = in.tellg();
  in.seekg(0, std::ios::beg);
  std::string s(static_cast<size_t>(std::max<std::streamoff>(0, n)), '\0');
  if (n > 0) in.read(&s[0], n);
  return s;
}

// One "u v" line (graph.hpp:93-103): text after '#' ignored, blank lines skipped,
// a first id without a second is an error.  Returns 0 blank, 1 edge, -1 malformed.
int parse_edge_line(const char* b, const char* e, uint64_t& u, uint64_t& v) {
  const char* h = static_cast<const char*>(std::memchr(b, '#', size_t(e - b)));
  if (h) e = h;
  auto skip = [&](const char*& p) {
    while (p < e && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
  };
  auto num = [&](const char*& p, uint64_t& x) {
    skip(p);
    if (p < e && *p == '+') ++p;
    if (p >= e || *p < '0' || *p > '9') return false;
    x = 0;
    while (p < e && *p >= '0' && *p <= '9') x = x * 10 + uint64_t(*p++ - '0');
    return true;
  };
  const char* p = b;
  if (!num(p, u)) return 0;
  if (!num(p, v)) return -1;
  return 1;
}

std::vector<std::pair<uint32_t, uint32_t>> load_edges(const std::string& path, int64_t n) {
  const std::string s = read_file(path, "edge list");
  const size_t len = s.size();
  const int T = int(std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(),
                                                         len / (1 << 20) + 1)));
  std::vector<size_t> cut(T + 1, len);
  cut[0] = 0;
  for (int t = 1; t < T; ++t) {  // chunk starts at line boundaries
    size_t c = len * size_t(t) / size_t(T);
    while (c < len && s[c - 1] != '\n') ++c;
    cut[t] = std::max(c, cut[t - 1]);
  }
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> part(T);
  std::vector<size_t> bad(T, std::string::npos), range(T, std::string::npos);
  std::vector<std::future<void>> jobs;
  for (int t = 0; t < T; ++t)
    jobs.push_back(std::async(std::launch::async, [&, t] {
      const char* d = s.data();
      size_t i = cut[t];
      while (i < cut[t + 1]) {
        const char* nl = static_cast<const char*>(std::memchr(d + i, '\n', cut[t + 1] - i));
        const size_t j = nl ? size_t(nl - d) : cut[t + 1];
        uint64_t u = 0, v = 0;
        const int r = parse_edge_line(d + i, d + j, u, v);
        if (r < 0 && bad[t] == std::string::npos) bad[t] = i;
        if (r > 0) {
          if ((u >= uint64_t(n) || v >= uint64_t(n)) && range[t] == std::string::npos) range[t] = i;
          part[t].emplace_back(uint32_t(u), uint32_t(v));
        }
        i = j + 1;
      }
    }));
  for (auto& j : jobs) j.get();
  for (int t = 0; t < T; ++t) {
    if (bad[t] != std::string::npos) {
      const size_t lineno = size_t(std::count(s.begin(), s.begin() + long(bad[t]), '\n')) + 1;
      throw Status(QGNN_EIO, path + ":" + std::to_string(lineno) + ": expected two node ids");
    }
    // build_graph (graph.hpp:62)
    QGNN_REQUIRE(range[t] == std::string::npos, QGNN_EINVAL, "edge endpoint out of range");
  }
  std::vector<std::pair<uint32_t, uint32_t>> all;
  size_t tot = 0;
  for (auto& p : part) tot += p.size();
  all.reserve(tot);
  for (auto& p : part) all.insert(all.end(), p.begin(), p.end());
  return all;
}

// graph.hpp:164-181
std::vector<int32_t> load_labels(const std::string& path, int64_t n) {
  const std::string s = read_file(path, "labels");
  std::vector<int32_t> labels(size_t(n), 0);
  int64_t row = 0;
  size_t i = 0;
  while (i < s.size()) {
    size_t j = s.find('\n', i);
    if (j == std::string::npos) j = s.size();
    std::string line = s.substr(i, j - i);
    i = j + 1;
    if (line.empty()) continue;
    QGNN_REQUIRE(row < n, QGNN_EIO, "too many label rows: " + path);
    try {
      labels[size_t(row++)] = std::stoi(line);
    } catch (const std::exception&) {
      throw Status(QGNN_EIO, path + ": bad label '" + line + "'");
    }
  }
  QGNN_REQUIRE(row == n, QGNN_EIO, "label count mismatch: " + path);
  return labels;
}

// graph.hpp:183-193
std::vector<uint8_t> load_mask(const std::string& path, int64_t n) {
  const std::string s = read_file(path, "mask");
  std::vector<uint8_t> mask(size_t(n), 0);
  const char* p = s.data();
  const char* e = p + s.size();
  while (p < e) {
    while (p < e && (*p == ' ' || *p == '\n' || *p == '\t' || *p == '\r')) ++p;
    if (p >= e || *p < '0' || *p > '9') break;  // >> stops at the first non-number
    uint64_t v = 0;
    while (p < e && *p >= '0' && *p <= '9') v = v * 10 + uint64_t(*p++ - '0');
    QGNN_REQUIRE(v < uint64_t(n), QGNN_EIO, "mask node id out of range: " + path);
    mask[size_t(v)] = 1;
  }
  return mask;
}

// the "nodes" (and, when present, "classes") fields of meta.json
int64_t meta_field(const std::string& s, const char* key, bool required, const std::string& dir) {
  const std::string k = std::string("\"") + key + "\"";
  const size_t at = s.find(k);
  if (at == std::string::npos) {
    QGNN_REQUIRE(!required, QGNN_EIO, std::string("bad dataset meta in ") + dir + ": no " + key);
    return -1;
  }
  size_t p = s.find(':', at + k.size());
  QGNN_REQUIRE(p != std::string::npos, QGNN_EIO, "bad dataset meta in " + dir);
  ++p;
  while (p < s.size() && (s[p] == ' ' || s[p] == '\n' || s[p] == '\t' || s[p] == '\r')) ++p;
  QGNN_REQUIRE(p < s.size() && s[p] >= '0' && s[p] <= '9', QGNN_EIO,
               std::string("bad dataset meta in ") + dir + ": " + key);
  int64_t v = 0;
  while (p < s.size() && s[p] >= '0' && s[p] <= '9') v = v * 10 + (s[p++] - '0');
  return v;
}

}  // namespace
}  // namespace qgnn_b200

using namespace qgnn_b200;

struct qgnn_dataset {
  int64_t nodes = 0, feature_dim = 0, classes = 0;
  std::vector<int64_t> adj_ptr;
  std::vector<int32_t> adj;
  std::vector<double> features;
  std::vector<float> features_f32;
  std::vector<int32_t> labels;
  std::vector<uint8_t> train, val, test;
};

extern "C" {

int qgnn_dataset_load(const char* dir_c, int device, qgnn_dataset** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(dir_c && out, QGNN_EINVAL, "dataset: null argument");
  const std::string dir(dir_c);
  const std::string base = dir + "/";
  std::string meta;
  {
    std::ifstream mf(base + "meta.json", std::ios::binary);
    QGNN_REQUIRE(mf, QGNN_EIO, "cannot open dataset meta: " + dir);
    meta.assign(std::istreambuf_iterator<char>(mf), std::istreambuf_iterator<char>());
  }
  auto* D = new qgnn_dataset;
  try {
    D->nodes = meta_field(meta, "nodes", true, dir);
    D->classes = meta_field(meta, "classes", false, dir);
    const int64_t n = D->nodes;
    // the five files in parallel: the edge list is the big one
    auto fe = std::async(std::launch::async, [&] { return load_edges(base + "edges.txt", n); });
    auto fl = std::async(std::launch::async, [&] { return load_labels(base + "labels.txt", n); });
    auto ftr = std::async(std::launch::async, [&] { return load_mask(base + "train_mask.txt", n); });
    auto fva = std::async(std::launch::async, [&] { return load_mask(base + "val_mask.txt", n); });
    auto fte = std::async(std::launch::async, [&] { return load_mask(base + "test_mask.txt", n); });
    {  // features.bin (graph.hpp:120-136)
      const std::string fp = base + "features.bin";
      std::ifstream in(fp, std::ios::binary);
      QGNN_REQUIRE(in, QGNN_EIO, "cannot open: " + fp);
      uint64_t r = 0, c = 0;
      in.read(reinterpret_cast<char*>(&r), 8);
      in.read(reinterpret_cast<char*>(&c), 8);
      QGNN_REQUIRE(in, QGNN_EIO, "truncated header: " + fp);
      QGNN_REQUIRE(r <= (1ull << 32) && c <= (1ull << 24), QGNN_EIO,
                   "implausible matrix dims: " + fp);
      D->features.resize(size_t(r * c));
      in.read(reinterpret_cast<char*>(D->features.data()),
              static_cast<std::streamsize>(D->features.size() * sizeof(double)));
      QGNN_REQUIRE(in, QGNN_EIO, "truncated payload: " + fp);
      QGNN_REQUIRE(int64_t(r) == n, QGNN_EIO, "dataset features row count mismatch: " + dir);
      D->feature_dim = int64_t(c);
      D->features_f32.resize(D->features.size());
      const size_t N = D->features.size();
      const int T = int(std::max(1u, std::thread::hardware_concurrency()));
      std::vector<std::future<void>> cv;
      for (int t = 0; t < T; ++t)
        cv.push_back(std::async(std::launch::async, [&, t] {
          for (size_t i = N * size_t(t) / size_t(T); i < N * size_t(t + 1) / size_t(T); ++i)
            D->features_f32[i] = static_cast<float>(D->features[i]);
        }));
      for (auto& f : cv) f.get();
    }
    const auto edges = fe.get();
    D->labels = fl.get();
    D->train = ftr.get();
    D->val = fva.get();
    D->test = fte.get();
    build_graph_csr(n, edges, device, D->adj_ptr, D->adj);
    for (int64_t v = 0; v < n; ++v)  // Graph::validate (graph.hpp:52-54)
      QGNN_REQUIRE(D->train[v] + D->val[v] + D->test[v] <= 1, QGNN_EINVAL,
                   "graph: overlapping masks");
    if (D->classes < 0) {
      int32_t c = 0;
      for (int32_t y : D->labels) c = std::max(c, y + 1);
      D->classes = c;
    }
  } catch (...) {
    delete D;
    throw;
  }
  *out = D;
  QGNN_API_END
}

int qgnn_dataset_arrays_get(const qgnn_dataset* d, qgnn_dataset_arrays* a) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(d && a, QGNN_EINVAL, "dataset: null argument");
  a->nodes = d->nodes;
  a->nnz = int64_t(d->adj.size());
  a->feature_dim = d->feature_dim;
  a->classes = d->classes;
  a->adj_ptr = d->adj_ptr.data();
  a->adj = d->adj.data();
  a->features = d->features.data();
  a->features_f32 = d->features_f32.data();
  a->labels = d->labels.data();
  a->train = d->train.data();
  a->val = d->val.data();
  a->test = d->test.data();
  QGNN_API_END
}

int qgnn_dataset_destroy(qgnn_dataset* d) {
  delete d;
  return QGNN_OK;
}

}  // extern "C"
