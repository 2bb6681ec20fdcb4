/*
 * qgnn_oracle.c — CPU restatement of the AdaQP (qgnn) boundary-message path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product in paper_2306_01381_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product path never does.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function
 * here against (a) the reference's own known-answer tests (test_quantcodec.cpp
 * pack KATs, chunk wire KAT, lattice/constant quantize, set ordering) and
 * (b) golden vectors produced by the compiled reference headers
 * (oracle/_ref/libqgnn_ref.so, recipe oracle/Makefile, fixtures under
 * tests/golden/ made by tests/golden/make_golden.py).
 *
 * All arithmetic is fp64 with no FMA contraction (build with
 * -ffp-contract=off), exactly as the reference's x86-64 build.
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/include/qgnn/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define QO_PHI 0x9e3779b97f4a7c15ull

/* status codes mirror include/qgnn_b200.h */
enum { QO_OK = 0, QO_EINVAL = 1, QO_EDECODE = 2 };

/* ---------------------------------------------------------------- rng ---- */
/* quantcodec/rng.hpp:52-57 */
uint64_t qo_mix(uint64_t z) {
  z += QO_PHI;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
/* rng.hpp:15 — RngStream(seed) key */
uint64_t qo_seed_key(uint64_t seed) { return qo_mix(seed ^ 0x6a09e667f3bcc909ull); }
/* rng.hpp:17-22 — fork(coord) */
uint64_t qo_fork(uint64_t key, uint64_t coord) { return qo_mix(key ^ qo_mix(coord + QO_PHI)); }
/* rng.hpp:30 — next_u64 with the counter already incremented to `ctr` */
uint64_t qo_draw_u64(uint64_t key, uint64_t ctr) { return qo_mix(key + ctr * QO_PHI); }
/* rng.hpp:33 */
double qo_draw_double(uint64_t key, uint64_t ctr) {
  return (double)(qo_draw_u64(key, ctr) >> 11) * 0x1.0p-53;
}
/* rng.hpp:36-41; *ctr is the stream counter, advanced in place */
uint64_t qo_next_below(uint64_t key, uint64_t* ctr, uint64_t n) {
  const uint64_t limit = ~(uint64_t)0 - ~(uint64_t)0 % n;
  uint64_t x = qo_draw_u64(key, ++*ctr);
  while (x >= limit) x = qo_draw_u64(key, ++*ctr);
  return x % n;
}
/* rng.hpp:44-49 */
double qo_next_gaussian(uint64_t key, uint64_t* ctr) {
  double u1 = qo_draw_double(key, ++*ctr);
  while (u1 <= 0.0) u1 = qo_draw_double(key, ++*ctr);
  const double u2 = qo_draw_double(key, ++*ctr);
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* -------------------------------------------------------------- quant ---- */
/* quant.hpp:16-18 */
uint64_t qo_packed_bytes(uint64_t count, int b) { return (count * (uint64_t)b + 7) / 8; }
static int valid_bits(int b) { return b == 2 || b == 4 || b == 8; }

/* quant.hpp:32-42 — LSB-first packing */
int qo_pack(const uint32_t* codes, uint64_t n, int b, uint8_t* out) {
  if (!valid_bits(b)) return QO_EINVAL;
  const uint32_t maxcode = (1u << b) - 1;
  memset(out, 0, qo_packed_bytes(n, b));
  for (uint64_t i = 0; i < n; ++i) {
    if (codes[i] > maxcode) return QO_EINVAL;
    const uint64_t bit = i * (uint64_t)b;
    out[bit / 8] |= (uint8_t)(codes[i] << (bit % 8));
  }
  return QO_OK;
}

/* quant.hpp:44-54 */
int qo_unpack(const uint8_t* bytes, int b, uint64_t n, uint32_t* codes) {
  if (!valid_bits(b)) return QO_EINVAL;
  const uint32_t mask = (1u << b) - 1;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bit = i * (uint64_t)b;
    codes[i] = (bytes[bit / 8] >> (bit % 8)) & mask;
  }
  return QO_OK;
}

/* quant.hpp:60-90 — stochastic quantize of one vector with stream `key`
 * (counter starts at 0; element i consumes draw i+1 when hi != lo). */
int qo_quantize(const double* h, uint64_t n, int b, uint64_t key, double* scale, double* zero,
                uint8_t* payload) {
  if (!valid_bits(b)) return QO_EINVAL;
  if (n == 0) return QO_EINVAL;
  double lo = h[0], hi = h[0];
  for (uint64_t i = 0; i < n; ++i) {
    if (!isfinite(h[i])) return QO_EINVAL;
    lo = h[i] < lo ? h[i] : lo; /* std::min(lo, x) keeps lo on ties */
    hi = hi < h[i] ? h[i] : hi; /* std::max(hi, x) */
  }
  *zero = lo;
  const uint32_t levels = (1u << b) - 1;
  const uint64_t nb = qo_packed_bytes(n, b);
  memset(payload, 0, nb);
  if (hi == lo) {
    *scale = 0.0;
    return QO_OK;
  }
  const double s = (hi - lo) / (double)levels;
  *scale = s;
  for (uint64_t i = 0; i < n; ++i) {
    const double x = (h[i] - lo) / s;
    double base = floor(x);
    const double frac = x - base;
    if (qo_draw_double(key, i + 1) < frac) base += 1.0;
    const double c = base < (double)levels ? base : (double)levels;
    const uint32_t code = (uint32_t)c;
    const uint64_t bit = i * (uint64_t)b;
    payload[bit / 8] |= (uint8_t)(code << (bit % 8));
  }
  return QO_OK;
}

/* quant.hpp:92-99 — mul then add, no contraction */
int qo_dequantize(const uint8_t* payload, int b, uint64_t n, double scale, double zero,
                  double* out) {
  if (!valid_bits(b)) return QO_EDECODE;
  const uint32_t mask = (1u << b) - 1;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t bit = i * (uint64_t)b;
    const uint32_t code = (payload[bit / 8] >> (bit % 8)) & mask;
    const double t = (double)code * scale;
    out[i] = t + zero;
  }
  return QO_OK;
}

/* quant.hpp:103-107 */
#define QO_CHUNK_HEADER 25
uint64_t qo_chunk_wire_bytes(uint64_t count, int b) { return QO_CHUNK_HEADER + qo_packed_bytes(count, b); }

/* quant.hpp:109-119 — little-endian header [u8 b][u64 count][f64 S][f64 Z] */
static void put_header(uint8_t* out, int b, uint64_t count, double s, double z) {
  out[0] = (uint8_t)b;
  memcpy(out + 1, &count, 8);
  memcpy(out + 9, &s, 8);
  memcpy(out + 17, &z, 8);
}

/* ------------------------------------------------------------- codec ---- */
/* codec.hpp:41-72.  Messages are rows of `values` (row stride ld) listed in
 * caller order by `rows`; ids[i] is message i's node id; bits[i] its width.
 * Writes the wire bytes to `out` (size from qo_encoded_size) and the
 * retrieval index in wire order: idx_pos[k] = caller position of the k-th
 * chunk, idx_off[k] = its byte offset. */
uint64_t qo_encoded_size(const int32_t* bits, uint64_t n, uint64_t dim) {
  uint64_t t = 0;
  for (uint64_t i = 0; i < n; ++i) t += qo_chunk_wire_bytes(dim, bits[i]);
  return t;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

int qo_encode_message_set(const double* values, uint64_t ld, const int64_t* rows,
                          const uint32_t* ids, const int32_t* bits, uint64_t n, uint64_t dim,
                          uint64_t set_key, uint8_t* out, int64_t* idx_pos, uint64_t* idx_off) {
  for (uint64_t i = 0; i < n; ++i)
    if (!valid_bits(bits[i])) return QO_EINVAL;
  uint32_t* sorted = (uint32_t*)malloc((n ? n : 1) * sizeof(uint32_t));
  memcpy(sorted, ids, n * sizeof(uint32_t));
  qsort(sorted, n, sizeof(uint32_t), cmp_u32);
  for (uint64_t i = 1; i < n; ++i)
    if (sorted[i] == sorted[i - 1]) {
      free(sorted);
      return QO_EINVAL;
    }
  free(sorted);
  uint64_t off = 0, k = 0;
  static const int widths[3] = {2, 4, 8};
  for (int wi = 0; wi < 3; ++wi) {
    const int b = widths[wi];
    for (uint64_t i = 0; i < n; ++i) {
      if (bits[i] != b) continue;
      double s, z;
      const uint64_t key = qo_fork(set_key, ids[i]);
      int st = qo_quantize(values + rows[i] * ld, dim, b, key, &s, &z, out + off + QO_CHUNK_HEADER);
      if (st) return st;
      put_header(out + off, b, dim, s, z);
      idx_pos[k] = (int64_t)i;
      idx_off[k] = off;
      ++k;
      off += qo_chunk_wire_bytes(dim, b);
    }
  }
  return QO_OK;
}

/* codec.hpp:80-96 + quant.hpp:121-134 — validates and dequantizes every
 * chunk; entry k (wire order) has expected (bits, dim, offset); output row k
 * of `out` (stride ld). */
int qo_decode_message_set(const uint8_t* bytes, uint64_t nbytes, const int32_t* e_bits,
                          const uint64_t* e_dim, const uint64_t* e_off, uint64_t n,
                          uint64_t total_bytes, double* out, uint64_t ld) {
  if (nbytes != total_bytes) return QO_EDECODE;
  uint64_t expect = 0;
  for (uint64_t k = 0; k < n; ++k) {
    if (e_off[k] != expect) return QO_EDECODE;
    const uint64_t o = e_off[k];
    if (o + QO_CHUNK_HEADER > nbytes) return QO_EDECODE;
    const int b = bytes[o];
    if (!valid_bits(b)) return QO_EDECODE;
    uint64_t count;
    double s, z;
    memcpy(&count, bytes + o + 1, 8);
    memcpy(&s, bytes + o + 9, 8);
    memcpy(&z, bytes + o + 17, 8);
    const uint64_t pb = qo_packed_bytes(count, b);
    if (o + QO_CHUNK_HEADER + pb > nbytes) return QO_EDECODE;
    if (b != e_bits[k] || count != e_dim[k]) return QO_EDECODE;
    qo_dequantize(bytes + o + QO_CHUNK_HEADER, b, count, s, z, out + k * ld);
    expect = o + qo_chunk_wire_bytes(count, b);
  }
  if (expect != nbytes) return QO_EDECODE;
  return QO_OK;
}

/* ---------------------------------------------------------- aggregate ---- */
/* tensorops/aggregate.hpp:94-119 — rows listed in `rows`; fp64 mul then add */
void qo_aggregate_rows(const double* self_alpha, const int64_t* local_ptr, const int32_t* local_row,
                       const double* local_alpha, const int64_t* remote_ptr,
                       const int32_t* remote_slot, const double* remote_alpha, const double* h,
                       const double* h_remote, uint64_t d, const int32_t* rows, uint64_t n_rows,
                       double* out) {
  for (uint64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows[k];
    double* dst = out + r * d;
    const double sa = self_alpha[r];
    for (uint64_t j = 0; j < d; ++j) dst[j] = sa * h[r * d + j];
    for (int64_t e = local_ptr[r]; e < local_ptr[r + 1]; ++e) {
      const double a = local_alpha[e];
      const double* src = h + (int64_t)local_row[e] * d;
      for (uint64_t j = 0; j < d; ++j) {
        const double t = a * src[j];
        dst[j] += t;
      }
    }
    if (remote_ptr)
      for (int64_t e = remote_ptr[r]; e < remote_ptr[r + 1]; ++e) {
        const double a = remote_alpha[e];
        const double* src = h_remote + (int64_t)remote_slot[e] * d;
        for (uint64_t j = 0; j < d; ++j) {
          const double t = a * src[j];
          dst[j] += t;
        }
      }
  }
}

/* aggregate.hpp:152-165 — partials[slot] += alpha * gbar[r], marginal rows ascending */
void qo_backward_remote_partials(const int64_t* remote_ptr, const int32_t* remote_slot,
                                 const double* remote_alpha, const int32_t* marginal_rows,
                                 uint64_t n_marginal, const double* gbar, uint64_t d,
                                 double* out /* num_remote x d, zeroed by caller */) {
  for (uint64_t k = 0; k < n_marginal; ++k) {
    const int64_t r = marginal_rows[k];
    const double* src = gbar + r * d;
    for (int64_t e = remote_ptr[r]; e < remote_ptr[r + 1]; ++e) {
      const double a = remote_alpha[e];
      double* dst = out + (int64_t)remote_slot[e] * d;
      for (uint64_t j = 0; j < d; ++j) {
        const double t = a * src[j];
        dst[j] += t;
      }
    }
  }
}

/* -------------------------------------------------------------- dense ---- */
/* tensorops/model.hpp:90-124 (no layer norm / dropout): z = h W, skipping
 * zero h entries, then ReLU when relu != 0.  pre_act may be NULL. */
void qo_layer_forward_rows(const double* h_agg, const double* w, uint64_t din, uint64_t dout,
                           const int32_t* rows, uint64_t n_rows, int relu, double* pre_act,
                           double* out) {
  double* z = (double*)malloc(dout * sizeof(double));
  for (uint64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows[k];
    for (uint64_t j = 0; j < dout; ++j) z[j] = 0.0;
    for (uint64_t i = 0; i < din; ++i) {
      const double hi = h_agg[r * din + i];
      if (hi == 0.0) continue;
      for (uint64_t j = 0; j < dout; ++j) {
        const double t = hi * w[i * dout + j];
        z[j] += t;
      }
    }
    for (uint64_t j = 0; j < dout; ++j) {
      if (pre_act) pre_act[r * dout + j] = z[j];
      out[r * dout + j] = relu ? (z[j] > 0.0 ? z[j] : 0.0) : z[j];
    }
  }
  free(z);
}

/* model.hpp:128-153 (ReLU branch) — dz = dh masked by act_in <= 0 */
void qo_layer_backward_rows(const double* act_in, const double* dh, uint64_t dout,
                            const int32_t* rows, uint64_t n_rows, int relu, double* dz) {
  for (uint64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows[k];
    for (uint64_t j = 0; j < dout; ++j) {
      double v = dh[r * dout + j];
      if (relu && act_in[r * dout + j] <= 0.0) v = 0.0;
      dz[r * dout + j] = v;
    }
  }
}

/* model.hpp:156-170 — dh_agg = dz W^T */
void qo_input_grad_rows(const double* dz, const double* w, uint64_t din, uint64_t dout,
                        const int32_t* rows, uint64_t n_rows, double* dh_agg) {
  for (uint64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows[k];
    for (uint64_t i = 0; i < din; ++i) {
      double acc = 0.0;
      for (uint64_t j = 0; j < dout; ++j) {
        const double t = dz[r * dout + j] * w[i * dout + j];
        acc += t;
      }
      dh_agg[r * din + i] = acc;
    }
  }
}

/* tensorops/matrix.hpp:51-65 — out[m x n] = a[k x m]^T b[k x n] */
void qo_matmul_transa(const double* a, const double* b, uint64_t k, uint64_t m, uint64_t n,
                      double* out) {
  memset(out, 0, m * n * sizeof(double));
  for (uint64_t kk = 0; kk < k; ++kk) {
    for (uint64_t i = 0; i < m; ++i) {
      const double aki = a[kk * m + i];
      if (aki == 0.0) continue;
      for (uint64_t j = 0; j < n; ++j) {
        const double t = aki * b[kk * n + j];
        out[i * n + j] += t;
      }
    }
  }
}

/* model.hpp:175-200 — masked softmax CE partial; returns loss sum, grad rows */
double qo_masked_ce_partial(const double* logits, uint64_t c, const int32_t* labels,
                            const int32_t* rows, uint64_t n_rows, double inv_denom, double* grad) {
  double loss = 0.0;
  for (uint64_t k = 0; k < n_rows; ++k) {
    const int64_t r = rows[k];
    const double* row = logits + r * c;
    double hi = row[0];
    for (uint64_t j = 1; j < c; ++j) hi = hi < row[j] ? row[j] : hi;
    double sum = 0.0;
    for (uint64_t j = 0; j < c; ++j) sum += exp(row[j] - hi);
    const double lse = hi + log(sum);
    loss += (lse - row[labels[r]]) * inv_denom;
    for (uint64_t j = 0; j < c; ++j)
      grad[r * c + j] = (exp(row[j] - lse) - ((int64_t)j == labels[r] ? 1.0 : 0.0)) * inv_denom;
  }
  return loss;
}

/* optim.hpp:47-62 — one Adam step over a flat parameter array; t is the new step count */
void qo_adam_step(double* p, double* m, double* v, const double* g, uint64_t n, uint64_t t,
                  double lr, double b1, double b2, double eps) {
  const double bc1 = 1.0 - pow(b1, (double)t);
  const double bc2 = 1.0 - pow(b2, (double)t);
  for (uint64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + (1.0 - b1) * g[i];
    v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
    const double mhat = m[i] / bc1;
    const double vhat = v[i] / bc2;
    p[i] -= lr * mhat / (sqrt(vhat) + eps);
  }
}

/* graphcore/coeffs.hpp:30-45 */
void qo_compute_coeffs(const int64_t* adj_ptr, const int32_t* adj, uint64_t n, int sage,
                       double* alpha, double* self_alpha) {
  for (uint64_t v = 0; v < n; ++v) {
    const double dv1 = (double)(adj_ptr[v + 1] - adj_ptr[v]) + 1.0;
    self_alpha[v] = 1.0 / dv1;
    for (int64_t i = adj_ptr[v]; i < adj_ptr[v + 1]; ++i) {
      const int64_t u = adj[i];
      const double du1 = (double)(adj_ptr[u + 1] - adj_ptr[u]) + 1.0;
      alpha[i] = sage ? 1.0 / dv1 : 1.0 / sqrt(du1 * dv1);
    }
  }
}
