/*
 * qgnn_b200.h — C-ABI of the B200-native AdaQP boundary-message path.
 *
 * The reference (qgnn, /root/reference/proj) has no FFI: its operator API is
 * a set of inline C++ functions called by trainer/engine.hpp.  Each entry
 * point below replaces one of them; the citation names the function and
 * file:line (relative to proj/include/qgnn/).  All signatures are plain C:
 * pointers, sizes, enums.  Device pointers are marked [dev]; everything is
 * asynchronous on the caller's cudaStream_t (passed as void*), and
 * device-detected errors (non-finite input, corrupt chunk) are latched in the
 * context's error word and reported by qgnn_ctx_check() at the phase
 * boundary, mapped onto the reference's exception taxonomy below.
 *
 * There is no CPU fallback: every compute entry point launches sm_100a
 * kernels and fails with QGNN_ECUDA when no device is present.
 */
#ifndef QGNN_B200_H
#define QGNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: common/errors.hpp:8-36 --------------------------------- */
enum {
  QGNN_OK = 0,
  QGNN_EINVAL = 1,    /* std::invalid_argument (bad width, empty, non-finite, shape) */
  QGNN_EDECODE = 2,   /* DecodeError (corrupt chunk / index mismatch) */
  QGNN_EPROTOCOL = 3, /* ProtocolError (routing, plan version, buffer size) */
  QGNN_ERESOURCE = 4, /* ResourceLimitError (brute-force solver limit) */
  QGNN_EDIVERGED = 5, /* DivergedError (non-finite loss) */
  QGNN_EIO = 6,       /* IoError */
  QGNN_ECUDA = 7,     /* CUDA runtime failure / no device */
  QGNN_ENCCL = 8      /* NCCL failure */
};

enum { QGNN_F32 = 0, QGNN_F64 = 1 };            /* element type of a dense buffer */
enum { QGNN_WIRE_GPU = 0, QGNN_WIRE_REF = 1 };  /* chunk layout, see qgnn_chunk_wire_bytes */

/* Message of the last failing call on this thread. */
const char* qgnn_last_error(void);
const char* qgnn_version(void);

/* ---- context ---------------------------------------------------------------- */
typedef struct qgnn_ctx qgnn_ctx;
/* Binds `device`, allocates the device error word and split-K scratch. */
int qgnn_ctx_create(int device, qgnn_ctx** out);
int qgnn_ctx_destroy(qgnn_ctx* ctx);
/* Synchronizes `stream`, reads and clears the device error word; returns the
 * status of the first latched error (QGNN_EINVAL for non-finite quantize input,
 * QGNN_EDECODE for a corrupt chunk) or QGNN_OK. */
int qgnn_ctx_check(qgnn_ctx* ctx, void* stream);

/* ---- RngStream: quantcodec/rng.hpp:13-61 ------------------------------------- */
uint64_t qgnn_rng_seed_key(uint64_t seed);               /* RngStream(seed) key, rng.hpp:15 */
uint64_t qgnn_rng_fork(uint64_t key, uint64_t coord);    /* fork(coord) key, rng.hpp:17-22 */
uint64_t qgnn_rng_u64(uint64_t key, uint64_t counter);   /* next_u64 at counter, rng.hpp:30 */

/* ---- sizes: quant.hpp:16-18, 103-107; plan.hpp:90-100 ------------------------ */
uint64_t qgnn_packed_bytes(uint64_t count, int bits);
/* QGNN_WIRE_REF: 25 + ceil(count*bits/8)  (byte-identical to append_chunk).
 * QGNN_WIRE_GPU: 16-byte header {f32 scale, f32 zero, u32 count, u8 bits, 3 pad}
 *                + payload padded to a 16-byte multiple.
 * bits == 0 denotes a raw full-precision row (BitMode::kFp): count * elem bytes
 * (QGNN_WIRE_GPU pads it to a 16-byte multiple so every chunk stays 16-aligned). */
uint64_t qgnn_chunk_wire_bytes(uint64_t count, int bits, int layout, int dtype);

/* encode_message_set's wire order (codec.hpp:56-69): width groups 2,4,8, caller
 * order inside each.  Host helper.  wire_pos[k] = caller index of chunk k;
 * offsets[i] = byte offset of caller message i; *total = set bytes. */
int qgnn_wire_layout(const int32_t* bits, int64_t n, int64_t dim, int layout, int dtype,
                     int64_t* wire_pos, uint64_t* offsets, uint64_t* total);

/* ---- K1 quantize + pack: quant.hpp:60-90 via codec.hpp:41-72 ------------------
 * Message i quantizes row rows[i] of `values` (dtype, row stride ld, dim
 * columns) at width bits[i] with RNG stream fork(set_keys[set_of[i]], ids[i])
 * and writes its chunk at out + offsets[i].  bits[i] == 0 copies the raw row
 * (fp mode, engine.hpp:473-481).  win_lo/win_hi (optional, dtype, [n]) fold
 * the row extrema into the message's trace window (trace.hpp:86-91).
 * set_of == NULL means every message belongs to set 0.  [dev] for all arrays.
 * envelope (QGNN_WIRE_GPU): source id | plan version << 8 (each mod 256); the
 * chunk header records (source, set index = destination, version) — the
 * routing fields of the reference's ExchangePayload (engine.hpp:530-541). */
int qgnn_quantize_pack(qgnn_ctx* ctx, const void* values, int dtype, int64_t ld, int64_t dim,
                       int64_t n, const int32_t* rows, const uint32_t* ids, const uint8_t* bits,
                       const uint64_t* offsets, const uint16_t* set_of, const uint64_t* set_keys,
                       int layout, uint8_t* out, void* win_lo, void* win_hi, uint32_t envelope,
                       void* stream);

/* decode_message_set's index checks (codec.hpp:82-95), host side: the n
 * entries in wire order (bits[k], offsets[k], dims[k]) must tile [0, n_bytes)
 * contiguously with qgnn_chunk_wire_bytes each and total_bytes == n_bytes.
 * Fails with QGNN_EDECODE and the reference's message ("message set: byte
 * count mismatch", "... index offsets not contiguous", "chunk: truncated
 * payload", "message set: trailing bytes").  The per-chunk width / count check
 * against the index runs on the device in K3. */
int qgnn_decode_validate(const uint8_t* bits, const uint64_t* offsets, const uint64_t* dims,
                         int64_t n, int layout, int dtype, uint64_t total_bytes,
                         uint64_t n_bytes);

/* ---- K3 unpack + dequantize + scatter: quant.hpp:92-99, codec.hpp:80-96 --------
 * Decodes message i's chunk at in + offsets[i] (validating width and count
 * against bits[i] / dim — DecodeError semantics) and stores (accumulate == 0,
 * engine.hpp:607-618) or adds (accumulate == 1, engine.hpp:729-733) the values
 * into row dst_rows[i] of `out` (dst_rows == NULL: row i).  expect_envelope
 * (optional [dev] [n], QGNN_WIRE_GPU): source | destination << 8 | plan
 * version << 16 expected of each chunk; a mismatch is latched as QGNN_EPROTOCOL
 * ("misrouted payload" / "plan version skew", engine.hpp:530-541). */
int qgnn_dequant_scatter(qgnn_ctx* ctx, const uint8_t* in, int64_t n, int64_t dim,
                         const uint8_t* bits, const uint64_t* offsets, int layout,
                         const int32_t* dst_rows, int accumulate, void* out, int dtype,
                         int64_t ld, const uint32_t* expect_envelope, void* stream);

/* ---- K4 CSR aggregation: aggregate.hpp:94-165 ----------------------------------
 * For each listed row r (rows != NULL: rows[k]; else row_begin + k):
 *   out[r] = self_alpha[r] * x[r]                    (self_alpha may be NULL -> 0)
 *          + sum_{e in [ptr_a[r], ptr_a[r+1])} alpha_a[e] * x[col_a[e]]
 *          + sum_{e in [ptr_b[r], ptr_b[r+1])} alpha_b[e] * y[col_b[e]]   (ptr_b may be NULL)
 * in that order.  aggregate_rows = (self, local CSR over h, remote CSR over
 * the halo); aggregate_backward_local = (self, local CSR with alpha_bwd);
 * backward_remote_partials = (no self, slot->marginal-row transpose CSR).
 * F64 reproduces the reference's mul-then-add order bit for bit; F32 uses FMA. */
int qgnn_csr_aggregate(qgnn_ctx* ctx, int dtype, int64_t dim, const void* x, int64_t ld_x,
                       const void* y, int64_t ld_y, const void* self_alpha, const int64_t* ptr_a,
                       const int32_t* col_a, const void* alpha_a, const int64_t* ptr_b,
                       const int32_t* col_b, const void* alpha_b, const int32_t* rows,
                       int64_t row_begin, int64_t n_rows, void* out, int64_t ld_out, void* stream);

/* Production fp32 K4 for one CSR row range — the kernels the engine runs at
 * scale (spmm.cu: 256-wide, grouped <= 128-wide and degree-sorted <= 64-wide
 * row kernels, hub rows split into 256-edge segments and reduced in segment
 * order inside the launch).  The plan is built once per (CSR, row range) on
 * the host from HOST copies of ptr_a / ptr_b (rows [row_begin, row_begin +
 * n_rows)); rows with more than hub_deg neighbours become hub segments;
 * max_dim bounds `dim` of later runs.  A run computes the same sum as
 * qgnn_csr_aggregate (F32, fused multiply-add) with [dev] arrays; x / y /
 * out / mask rows must be 16-byte aligned with ld a multiple of 4 and the
 * columns in [dim, round_up(dim, 4)) zero.  mask != NULL applies the ReLU
 * backward (layer_backward_rows, model.hpp:128-153) to the result:
 * out[r][c] = mask[r][c] > 0 ? sum : 0. */
typedef struct qgnn_spmm_plan qgnn_spmm_plan;
int qgnn_spmm_plan_create(qgnn_ctx* ctx, const int64_t* ptr_a, const int64_t* ptr_b,
                          int64_t row_begin, int64_t n_rows, int64_t max_dim, int64_t hub_deg,
                          qgnn_spmm_plan** out);
int qgnn_spmm_plan_run(qgnn_spmm_plan* plan, int64_t dim, const float* x, int64_t ld_x,
                       const float* y, int64_t ld_y, const float* self_alpha,
                       const int64_t* ptr_a, const int32_t* col_a, const float* alpha_a,
                       const int64_t* ptr_b, const int32_t* col_b, const float* alpha_b,
                       const float* mask, int64_t ld_mask, float* out, int64_t ld_out,
                       void* stream);
int qgnn_spmm_plan_destroy(qgnn_spmm_plan* plan);

/* ---- K5 dense transform: model.hpp:90-170, matrix.hpp:51-65 --------------------
 * forward:      out[r] = act(A[r] W)            W: din x dout row-major (layer_forward_rows)
 * input grad:   out[r] = A[r] W^T               (input_grad_rows)
 * weight grad:  out (+)= A[rows]^T B[rows]      (matmul_transa; deterministic split-K) */
int qgnn_dense_forward(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* W,
                       int64_t din, int64_t dout, const int32_t* rows, int64_t row_begin,
                       int64_t n_rows, int relu, void* out, int64_t ld_out, void* stream);
int qgnn_dense_input_grad(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* W,
                          int64_t din, int64_t dout, const int32_t* rows, int64_t row_begin,
                          int64_t n_rows, void* out, int64_t ld_out, void* stream);
int qgnn_dense_weight_grad(qgnn_ctx* ctx, int dtype, const void* A, int64_t lda, const void* B,
                           int64_t ldb, int64_t m, int64_t n, const int32_t* rows,
                           int64_t row_begin, int64_t n_rows, int accumulate, void* out,
                           void* stream);
/* layer_backward_rows (model.hpp:128-153), ReLU only: dz = act > 0 ? dh : 0 */
int qgnn_relu_backward(qgnn_ctx* ctx, int dtype, const void* act, int64_t ld_act, const void* dh,
                       int64_t ld_dh, int64_t dim, int64_t row_begin, int64_t n_rows, void* dz,
                       int64_t ld_dz, void* stream);
/* masked_ce_partial (model.hpp:175-200) + count_correct (:216-227): writes grad
 * rows of the listed rows, adds the scaled loss into *loss_acc [dev, f64] and
 * argmax hits of the rows in correct_rows into *correct_acc [dev, u64]. */
int qgnn_masked_ce(qgnn_ctx* ctx, int dtype, const void* logits, int64_t ld, int64_t classes,
                   const int32_t* labels, const int32_t* rows, int64_t n_rows, double inv_denom,
                   void* grad, int64_t ld_grad, double* loss_acc, void* stream);
int qgnn_count_correct(qgnn_ctx* ctx, int dtype, const void* logits, int64_t ld, int64_t classes,
                       const int32_t* labels, const int32_t* rows, int64_t n_rows,
                       unsigned long long* correct_acc, void* stream);
/* optimizer_step Adam branch (optim.hpp:47-62); bc1/bc2 = 1 - beta^t from the host. */
int qgnn_adam_step(qgnn_ctx* ctx, int dtype, void* p, void* m, void* v, const void* g, int64_t n,
                   double lr, double beta1, double beta2, double eps, double bc1, double bc2,
                   void* stream);

/* ---- host: graph / partition / coefficients (graphcore/{partition,coeffs}.hpp) ------------------ */
/* partition_graph (partition.hpp:90-135): seeded BFS region growing -> owner[n]. */
int qgnn_partition_graph(const int64_t* adj_ptr, const int32_t* adj, int64_t n, int64_t n_parts,
                         uint64_t seed, uint32_t* owner);
/* compute_coeffs (coeffs.hpp:30-45): alpha per CSR slot + self alpha (f64). */
int qgnn_compute_coeffs(const int64_t* adj_ptr, const int32_t* adj, int64_t n, int sage,
                        double* alpha, double* self_alpha);
/* Exchange schedule of one tensor key for `rank` of `world` GPUs hosting
 * partitions [rank * P / world, (rank + 1) * P / world) — replaces the
 * reference's pair_wire_bytes / negotiate_buffers (assigner/plan.hpp:90-154)
 * for a uniform width `bits` (0 = raw rows): send_bytes[world] / recv_bytes[world]
 * = bytes this rank sends to / receives from each rank (same-rank pairs are
 * zero-copy, 0).  bwd selects the backward partial-gradient direction. */
int qgnn_exchange_plan(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                       const uint32_t* owner, int64_t n_parts, int world, int rank, int64_t dim,
                       int bits, int bwd, int layout, int dtype, uint64_t* send_bytes,
                       uint64_t* recv_bytes);

/* partitions_from_owner (partition.hpp:39-84): one handle per device p in
 * out[0..n_parts).  Lists (QGNN_PART_*) are ascending node ids exactly as the
 * reference's Partition: owned / central / marginal, remote_in[q] (nodes owned
 * by q that p consumes), remote_out[q] (owned nodes q consumes).  Any n_parts. */
typedef struct qgnn_partition qgnn_partition;
enum { QGNN_PART_OWNED = 0, QGNN_PART_CENTRAL = 1, QGNN_PART_MARGINAL = 2,
       QGNN_PART_REMOTE_IN = 3, QGNN_PART_REMOTE_OUT = 4 };
int qgnn_partitions_from_owner(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                               const uint32_t* owner, int64_t n_parts, qgnn_partition** out);
/* *ids stays valid until qgnn_partition_destroy; q is used by REMOTE_IN/OUT. */
int qgnn_partition_list(const qgnn_partition* part, int which, int64_t q, const uint32_t** ids,
                        int64_t* len);
int qgnn_partition_destroy(qgnn_partition* part);

/* DeviceAggView::build (tensorops/aggregate.hpp:41-89) with compute_coeffs
 * (coeffs.hpp:30-45; sage = AggMode::kSageMean) for partition `part` of the
 * owner map: the reference's row order (owned ascending) and slot order
 * (remote_in by ascending source, ids ascending).  The GPU engine uses its own
 * central-first layout of the same view internally. */
typedef struct qgnn_agg_view qgnn_agg_view;
typedef struct {
  int64_t num_owned, num_remote, local_nnz, remote_nnz, n_parts, n_central, n_marginal;
  const double* self_alpha;                    /* [num_owned] */
  const int64_t* local_ptr;                    /* [num_owned + 1] */
  const uint32_t* local_row;                   /* [local_nnz] owned-row index */
  const double* local_alpha_fwd;               /* [local_nnz] */
  const double* local_alpha_bwd;               /* [local_nnz] */
  const int64_t* remote_ptr;                   /* [num_owned + 1] */
  const uint32_t* remote_slot;                 /* [remote_nnz] */
  const double* remote_alpha;                  /* [remote_nnz] */
  const uint32_t* slot_node;                   /* [num_remote] */
  const uint32_t* slot_owner;                  /* [num_remote] */
  const int64_t* device_slot_offset;           /* [n_parts + 1] */
  const uint32_t* central_rows;                /* [n_central] */
  const uint32_t* marginal_rows;               /* [n_marginal] */
} qgnn_agg_view_arrays;
int qgnn_agg_view_build(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                        const uint32_t* owner, const qgnn_partition* part, int sage,
                        qgnn_agg_view** out);
int qgnn_agg_view_arrays_get(const qgnn_agg_view* view, qgnn_agg_view_arrays* out);
int qgnn_agg_view_destroy(qgnn_agg_view* view);

/* GPU-side setup: the same two builders computed on `device`
 * from a device-resident copy of the graph — per-node consumer sets and every
 * per-edge pass (local/remote split with the fp64 coefficients, remote-CSR
 * transpose) run as kernels; outputs are identical to qgnn_partitions_from_owner /
 * qgnn_agg_view_build (same handles, same accessors, same destroy calls). */
int qgnn_partitions_from_owner_gpu(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                                   const uint32_t* owner, int64_t n_parts, int device,
                                   qgnn_partition** out);
int qgnn_agg_view_build_gpu(const int64_t* adj_ptr, const int32_t* adj, int64_t n,
                            const uint32_t* owner, const qgnn_partition* part, int sage,
                            int device, qgnn_agg_view** out);

/* load_dataset (cli/synth.hpp:184-205) of a dataset directory written by the
 * reference's save_dataset (edges.txt, features.bin, labels.txt,
 * {train,val,test}_mask.txt, meta.json; formats graph.hpp:80-200).  The edge list
 * is parsed on host threads and build_graph's symmetric, deduplicated, sorted CSR
 * (graph.hpp:59-78) is built on `device` (radix sort of the directed pairs; device
 * < 0: on the host).  features = the stored f64 matrix, features_f32 = the same
 * rounded to fp32 (the production engine's input).  Errors: QGNN_EIO (IoError,
 * same messages), QGNN_EINVAL (edge endpoint out of range, overlapping masks). */
typedef struct qgnn_dataset qgnn_dataset;
typedef struct {
  int64_t nodes, nnz, feature_dim, classes;
  const int64_t* adj_ptr;       /* [nodes + 1] */
  const int32_t* adj;           /* [nnz] */
  const double* features;       /* [nodes x feature_dim] as stored */
  const float* features_f32;    /* [nodes x feature_dim] */
  const int32_t* labels;        /* [nodes] */
  const uint8_t* train;         /* [nodes] */
  const uint8_t* val;
  const uint8_t* test;
} qgnn_dataset_arrays;
int qgnn_dataset_load(const char* dir, int device, qgnn_dataset** out);
int qgnn_dataset_arrays_get(const qgnn_dataset* d, qgnn_dataset_arrays* out);
int qgnn_dataset_destroy(qgnn_dataset* d);

/* BitWidthPlan::Lookup::bits_for (assigner/plan.hpp:60-72) over one
 * (key, src, dst) entry list (ids ascending, bits parallel): out[k] = bits of
 * query[k]; an unknown id fails with QGNN_EINVAL "plan: unknown message id". */
int qgnn_plan_bits_for(const uint32_t* ids, const int32_t* bits, int64_t n,
                       const uint32_t* query, int64_t n_query, int32_t* out);

/* ---- K2 exchange: ring_all2all / comm_seconds (commsim/exchange.hpp:45-78,
 * trainer/engine.hpp:507-522) and the mailbox send / take (engine.hpp:502,
 * :528-529) ------------------------------------------------------------------
 * One rank of a group of `world` ranks.  id128 = qgnn_nccl_unique_id (NCCL
 * over NVLink / NVSwitch; NULL allowed for world == 1) or qgnn_loopback_id
 * (ranks as threads of one process on one device: tests). */
typedef struct qgnn_comm qgnn_comm;
int qgnn_comm_create(const void* id128, int world, int rank, int device, qgnn_comm** out);
int qgnn_comm_destroy(qgnn_comm* comm);
/* Irregular all-to-all of packed payloads in one grouped send/receive: this
 * rank sends send_bytes[r] bytes from send + send_off[r] to rank r and
 * receives recv_bytes[r] bytes into recv + recv_off[r] (host arrays [world];
 * [dev] buffers; r == rank is a device copy).  Sizes come from
 * qgnn_exchange_plan, so both sides agree without a handshake
 * (negotiate_buffers, plan.hpp:140-154); the loopback transport checks the
 * agreement and fails with QGNN_EPROTOCOL like engine.hpp:546-550.
 * Asynchronous on `stream`. */
int qgnn_exchange(qgnn_comm* comm, const void* send, const uint64_t* send_off,
                  const uint64_t* send_bytes, void* recv, const uint64_t* recv_off,
                  const uint64_t* recv_bytes, void* stream);

/* ---- host: assigner (assigner/solve.hpp) ---------------------------------------
 * One instance = one tensor key across device pairs.  Messages are flat,
 * grouped by pair: pair p has pair_count[p] messages (id, dim, lo, hi,
 * sum_alpha_sq).  Runs group_and_order (solve.hpp:24-52) then the exact
 * solve_assignment (solve.hpp:264-309), or brute_force_assignment
 * (solve.hpp:220-258) when brute != 0; writes per-message bits (input order)
 * and eval = {objective, variance_term, z_seconds}. */
int qgnn_solve_instance(int64_t n_pairs, const uint32_t* pair_src, const uint32_t* pair_dst,
                        const uint64_t* pair_count, const uint32_t* m_id, const uint64_t* m_dim,
                        const double* m_lo, const double* m_hi, const double* m_asq,
                        int64_t n_devices, const double* theta, const double* gamma,
                        double lambda, int64_t group_size, int brute, int32_t* out_bits,
                        double* eval);
/* fit_cost_model (cost_model.hpp:78-109) for one pair: least squares on
 * (bits, seconds) samples with clamp-to-zero. */
int qgnn_fit_affine(const double* bits, const double* seconds, int64_t n, double* theta,
                    double* gamma);

/* ---- engine: trainer/engine.hpp:95-884 ------------------------------------------ */
typedef struct qgnn_engine qgnn_engine;

typedef struct {
  int32_t sage;            /* AggMode: 0 GCN, 1 SAGE-mean */
  int32_t n_dims;          /* dims = feature, hidden..., classes */
  int64_t dims[8];
  int32_t bit_mode;        /* BitMode: 0 fp, 1 fixed, 2 uniform, 3 adaptive */
  int32_t fixed_bits;
  double lambda;
  int64_t group_size;
  int64_t period;
  uint64_t seed;
  int64_t n_parts;         /* simulated devices = graph partitions (all ranks) */
  double lr;
  double theta, gamma;     /* uniform affine cost model (CostModel::uniform) */
  int32_t dtype;           /* QGNN_F32 production, QGNN_F64 reference-order parity */
  int32_t layout;          /* QGNN_WIRE_GPU or QGNN_WIRE_REF */
  int32_t rank, world;     /* process rank / count; parts are split contiguously */
  int32_t device;          /* CUDA device of this rank */
  int32_t overlap;         /* 0: the compute stream waits for each exchange before the
                              central rows (serialized); 1 (default): central SpMM + GEMM
                              overlap the exchange on the comm stream; 2: one GPU, K1/K3
                              also on a side stream next to the central rows */
  int32_t kstats;          /* 1: time every kernel class with CUDA events (bench roofline) */
  int32_t transport;       /* world == 1: 0 zero copy between the partitions of the GPU
                              (default); 1 every pair through NCCL self send/receive (the
                              multi-GPU exchange path, run and timed on one device).
                              world > 1: 0 grouped NCCL send/receive (default); 2 peer
                              store — K1 writes each remote pair's chunks straight into
                              the receiver's arena (CUDA IPC / peer memory over NVLink),
                              ordered by ready / consumed flags, no exchange copies */
  int32_t layer_norm;      /* TrainSettings::layer_norm (engine.hpp:42): LN after every
                              layer's transform (model.hpp:62-73, 108-112) */
  double dropout;          /* TrainSettings::dropout (engine.hpp:43): inverted dropout on
                              the hidden layers' outputs (model.hpp:114-119) */
} qgnn_settings;

typedef struct {
  uint64_t epoch;
  double train_loss, val_acc, test_acc;
  uint64_t bytes_total;      /* actual wire bytes this epoch (all pairs) */
  uint64_t ref_bytes_total;  /* reference-layout-equivalent bytes (25 + ceil(Db/8)) */
  uint64_t msgs_b2, msgs_b4, msgs_b8, msgs_fp;
  uint64_t plan_version;
  double ms_total;           /* device time of the epoch (CUDA events) */
  /* per kernel class, this epoch (settings.kstats = 1; 0 otherwise): K1 quantize,
   * exchange (comm stream), K3 dequantize, K4 SpMM (all variants), K5 GEMMs,
   * everything else (ReLU, loss, all-gather sum + Adam) */
  double ms_quant, ms_exchange, ms_dequant, ms_spmm, ms_gemm, ms_other;
  double resolve_seconds;    /* host solver time if a re-solve ran */
} qgnn_epoch_metrics;

/* Graph: symmetric sorted CSR without self loops (graph.hpp:20-56) + node
 * features (f32 or f64 per settings dtype, n x dims[0]), labels and masks.
 * owner == NULL partitions with partition_graph(g, n_parts, seed) like the
 * reference engine (engine.hpp:212); otherwise partitions_from_owner. */
int qgnn_engine_create(const qgnn_settings* s, int64_t n_nodes, const int64_t* adj_ptr,
                       const int32_t* adj, const void* features, const int32_t* labels,
                       const uint8_t* train, const uint8_t* val, const uint8_t* test,
                       const uint32_t* owner, const void* nccl_unique_id, qgnn_engine** out);
int qgnn_engine_destroy(qgnn_engine* e);
/* One epoch (run_epoch, engine.hpp:384-426). */
int qgnn_engine_run_epoch(qgnn_engine* e, qgnn_epoch_metrics* out);
/* run_epoch split in two: launch enqueues the epoch on the engine's streams and
 * returns; finish waits for it and fills the metrics (loss / accuracy read
 * back).  In between the caller may stage the next epoch's inputs with
 * qgnn_engine_set_features (the copy overlaps the running epoch).  Weights
 * cannot be read or written while an epoch is in flight (QGNN_EPROTOCOL). */
int qgnn_engine_launch_epoch(qgnn_engine* e);
int qgnn_engine_finish_epoch(qgnn_engine* e, qgnn_epoch_metrics* out);
/* Re-upload node features (n_nodes x F, f32/f64, node order).  From pinned
 * (or device) memory the copy is asynchronous: node-range chunks stream in on a
 * copy stream and the next run_epoch gathers each partition as soon as its
 * chunk has landed, overlapping the upload with the first layer; `features`
 * must stay valid until that run_epoch returns.  From pageable memory the call
 * stages through pinned memory and returns after the upload. */
int qgnn_engine_set_features(qgnn_engine* e, const void* features);
/* Weights of layer l (din x dout, settings dtype) to host memory. */
int qgnn_engine_get_weights(qgnn_engine* e, int layer, void* out);
int qgnn_engine_set_weights(qgnn_engine* e, int layer, const void* in);
/* Facts: [fwd messages per tensor (all pairs), n_parts, parts_on_rank, max_owned,
 * max_halo, kernels of ours launched in the last epoch]. */
int qgnn_engine_info(qgnn_engine* e, int64_t* out6);
/* Per kernel class k (QGNN_K_*), accumulated since the last call (needs
 * settings.kstats): out[3k] = total device ms, out[3k+1] = launches,
 * out[3k+2] = algorithmic bytes (SURVEY.md §8d model).  With n >= 4 *
 * QGNN_K_COUNT the layout is 4 per class and out[4k+3] = gathered row bytes of
 * the SpMM classes (nnz x dim x elem, the L2 gather model).  Returns the
 * number of classes written. */
enum {
  QGNN_K_QUANT = 0, QGNN_K_DEQUANT, QGNN_K_SPMM_FWD, QGNN_K_SPMM_BWD, QGNN_K_PARTIALS,
  QGNN_K_GEMM_FWD, QGNN_K_GEMM_DGRAD, QGNN_K_GEMM_WGRAD, QGNN_K_ELEMWISE, QGNN_K_EXCHANGE,
  QGNN_K_COUNT
};
int qgnn_engine_kernel_stats(qgnn_engine* e, double* out, int n);
/* Switch per-kernel event timing on/off between epochs.  With it off (and one
 * GPU, fixed/adaptive widths) the steady-state epoch runs as one captured CUDA
 * graph, re-captured when the plan or a workspace changes; with it on every
 * kernel is launched eagerly between timing events. */
int qgnn_engine_set_kstats(qgnn_engine* e, int on);

/* NCCL bootstrap for world > 1: rank 0 creates the id, every rank passes it to
 * qgnn_engine_create.  128 bytes. */
int qgnn_nccl_unique_id(void* out128);
/* In-process loopback transport (tests, one device): every rank of `group` runs
 * its engine in its own host thread of one process and passes this id instead
 * of an NCCL id; exchanges and all-gathers become device copies between the
 * ranks' buffers over the same routing as the NCCL path (the analogue of the
 * reference's in-process mailbox, engine.hpp:331,502,528-529). */
int qgnn_loopback_id(uint64_t group, void* out128);

#ifdef __cplusplus
}
#endif
#endif /* QGNN_B200_H */
