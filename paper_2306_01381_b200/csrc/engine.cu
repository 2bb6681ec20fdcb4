// engine.cu — the GPU engine: the reference's per-epoch phase schedule
// (trainer/engine.hpp:384-426) over partitions resident in HBM.
//
// One process per GPU hosts a contiguous range of the P graph partitions
// ("devices" in the reference).  Per layer and direction the boundary path is
//   K1 quantize+pack (all destinations of a partition in one launch)
//   -> exchange: partitions on the same GPU are zero-copy (the receiver's
//      decode reads the sender's send region in place); partitions on other
//      GPUs move through grouped ncclSend/ncclRecv on a dedicated stream
//   || central-row SpMM + GEMM on the compute stream (overlaps the exchange)
//   -> K3 dequant+scatter into the halo (fwd) / accumulate into dh (bwd)
//   -> marginal-row SpMM + GEMM.
// Central rows are laid out first in every partition, so the central and
// marginal subsets are contiguous row ranges for SpMM/GEMM.  Per-message
// metadata (source row, id, bit width, wire offset) is built on the host per
// plan version and uploaded once; RNG stream keys are uploaded per epoch.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <condition_variable>
#include <future>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <thread>
#include <vector>

#include "common.cuh"
#include "dbuf.cuh"
#include "host.hpp"
#include "setup.cuh"
#include "rng.cuh"

namespace qgnn_b200 {

// ------------------------------------------------------------------ NCCL ---
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  if (api.h) return api;
  // prefer the NCCL already loaded into the process (torch's), else the system one
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  QGNN_REQUIRE(h, QGNN_ENCCL, "cannot load libnccl.so.2");
  auto sym = [&](const char* n) {
    void* p = dlsym(h, n);
    QGNN_REQUIRE(p, QGNN_ENCCL, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.CommGetAsyncError =
      reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
  api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
  api.h = h;
  return api;
}

#define QGNN_NCCL(call)                                                                  \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      throw ::qgnn_b200::Status(QGNN_ENCCL, std::string(#call) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

// Row-range plan of the production fp32 SpMM (spmm.cu:spmm_f32): rows with
// more than hub_deg neighbours (a + b lists) are split into 256-edge segments
// (reduced in segment order by the last-arriving segment, or k_spmm_hubred),
// the other rows are listed by descending degree for the multi-row narrow
// kernel (k_spmm_sorted).  maxd: widest row the partial-row workspace holds
// (0: no workspace, fp64 engines).
struct Hubs {
DBuf<int32_t> rows, seg_ptr, order, seg_hub, cnt;
DBuf<int64_t> seg;
DBuf<float> part;
HubPlan plan;
};

inline void build_hub_plan(Hubs& h, const int64_t* pa, const int64_t* pb, int64_t r0, int64_t r1,
                         int64_t maxd, int64_t kHubDeg) {
  constexpr int64_t kSeg = 256;
  std::vector<int32_t> rows, sptr{0};
  std::vector<int64_t> seg;
  std::vector<int32_t> seg_hub;  // hub index of each segment
  std::vector<std::pair<int64_t, int32_t>> by_deg;  // (-degree, row) of the non-hub rows
  int64_t total_deg = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t a0 = pa[r], a1 = pa[r + 1];
    const int64_t b0 = pb ? pb[r] : 0, b1 = pb ? pb[r + 1] : 0;
    const int64_t deg = (a1 - a0) + (b1 - b0);
    total_deg += deg;
    if (deg <= kHubDeg) {
      by_deg.emplace_back(-deg, int32_t(r));
      continue;
    }
    rows.push_back(int32_t(r));
    for (int64_t e = 0; e < deg; e += kSeg) {  // edge positions in the (a ++ b) list
      const int64_t f = std::min(deg, e + kSeg);
      const int64_t la = a1 - a0;
      seg.push_back(a0 + std::min(e, la));
      seg.push_back(a0 + std::min(f, la));
      seg.push_back(b0 + std::max<int64_t>(0, e - la));
      seg.push_back(b0 + std::max<int64_t>(0, f - la));
    }
    sptr.push_back(int32_t(seg.size() / 4));
    seg_hub.resize(seg.size() / 4, int32_t(rows.size() - 1));
  }
  // degree-descending row order for the multi-row narrow kernel (spmm.cu:k_spmm_sorted)
  std::sort(by_deg.begin(), by_deg.end());
  std::vector<int32_t> order(by_deg.size());
  for (size_t i = 0; i < by_deg.size(); ++i) order[i] = by_deg[i].second;
  h.order.upload(order);
  h.plan.order = order.empty() ? nullptr : h.order.p;
  h.plan.n_order = int64_t(order.size());
  h.plan.avg_deg = r1 > r0 ? double(total_deg) / double(r1 - r0) : 0.0;
  h.seg_hub.upload(seg_hub);
  h.cnt.alloc(std::max<size_t>(1, rows.size()));  // zeroed
  h.plan.seg_hub = h.seg_hub.p;
  h.plan.cnt = h.cnt.p;
  h.rows.upload(rows);
  h.seg_ptr.upload(sptr);
  h.seg.upload(seg);
  const int64_t n_segs = int64_t(seg.size() / 4);
  if (maxd > 0) h.part.alloc(std::max<int64_t>(1, n_segs) * maxd, false);
  h.plan.hub_deg = kHubDeg;
  h.plan.n_hubs = int64_t(rows.size());
  h.plan.n_segs = n_segs;
  h.plan.hubs = h.rows.p;
  h.plan.seg_ptr = h.seg_ptr.p;
  h.plan.seg = h.seg.p;
  h.plan.part = reinterpret_cast<float*>(h.part.p);
  h.plan.ldp = maxd;
}


// ------------------------------------------------------ small kernels ----
template <typename T>
__global__ void k_sum_parts(const T* __restrict__ all, int parts, int64_t n, T* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  T s = T(0);
  for (int p = 0; p < parts; ++p) {  // ascending device order, engine.hpp:786-788
    if constexpr (sizeof(T) == 8)
      s = __dadd_rn(s, all[static_cast<int64_t>(p) * n + i]);
    else
      s += all[static_cast<int64_t>(p) * n + i];
  }
  out[i] = s;
}

template <typename T>
__global__ void k_fill2(T* __restrict__ a, T va, T* __restrict__ b, T vb, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    a[i] = va;
    b[i] = vb;
  }
}

// ------------------------------------------------------- loopback comm ----
// In-process transport for world > 1 on ONE device (tests): every rank is an
// Engine in its own host thread; collectives publish device pointers / events
// in a shared group and copy with cudaMemcpyAsync between the ranks' buffers.
// It exercises the same routing (arena offsets, remote pairs, rank slices) as
// the NCCL path — the analogue of the reference's in-process mailbox.
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<void*> engines, ptr;
  std::vector<cudaEvent_t> ev, ev2;
  // per rank: (peer, p, q, bytes) of its grouped sends / receives, in issue order
  std::vector<std::vector<std::array<int64_t, 4>>> sends, recvs;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
// Peer-store flags.  signal: every prior write of this stream (the K1 stores into
// peer arenas, or the reads of the receive regions) is ordered before the flag
// store (kernel boundary + system fence, release at system scope).  wait: acquire
// at system scope; gives up after QGNN_P2P_TIMEOUT_MS (30 s) with a ProtocolError
// ("missing payload") instead of hanging the GPU.
__global__ void k_p2p_signal(uint64_t* const* __restrict__ dst, int n, uint64_t v) {
  const int i = threadIdx.x;
  if (i >= n || !dst[i]) return;
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst[i]), "l"(v) : "memory");
}
__global__ void k_p2p_wait(const uint64_t* __restrict__ flags, int n, int skip, uint64_t v,
                           uint64_t timeout_ns, int* err) {
  const int i = threadIdx.x;
  if (i >= n || i == skip) return;
  uint64_t t0, t, x;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(flags + i) : "memory");
    if (x >= v) break;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {  // ProtocolError "exchange: missing payload" (engine.hpp:530)
      atomicOr(err, kErrMissing);
      break;
    }
    __nanosleep(200);
  }
}

static std::mutex g_loop_mu;
static std::map<uint64_t, std::shared_ptr<LoopGroup>> g_loops;
constexpr char kLoopMagic[8] = {'Q', 'G', 'N', 'N', 'L', 'O', 'O', 'P'};

// NVTX phase ranges (SURVEY §5 tracing): host-side ranges around each layer's
// enqueue, the loss, the step and the adaptive re-solve; header-only NVTX 3, a no-op
// unless a profiler is attached (inside a replayed CUDA graph they appear only while
// the graph is captured).
struct NvtxRange {
  NvtxRange(const char* what, int64_t idx) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%s %lld", what, static_cast<long long>(idx));
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

// ------------------------------------------------------------ engine ----
enum BitMode { kFp = 0, kFixed = 1, kUniform = 2, kAdaptive = 3 };
constexpr int kChoices[3] = {2, 4, 8};

struct KeyInfo {
  int t;
  bool bwd;
  int64_t dim;
  uint64_t code;  // engine.hpp:455-457
};

// Messages of one ordered pair for one key (codec wire order within the set).
struct PairMsgs {
  std::vector<uint32_t> ids;  // caller order (ascending id)
  std::vector<uint8_t> bits;
  std::vector<uint64_t> off;  // byte offset inside the set
  uint64_t bytes = 0, ref_bytes = 0;
};

struct KStat {
  double ms = 0;
  double launches = 0;
  double bytes = 0;
  double gbytes = 0;  // SpMM classes: gathered row bytes (nnz x dim x elem), the L2 gather model
};

class EngineBase {
 public:
  virtual ~EngineBase() = default;
  virtual void run_epoch(qgnn_epoch_metrics* m) = 0;
  virtual void launch_epoch() = 0;
  virtual void finish_epoch(qgnn_epoch_metrics* m) = 0;
  virtual void set_features(const void* f) = 0;
  virtual void get_weights(int l, void* out) = 0;
  virtual void set_weights(int l, const void* in) = 0;
  virtual void info(int64_t* out) = 0;
  virtual int kernel_stats(double* out, int n) = 0;
  virtual void set_kstats(bool on) = 0;
};

template <typename T>
class Engine final : public EngineBase {
 public:
  Engine(const qgnn_settings& s, int64_t n, const int64_t* ptr, const int32_t* adj,
         const void* features, const int32_t* labels, const uint8_t* train, const uint8_t* val,
         const uint8_t* test, const uint32_t* owner, const void* nccl_id);
  ~Engine() override;
  void run_epoch(qgnn_epoch_metrics* m) override {
    launch_epoch();
    finish_epoch(m);
  }
  void launch_epoch() override;
  void set_kstats(bool on) override {
    QGNN_REQUIRE(!in_flight_, QGNN_EPROTOCOL, "set_kstats: an epoch is in flight");
    s_.kstats = on ? 1 : 0;
  }
  void finish_epoch(qgnn_epoch_metrics* m) override;
  bool in_flight_ = false;
  // CUDA graph of the steady-state epoch (one GPU, no pending feature upload):
  // captured once per plan version / arena and replayed with one launch
  struct EpochGraph {
    cudaGraphExec_t exec = nullptr;
    uint64_t plan = ~uint64_t(0);
    void* arena = nullptr;
    void* scratch = nullptr;  // context workspaces baked into the graph
    void* gemm_b = nullptr;
    std::vector<std::tuple<int, size_t, double>> ev_used;
    int64_t launches = 0;
    double gbytes[QGNN_K_COUNT] = {};
  } graphs_[2];  // [0]: steady state, [1]: first layer consumes a pending feature upload
  bool capturing_ = false;
  bool graphs_enabled() const {
    const char* e = std::getenv("QGNN_GRAPH");
    // per-kernel event timing (kstats) cannot time events recorded inside a graph
    return (!e || std::atoi(e) != 0) && s_.world == 1 && s_.bit_mode != kUniform && !s_.kstats;
  }
  void epoch_body();
  DBuf<double> adam_bc_;  // [2] bias corrections of this epoch's step
  double* adam_bc_host_ = nullptr;
  // adaptive re-solve: trace windows of all keys gathered here once per period
  // (persistent device buffer for the cross-rank gather, pinned host copy)
  DBuf<T> win_dev_;
  T* win_host_ = nullptr;
  size_t win_cap_ = 0;
  void set_features(const void* f) override;
  void get_weights(int l, void* out) override;
  void set_weights(int l, const void* in) override;
  void info(int64_t* out) override;
  int kernel_stats(double* out, int n) override;

 private:
  struct PartDev {
    int id = 0;
    View view;
    // static graph arrays
    DBuf<int64_t> lptr, rptr, sptr;
    DBuf<int32_t> lcol, rslot, srow;
    DBuf<T> lafwd, labwd, ralpha, salpha, self_alpha;
    DBuf<int32_t> labels, train_rows, val_rows, test_rows, loss_rows, ref_order;
    DBuf<int32_t> ref_row;            // GPU row -> reference row (dropout coordinates)
    std::vector<DBuf<T>> act, istd;   // chain: act_in (y or z) and LN inv_std per layer
    int64_t n_train = 0, n_val = 0, n_test = 0;
    // activations
    std::vector<DBuf<T>> h, hagg;  // h[0..L], hagg[0..L-1]
    DBuf<T> halo, partials, dh, dh_next, dz, gbar;
    DBuf<T> gpart;  // transform-first last layer: backward_remote_partials of dz
    DBuf<int32_t> row_node_d;  // GPU row -> node id (feature gather)
    // 1[h[l] > 0] as 32-column bit words per hidden layer l, written by layer l's
    // forward GEMM epilogue and read as layer l + 1's ReLU-backward mask (32 B per
    // 256-wide row instead of the 1 KB activation row); rows covered this epoch
    std::vector<DBuf<uint32_t>> hbits;
    std::vector<int64_t> hbits_rows;
    // per key: sender metadata
    struct SendMeta {
      DBuf<int32_t> rows;
      DBuf<uint32_t> ids;
      DBuf<uint8_t> bits;
      DBuf<uint64_t> off;
      DBuf<uint16_t> set;
      uint64_t* keys = nullptr;  // [P] view into Engine::keys_all_
      DBuf<T> wlo, whi;
      int64_t n = 0;
      std::vector<int64_t> q_begin;  // [P+1] message ranges per destination
    };
    struct RecvMeta {
      DBuf<int32_t> dst;
      DBuf<uint8_t> bits;
      DBuf<uint64_t> off;
      int64_t n = 0;
      std::vector<int64_t> p_begin;  // [P+1] message ranges per source
      // backward keys: destination rows with their incoming messages in ascending
      // source order (one fused scatter-add launch instead of one per source)
      DBuf<int32_t> acc_rows, acc_ptr, acc_msg;
      // expected chunk envelope per message (source | destination << 8 |
      // plan version << 16, each mod 256; GPU layout): checked by K3
      DBuf<uint32_t> env;
      int64_t n_acc_rows = 0;
      // forward keys (fp32 GPU layout): chunk word of every remote CSR entry (offset /
      // 16 + width code of the entry's message), rebuilt with every plan, so the
      // marginal SpMM reaches each packed halo row in one dependent round trip
      DBuf<int32_t> words;
    };
    std::vector<SendMeta> snd;
    std::vector<RecvMeta> rcv;
    double* loss = nullptr;               // [1] view into Engine::epoch_out_
    unsigned long long* correct = nullptr;  // [2] view into Engine::epoch_out_
    DBuf<double> ce_terms;
    // hub rows (slots) per SpMM call site, segmented (spmm.cu:k_spmm_hubseg)
    Hubs hub_fc, hub_fm, hub_bwd, hub_part;
  };

  int64_t ld_of(int64_t d) const { return round_up(d, 8); }
  // rows with more neighbours than this are split across a CTA (QGNN_HUB_DEG overrides)
  int64_t kHubDeg = 128;
  // K4 dispatch: fp32 -> nnz-balanced row-range kernel with hub splitting (all
  // feature buffers are zero-padded to a multiple of 4 columns); fp64 -> the
  // reference-order kernel.  Returns the number of kernels launched.
  // rows [r0, r1) whose (a + b) degree exceeds kHubDeg -> 256-edge segments
  template <typename H>
  void build_hubs(H& h, const std::vector<int64_t>& pa, const std::vector<int64_t>* pb, int64_t r0,
                  int64_t r1, int64_t maxd) {
    build_hub_plan(h, pa.data(), pb ? pb->data() : nullptr, r0, r1, sizeof(T) == 4 ? maxd : 0,
                   kHubDeg);
  }

  int spmm(int64_t dim, const T* x, int64_t ldx, const T* y, int64_t ldy, const T* sa,
           const int64_t* pa, const int32_t* ca, const T* aa, const int64_t* pb,
           const int32_t* cb, const T* ab, int64_t r0, int64_t n, T* out, int64_t ldo,
           const HubPlan* hubs, const T* mask = nullptr, int64_t ldm = 0,
           const PackedHalo* pk = nullptr) {
    if constexpr (sizeof(T) == 4) {
      return spmm_f32(ctx_, int(round_up(dim, 4)), x, ldx, y, ldy, sa, pa, ca, aa, pb, cb, ab, r0,
                      n, out, ldo, hubs, s_main_, mask, ldm, pk);
    } else {
      const int st = qgnn_csr_aggregate(ctx_, dtype_, dim, x, ldx, y, ldy, sa, pa, ca, aa, pb, cb,
                                        ab, nullptr, r0, n, out, ldo, s_main_);
      if (st) throw Status(st, qgnn_last_error());
      return 1;
    }
  }
  // f(i) for every hosted partition on its own host thread (setup and plan
  // uploads: per-partition host loops, uploads and allocations are independent)
  template <typename F>
  void par_parts(F&& f) {
    std::vector<std::future<void>> jobs;
    for (size_t i = 0; i < parts_dev_.size(); ++i)
      jobs.push_back(std::async(std::launch::async, [&, i] {
        QGNN_CUDA(cudaSetDevice(s_.device));
        f(i);
      }));
    for (auto& j : jobs) j.get();
  }
  void build_messages();
  void negotiate_sizes();
  DBuf<uint64_t> neg_;
  void layout_pair(int k, int p, int q);
  void upload_key_meta(int k);
  void compute_bits_uniform();
  void prepare_epoch();
  void quantize(PartDev& P, int k, const T* src, int64_t ld, cudaStream_t st = nullptr);
  // one GPU: encode / decode on the side stream, overlapping the compute stream
  // (per-kernel timing runs serialised so each class's time is its own)
  bool side_overlap() const {
    return zero_copy() && (side_enabled() || s_.overlap >= 2) && !s_.kstats;
  }
  // K1/K3 on a side stream alongside the central rows (QGNN_SIDE_STREAM=1).  Off by
  // default since the SpMM/GEMM kernels saturate the GPU: in the captured graph the
  // concurrent encode/decode cost 1.6 ms/epoch more than running it in line.
  static bool merge_gemm_enabled() {  // QGNN_MERGE_GEMM=0: separate central / marginal GEMMs
    const char* e = std::getenv("QGNN_MERGE_GEMM");
    return !e || std::atoi(e) != 0;
  }
  static bool direct_words_enabled() {  // QGNN_CHUNK_WORDS=0: slot-indexed packed gathers
    const char* e = std::getenv("QGNN_CHUNK_WORDS");
    return !e || std::atoi(e) != 0;
  }
  static bool k3_words_enabled() {  // QGNN_K3_WORDS=0: message-indexed backward scatter-add
    const char* e = std::getenv("QGNN_K3_WORDS");
    return !e || std::atoi(e) != 0;
  }
  static bool one_dgrad_enabled() {  // QGNN_ONE_DGRAD=0: split input gradients (A/B only)
    const char* e = std::getenv("QGNN_ONE_DGRAD");
    return !e || std::atoi(e) != 0;
  }
  static bool side_enabled() {
    const char* e = std::getenv("QGNN_SIDE_STREAM");
    return e && std::atoi(e) != 0;
  }
  void fork_side() {  // s_comm_ continues after everything queued on s_main_
    QGNN_CUDA(cudaEventRecord(ev_fork_, s_main_));
    QGNN_CUDA(cudaStreamWaitEvent(s_comm_, ev_fork_, 0));
  }
  void join_side() {  // s_main_ continues after everything queued on s_comm_
    QGNN_CUDA(cudaEventRecord(ev_join_, s_comm_));
    QGNN_CUDA(cudaStreamWaitEvent(s_main_, ev_join_, 0));
  }
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  void decode_halo(int k, int64_t din, int64_t ldi, cudaStream_t st);
  // §8f rank 1: forward key k's marginal SpMM reads the halo rows straight from
  // the exchange arena (no K3 store, no fp32 halo) when every partition's
  // marginal range runs through a kernel with a packed variant (fp32, GPU layout)
  bool packed_fwd(int k, int64_t din, int64_t ldi);
  PackedHalo packed_halo(PartDev& D, int k, int64_t din);
  void exchange(int k);
  void forward_layer(int l);
  void forward_last_tf(int l);
  void backward_last_tf(int l);
  bool tf_last_ = false;  // last layer aggregates after the transform (fp32, dout < din)
  // fp32 + GPU wire layout: ReLU backward folded into the producers of dh (masked by h)
  bool relu_fused() const { return sizeof(T) == 4 && s_.layout == QGNN_WIRE_GPU && !chain_; }
  int64_t hbits_ld(int64_t l) const { return ceil_div(dims_[l], 32); }  // words per row
  // layer t's ReLU-backward mask: its bit words when this epoch's forward wrote them
  // for every row (ldm < 0 selects them in the kernels), else the activation rows
  std::pair<const T*, int64_t> relu_mask(PartDev& D, int64_t t, int64_t ldi) {
    if (!D.hbits.empty() && D.hbits_rows[t] == D.view.num_owned)
      return {reinterpret_cast<const T*>(D.hbits[t].p), -hbits_ld(t)};
    return {D.h[t].p, ldi};
  }
  static bool mask_bits_enabled() {  // QGNN_MASK_BITS=0: float activation rows as the mask
    const char* e = std::getenv("QGNN_MASK_BITS");
    return !e || std::atoi(e) != 0;
  }
  // LayerNorm / dropout (TrainSettings::layer_norm, dropout; model.hpp:62-153): the
  // transform writes act[t], chain.cu turns it into h[l] and back-propagates
  bool chain_ = false;
  bool chain_layer(int64_t l) const {  // layer l (1-based) runs the explicit chain
    return chain_ && (s_.layer_norm || l < L_);
  }
  ChainArgs chain_args(const PartDev& D, int64_t l) const {
    ChainArgs c;
    c.ln = s_.layer_norm;
    c.relu = l < L_ ? 1 : 0;
    if (s_.dropout > 0.0 && l < L_) {
      c.keep = 1.0 - s_.dropout;
      c.keep_thr = uint64_t(std::ceil(std::ldexp(c.keep, 53)));
      c.drop_key = drop_keys_.p + (D.id - p0_) * L_ + l;
      c.ref_row = D.ref_row.p;
    }
    return c;
  }
  DBuf<uint64_t> drop_keys_;        // [local parts][L + 1] fork({0x4, epoch, l, device}) keys
  uint64_t* drop_keys_host_ = nullptr;
  bool dh_masked_ = false;  // dh already carries the ReLU-backward mask of its layer
  // tensor-pipe work of a GEMM over n rows: 2 n din dout per product, three TF32
  // products (3xTF32) on the fp32 path (reported per GEMM class next to the bytes)
  double gemm_flops(double n, int64_t din, int64_t dout) const {
    return 2.0 * n * double(din) * double(dout) * (sizeof(T) == 4 ? 3.0 : 1.0);
  }
  int gemm_nk() const {  // kernels of the last dense_forward / input_grad call
    return (sizeof(T) == 4 && use_tc_gemm()) ? std::max(1, ctx_->last_gemm_launches) : 1;
  }
  void loss_phase();
  void backward_layer(int l);
  void backward_last();
  // bwd_finish scatter-add (engine.hpp:718-738) of every received partial into dh_next.
  // fp32 + GPU layout: one launch, warp per destination row summing its messages
  // in ascending source order; otherwise one exact-order launch per source.
  void scatter_add_all(PartDev& D, int k, int64_t din, int64_t ldi, const T* mask,
                       int64_t ldm) {
    auto& R = D.rcv[k];
    if (!R.n) return;
    double wire = 0;
    for (int64_t src = 0; src < P_; ++src)
      if (src != D.id) wire += double(msgs_[k][src][D.id].bytes);
    if constexpr (sizeof(T) == 4) {
      if (s_.layout == QGNN_WIRE_GPU) {
        kbegin(QGNN_K_DEQUANT);
        dequant_rows_add_f32(ctx_, arena_.p, R.n_acc_rows, R.acc_rows.p, R.acc_ptr.p, R.acc_msg.p,
                             R.words.p, int(din), R.bits.p, R.off.p, D.dh_next.p, ldi, mask, ldm,
                             R.env.p, s_main_);
        kend(QGNN_K_DEQUANT, double(R.n_acc_rows) * 2 * din * sizeof(T) + double(R.n) * 13 + wire,
             s_main_);
        return;
      }
    }
    for (int64_t src = 0; src < P_; ++src) {  // ascending source (engine.hpp:720-734)
      const int64_t b = R.p_begin[src], e = R.p_begin[src + 1];
      if (e == b) continue;
      kbegin(QGNN_K_DEQUANT);
      dequant_add(D, R, b, e, din, ldi, mask, ldm);
      kend(QGNN_K_DEQUANT, double(e - b) * (2 * din * sizeof(T) + 13) +
                               double(msgs_[k][src][D.id].bytes), s_main_);
    }
  }
  // ascending-source scatter-add of decoded rows [b, e) of R into dh_next (mask: fp32 ReLU bwd)
  template <typename R_>
  void dequant_add(PartDev& D, R_& R, int64_t b, int64_t e, int64_t din, int64_t ldi, const T* mask,
                   int64_t ldm) {
    if constexpr (sizeof(T) == 4) {
      if (s_.layout == QGNN_WIRE_GPU) {
        dequant_add_masked_f32(ctx_, arena_.p, e - b, int(din), R.bits.p + b, R.off.p + b,
                               R.dst.p + b, D.dh_next.p, ldi, mask, ldm,
                               R.env.p ? R.env.p + b : nullptr, s_main_);
        return;
      }
    }
    const int st = qgnn_dequant_scatter(ctx_, arena_.p, e - b, din, R.bits.p + b, R.off.p + b,
                                        s_.layout, R.dst.p + b, 1, D.dh_next.p, dtype_, ldi,
                                        R.env.p ? R.env.p + b : nullptr, s_main_);
    if (st) throw Status(st, qgnn_last_error());
  }
  void step();
  void adaptive_round(qgnn_epoch_metrics* m);
  size_t window_layout(std::vector<int64_t>& stride, std::vector<int64_t>& koff);
  uint64_t msg_offset_send(int k, int p, int q) const { return send_base_[k][p][q]; }
  void arena_layout();
  // profiling
  void kbegin(int cls, cudaStream_t st = nullptr);
  void kend(int cls, double bytes, cudaStream_t s, int nk = 1, double gbytes = 0);
  void flush_kstats();

  qgnn_settings s_;
  int64_t P_ = 0, L_ = 0, p0_ = 0, p1_ = 0;
  std::vector<int64_t> dims_;
  uint64_t root_ = 0;
  uint64_t epoch_ = 0;
  qgnn_ctx* ctx_ = nullptr;
  cudaStream_t s_main_ = nullptr, s_comm_ = nullptr;
  cudaEvent_t ev_a_ = nullptr, ev_b_ = nullptr, ev_x_ = nullptr, ev_q_ = nullptr;
  ncclComm_t comm_ = nullptr;
  // one GPU: route same-GPU pairs through NCCL self send/receive instead of
  // zero copy (settings.transport = 1): the multi-GPU exchange code path,
  // exercised and timed on a single device
  bool self_xfer_ = false;
  bool zero_copy() const { return s_.world == 1 && !self_xfer_; }
  // K1 chunk envelope of sender partition p: source | plan version << 8 (GPU layout)
  uint32_t envelope(int p) const {
    return s_.layout == QGNN_WIRE_GPU
               ? (uint32_t(p + env_skew_src_) & 0xffu) |
                     (uint32_t(plan_version_ + env_skew_ver_) & 0xffu) << 8
               : 0u;
  }
  // test hook (QGNN_TEST_ENVELOPE=source|version): senders stamp a wrong source
  // or plan version, which the receivers' K3 must reject (ProtocolError)
  int env_skew_src_ = 0, env_skew_ver_ = 0;
  std::shared_ptr<LoopGroup> loop_;     // loopback transport (tests), else NCCL
  cudaEvent_t ev_c_ = nullptr, ev_d_ = nullptr;
  std::vector<cudaEvent_t> peer_x_;     // loopback: peers' exchange-done events
  DBuf<double> dloss_;
  DBuf<uint64_t> dstat_;  // per-rank epoch status, all-gathered in finish_epoch
  DBuf<uint64_t> keys_all_;      // [key][hosted partition][destination] RNG set keys
  uint64_t* keys_host_ = nullptr;  // pinned staging of keys_all_
  DBuf<uint64_t> epoch_out_;     // [hosted partitions] loss (f64 bits), then [2 x] hit counts
  uint64_t* epoch_out_host_ = nullptr;  // pinned readback of epoch_out_
  DBuf<unsigned long long> dcorr_;
  template <typename X>
  void allgather_dev(X* base, int64_t slice, cudaStream_t s);
  void wait_exchange();
  int dtype_ = QGNN_F32;

  // host graph facts
  int64_t n_nodes_ = 0;
  std::vector<uint32_t> owner_;
  std::vector<Part> parts_;
  std::vector<KeyInfo> keys_;
  // msgs_[k][p][q]
  std::vector<std::vector<std::vector<PairMsgs>>> msgs_;
  std::vector<std::vector<std::vector<uint64_t>>> send_base_, recv_base_;
  // ---- peer-store transport (settings.transport = 2, world > 1):
  // K1 stores each remote pair's chunks straight into the receiver's arena (peer
  // memory over NVLink: CUDA IPC across processes, plain device pointers between
  // in-process loopback ranks), so the exchange moves no bytes of its own.  The
  // arena layout is plan-independent (worst-case widths), every rank derives every
  // rank's receive offsets, and per-rank flags at the arena's tail order the stores:
  // flags[0, world) = exchanges whose stores peer r has finished (ready), flags[world,
  // 2 world) = exchanges peer r has finished reading (consumed).
  bool p2p_ = false;
  bool send_open_ = false;       // this exchange's consumed-wait / ready-signal pending
  uint64_t xseq_ = 0;            // exchanges completed (identical on every rank)
  std::vector<uint8_t*> peer_arena_;                       // [world] (own = arena_.p)
  std::vector<uint64_t> flags_off_;                        // [world] flag block offsets
  std::vector<std::vector<std::vector<uint64_t>>> p2p_recv_;  // [k][q][p] in q's arena
  std::vector<bool> ipc_opened_;
  DBuf<uint64_t*> sig_ready_, sig_cons_;  // peers' flag words this rank writes
  void watchdog_wait(cudaEvent_t ev);
  void p2p_layout();
  void p2p_connect();
  void p2p_begin_send();
  static uint64_t p2p_timeout_ns() {
    const char* e = std::getenv("QGNN_P2P_TIMEOUT_MS");
    return uint64_t(e ? std::max(1L, std::atol(e)) : 30000L) * 1000000ull;
  }
  DBuf<uint8_t> arena_;
  size_t arena_bytes_ = 0;
  std::vector<std::unique_ptr<PartDev>> parts_dev_;
  // adaptive plan
  uint64_t plan_version_ = 0;
  std::vector<std::vector<std::vector<double>>> rx_asq_;  // [p][q][i] fwd stats
  // weights
  std::vector<int64_t> woff_;  // offsets of layer l in the flat parameter vector
  int64_t nparams_ = 0;
  DBuf<T> w_, adam_m_, adam_v_, wgrad_all_, wsum_;
  uint64_t adam_t_ = 0;
  int64_t global_train_ = 0, global_val_ = 0, global_test_ = 0;
  // profiling
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool_;
  std::vector<std::tuple<int, size_t, double>> ev_used_;  // (class, pool index, bytes)
  size_t ev_next_ = 0;
  KStat kst_[QGNN_K_COUNT];
  int cur_cls_ = -1;
  int64_t launches_ = 0, launches_last_ = 0;
  DBuf<T> feat_all_;  // node-ordered features (pinned-input fast path)
  // async feature upload: node-range chunks on s_copy_, one event per chunk;
  // partition p's gather waits for the chunk holding its largest node id
  cudaStream_t s_copy_ = nullptr;
  cudaEvent_t ev_feat_free_ = nullptr;
  std::vector<int64_t> feat_bounds_;    // chunk c = nodes [bounds[c], bounds[c + 1])
  std::vector<cudaEvent_t> ev_feat_;    // per chunk
  std::vector<int> part_chunk_;         // local partition -> chunk it waits for
  bool feat_pending_ = false;
  void gather_features(PartDev& D);
  bool bits_dirty_ = true;
  void recount_bits();
  // per-epoch message counters
  uint64_t msgs_b_[4] = {0, 0, 0, 0};
  double resolve_seconds_ = 0;
};

// ------------------------------------------------------------ profiling ---
template <typename T>
void Engine<T>::kbegin(int cls, cudaStream_t st) {
  if (!s_.kstats) return;
  if (ev_next_ == ev_pool_.size()) {
    cudaEvent_t a, b;
    QGNN_CUDA(cudaEventCreate(&a));
    QGNN_CUDA(cudaEventCreate(&b));
    ev_pool_.emplace_back(a, b);
  }
  cur_cls_ = cls;
  QGNN_CUDA(cudaEventRecord(ev_pool_[ev_next_].first, st ? st : s_main_));
}

template <typename T>
void Engine<T>::kend(int cls, double bytes, cudaStream_t s, int nk, double gbytes) {
  launches_ += nk;  // kernels of ours inside the region (always counted)
  if (!s_.kstats) return;
  kst_[cls].gbytes += gbytes;
  QGNN_CUDA(cudaEventRecord(ev_pool_[ev_next_].second, s));
  ev_used_.emplace_back(cls, ev_next_, bytes);
  ++ev_next_;
}

template <typename T>
void Engine<T>::flush_kstats() {
  if (!s_.kstats) return;
  for (auto& [cls, idx, bytes] : ev_used_) {
    float ms = 0;
    QGNN_CUDA(cudaEventElapsedTime(&ms, ev_pool_[idx].first, ev_pool_[idx].second));
    kst_[cls].ms += ms;
    kst_[cls].launches += 1;
    kst_[cls].bytes += bytes;
  }
  ev_used_.clear();
  ev_next_ = 0;
}

// ---------------------------------------------------------------- setup ---
template <typename T>
Engine<T>::Engine(const qgnn_settings& s, int64_t n, const int64_t* ptr, const int32_t* adj,
                  const void* features, const int32_t* labels, const uint8_t* train,
                  const uint8_t* val, const uint8_t* test, const uint32_t* owner,
                  const void* nccl_id)
    : s_(s) {
  dtype_ = sizeof(T) == 8 ? QGNN_F64 : QGNN_F32;
  QGNN_REQUIRE(s.n_dims >= 2 && s.n_dims <= 8, QGNN_EINVAL, "engine: dims must list in and out");
  QGNN_REQUIRE(s.n_parts >= 1, QGNN_EINVAL, "engine: n_parts must be >= 1");
  QGNN_REQUIRE(s.world >= 1 && s.rank >= 0 && s.rank < s.world, QGNN_EINVAL, "engine: bad rank");
  QGNN_REQUIRE(s.n_parts % s.world == 0, QGNN_EINVAL, "engine: n_parts must divide by world");
  QGNN_REQUIRE(s.bit_mode >= 0 && s.bit_mode <= 3, QGNN_EINVAL, "engine: bad bit mode");
  if (s.bit_mode == kFixed)
    QGNN_REQUIRE(s.fixed_bits == 2 || s.fixed_bits == 4 || s.fixed_bits == 8, QGNN_EINVAL,
                 "engine: fixed bit width must be 2, 4, or 8");
  QGNN_REQUIRE(labels && train && val && test, QGNN_EINVAL, "engine: missing labels");
  P_ = s.n_parts;
  L_ = s.n_dims - 1;
  // z = A(hW) for the last layer when it narrows (e.g. 256 -> 47 classes): the
  // exchanged tensors are unchanged, the SpMMs gather dout- instead of din-wide rows
  tf_last_ = sizeof(T) == 4 && L_ >= 2 && s.dims[L_] < s.dims[L_ - 1];
  if (const char* e = std::getenv("QGNN_TF_LAST")) tf_last_ = tf_last_ && std::atoi(e) != 0;
  if (const char* e = std::getenv("QGNN_HUB_DEG")) kHubDeg = std::max<int64_t>(1, std::atoll(e));
  QGNN_REQUIRE(s.dropout >= 0.0 && s.dropout < 1.0, QGNN_EINVAL, "engine: dropout must be in [0, 1)");
  chain_ = s.layer_norm != 0 || s.dropout > 0.0;
  dims_.assign(s.dims, s.dims + s.n_dims);
  p0_ = s.rank * (P_ / s.world);
  p1_ = p0_ + P_ / s.world;
  n_nodes_ = n;
  root_ = rng_seed_key(s.seed);
  QGNN_CUDA(cudaSetDevice(s.device));
  QGNN_REQUIRE(qgnn_ctx_create(s.device, &ctx_) == QGNN_OK, QGNN_ECUDA, qgnn_last_error());
  ctx_->b_reuse = true;  // private ctx: weights change only in step() / set_weights (wgen)
  int lo_pri = 0, hi_pri = 0;
  QGNN_CUDA(cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri));
  QGNN_CUDA(cudaStreamCreateWithPriority(&s_main_, cudaStreamNonBlocking, lo_pri));
  QGNN_CUDA(cudaStreamCreateWithPriority(&s_comm_, cudaStreamNonBlocking, hi_pri));
  QGNN_CUDA(cudaEventCreate(&ev_a_));
  QGNN_CUDA(cudaEventCreate(&ev_b_));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_x_, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_q_, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_c_, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_d_, cudaEventDisableTiming));
  QGNN_CUDA(cudaStreamCreateWithFlags(&s_copy_, cudaStreamNonBlocking));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&ev_feat_free_, cudaEventDisableTiming));
  if (s.world > 1) {
    QGNN_REQUIRE(nccl_id, QGNN_EINVAL, "engine: world > 1 needs an NCCL unique id");
    if (std::memcmp(nccl_id, kLoopMagic, 8) == 0) {
      uint64_t key;
      std::memcpy(&key, static_cast<const char*>(nccl_id) + 8, 8);
      std::lock_guard<std::mutex> lk(g_loop_mu);
      auto& g = g_loops[key];
      if (!g) {
        g = std::make_shared<LoopGroup>();
        g->world = s.world;
        g->engines.assign(s.world, nullptr);
        g->ptr.assign(s.world, nullptr);
        g->ev.assign(s.world, nullptr);
        g->ev2.assign(s.world, nullptr);
        g->sends.assign(s.world, {});
        g->recvs.assign(s.world, {});
      }
      QGNN_REQUIRE(g->world == s.world && !g->engines[s.rank], QGNN_EPROTOCOL,
                   "loopback group: world mismatch or rank already registered");
      g->engines[s.rank] = this;
      loop_ = g;
    } else {
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof(id));
      QGNN_NCCL(nccl().CommInitRank(&comm_, s.world, id, s.rank));
    }
    p2p_ = s.transport == 2;
  } else if (s.transport == 1) {
    self_xfer_ = true;
    const int dev = s.device;  // one-rank communicator: no bootstrap network needed
    QGNN_NCCL(nccl().CommInitAll(&comm_, 1, &dev));
  }

  // partition (engine.hpp:212) and coefficients (:213)
  if (owner)
    owner_.assign(owner, owner + n);
  else
    owner_ = partition_owner_bfs(ptr, adj, n, P_, s.seed);
  // §8f rank 3: consumer sets, coefficients, views and Σα² weights on the GPU
  // (QGNN_GPU_SETUP=0: the host builders of host_graph.cpp; identical outputs)
  const bool gpu_setup = [] {
    const char* e = std::getenv("QGNN_GPU_SETUP");
    return !e || std::atoi(e) != 0;
  }();
  const bool prof = std::getenv("QGNN_SETUP_PROFILE") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!prof) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[qgnn setup] %-22s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  phase("streams / comm");
  std::unique_ptr<GraphDev> gdev;
  std::vector<double> alpha, self_alpha;
  if (gpu_setup) {
    gdev = std::make_unique<GraphDev>(ptr, adj, n, owner_.data(), P_, s_main_);
    phase("graph upload");
    parts_ = partitions_from_owner_gpu(*gdev, owner_.data());
    phase("partitions (gpu)");
  } else {
    parts_ = partitions_from_owner(ptr, adj, n, owner_.data(), P_);
    compute_coeffs(ptr, adj, n, s.sage != 0, alpha, self_alpha);
    phase("partitions+coeffs (host)");
  }

  for (int64_t v = 0; v < n; ++v) {
    global_train_ += train[v] != 0;
    global_val_ += val[v] != 0;
    global_test_ += test[v] != 0;
  }
  QGNN_REQUIRE(global_train_ > 0, QGNN_EINVAL, "engine: empty train mask");
  if (const char* e = std::getenv("QGNN_TEST_ENVELOPE")) {
    env_skew_src_ = std::string(e) == "source" ? 1 : 0;
    env_skew_ver_ = std::string(e) == "version" ? 1 : 0;
  }

  // keys: forward t = 0..L-1, backward t = 1..L-1 (engine.hpp:345-352)
  for (int64_t t = 0; t < L_; ++t) keys_.push_back({int(t), false, dims_[t], uint64_t(2 * t)});
  for (int64_t t = 1; t < L_; ++t) keys_.push_back({int(t), true, dims_[t], uint64_t(2 * t + 1)});

  // views of hosted partitions (parallel)
  parts_dev_.resize(p1_ - p0_);
  std::vector<ViewDev<T>> vdev(size_t(p1_ - p0_));
  if (gpu_setup) {
    for (int64_t i = 0; i < p1_ - p0_; ++i) {
      parts_dev_[i] = std::make_unique<PartDev>();
      parts_dev_[i]->id = int(p0_ + i);
      build_view_gpu<T>(*gdev, parts_[p0_ + i], s.sage != 0, true, parts_dev_[i]->view, vdev[i],
                        false);
    }
  } else {
    std::vector<std::future<View>> futs;
    for (int64_t p = p0_; p < p1_; ++p)
      futs.push_back(std::async(std::launch::async, [&, p] {
        return build_view(ptr, adj, n, parts_[p], P_, alpha, self_alpha, s.sage != 0);
      }));
    for (int64_t i = 0; i < p1_ - p0_; ++i) {
      parts_dev_[i] = std::make_unique<PartDev>();
      parts_dev_[i]->id = int(p0_ + i);
      parts_dev_[i]->view = futs[i].get();
    }
  }

  phase("views");
  // forward-statistics weights of every pair (engine.hpp:262-273), for adaptive
  if (s.bit_mode == kAdaptive && gpu_setup) {
    rx_asq_ = rx_alpha_sq_gpu(*gdev, parts_, s.sage != 0);
  } else if (s.bit_mode == kAdaptive) {
    rx_asq_.assign(P_, std::vector<std::vector<double>>(P_));
    for (int64_t p = 0; p < P_; ++p)
      for (int64_t q = 0; q < P_; ++q) {
        if (p == q) continue;
        const auto& ids = parts_[p].remote_out[q];
        auto& out = rx_asq_[p][q];
        out.assign(ids.size(), 0.0);
        for (size_t i = 0; i < ids.size(); ++i) {
          const uint32_t u = ids[i];
          double acc = 0.0;
          for (int64_t e = ptr[u]; e < ptr[u + 1]; ++e) {  // ascending v == receiver row order
            const uint32_t v = static_cast<uint32_t>(adj[e]);
            if (owner_[v] != static_cast<uint32_t>(q)) continue;
            const double a = s.sage ? self_alpha[v] : alpha[e];
            acc += a * a;
          }
          out[i] = acc;
        }
      }
  }

  phase("rx alpha^2");
  gdev.reset();  // the device copy of the graph is only needed for setup
  // device state per hosted partition (partitions on worker threads)
  par_parts([&](size_t ip) {
    PartDev& D = *parts_dev_[ip];
    const View& V = D.view;
    if (gpu_setup) {  // built in place on the device
      ViewDev<T>& vd = vdev[ip];
      D.lptr = std::move(vd.lptr);
      D.lcol = std::move(vd.lcol);
      D.lafwd = std::move(vd.lafwd);
      D.labwd = std::move(vd.labwd);
      D.rptr = std::move(vd.rptr);
      D.rslot = std::move(vd.rslot);
      D.ralpha = std::move(vd.ralpha);
      D.sptr = std::move(vd.sptr);
      D.srow = std::move(vd.srow);
      D.salpha = std::move(vd.salpha);
      D.self_alpha = std::move(vd.self_alpha);
    } else {
      auto tocast = [](const std::vector<double>& v) { return std::vector<T>(v.begin(), v.end()); };
      D.lptr.upload(V.local_ptr);
      D.lcol.upload(V.local_col);
      D.lafwd.upload(tocast(V.local_afwd));
      D.labwd.upload(tocast(V.local_abwd));
      D.rptr.upload(V.remote_ptr);
      D.rslot.upload(V.remote_slot);
      D.ralpha.upload(tocast(V.remote_alpha));
      D.sptr.upload(V.slot_ptr);
      D.srow.upload(V.slot_row);
      D.salpha.upload(tocast(V.slot_alpha));
      D.self_alpha.upload(tocast(V.self_alpha));
    }
    std::vector<int32_t> lab(V.num_owned), tr, va, te;
    for (int64_t g = 0; g < V.num_owned; ++g) {
      const uint32_t node = V.row_node[g];
      lab[g] = labels[node];
    }
    for (int64_t r = 0; r < V.num_owned; ++r) {  // reference row order
      const int32_t g = V.gpu_row_of_ref[r];
      const uint32_t node = V.row_node[g];
      if (train[node]) tr.push_back(g);
      if (val[node]) va.push_back(g);
      if (test[node]) te.push_back(g);
    }
    D.labels.upload(lab);
    D.train_rows.upload(tr);
    D.val_rows.upload(va);
    D.test_rows.upload(te);
    {
      std::vector<int32_t> all(tr);
      all.insert(all.end(), va.begin(), va.end());
      all.insert(all.end(), te.begin(), te.end());
      D.loss_rows.upload(all);
    }
    D.n_train = int64_t(tr.size());
    D.n_val = int64_t(va.size());
    D.n_test = int64_t(te.size());
    D.ref_order.upload(V.gpu_row_of_ref);
    {
      std::vector<int32_t> rn(V.row_node.begin(), V.row_node.end());
      D.row_node_d.upload(rn);
    }
    const int64_t no = V.num_owned, nr = V.num_remote;
    int64_t maxd = 0;
    for (int64_t d : dims_) maxd = std::max(maxd, ld_of(d));
    D.h.resize(L_ + 1);
    D.hagg.resize(L_);
    for (int64_t l = 0; l <= L_; ++l) D.h[l].alloc(no * ld_of(dims_[l]));
    for (int64_t t = 0; t < L_; ++t) D.hagg[t].alloc(no * ld_of(dims_[t]));
    D.halo.alloc(std::max<int64_t>(1, nr) * maxd);
    D.partials.alloc(std::max<int64_t>(1, nr) * maxd);
    D.dh.alloc(no * maxd);
    D.dh_next.alloc(no * maxd);
    D.dz.alloc(no * maxd);
    D.gbar.alloc(no * maxd);
    if (tf_last_) D.gpart.alloc(std::max<int64_t>(1, nr) * ld_of(dims_[L_]));
    if (relu_fused() && mask_bits_enabled()) {
      D.hbits.resize(L_);
      D.hbits_rows.assign(L_, 0);
      for (int64_t l = 1; l < L_; ++l) D.hbits[l].alloc(std::max<int64_t>(1, no) * hbits_ld(l), false);
    }
    if (chain_) {  // act_in per layer (+ inv_std with LN), GPU -> reference rows for dropout
      D.act.resize(L_);
      D.istd.resize(L_);
      for (int64_t t = 0; t < L_; ++t) {
        if (!chain_layer(t + 1)) continue;
        D.act[t].alloc(no * ld_of(dims_[t + 1]));
        if (s_.layer_norm) D.istd[t].alloc(std::max<int64_t>(1, no));
      }
      if (s_.dropout > 0.0) D.ref_row.upload(V.ref_row);
    }
    // loss / hit counts and RNG set keys: views into per-rank buffers (constructor, below)
    D.ce_terms.alloc(std::max<int64_t>(1, D.n_train));
    if constexpr (sizeof(T) == 4) {
      build_hubs(D.hub_fc, V.local_ptr, nullptr, 0, V.n_central, maxd);
      build_hubs(D.hub_fm, V.local_ptr, &V.remote_ptr, V.n_central, no, maxd);
      build_hubs(D.hub_bwd, V.local_ptr, nullptr, 0, no, maxd);
      build_hubs(D.hub_part, V.slot_ptr, nullptr, 0, nr, maxd);
    }
    D.snd.resize(keys_.size());
    D.rcv.resize(keys_.size());
  });
  {  // feature-upload chunks: boundaries at each local partition's largest node id
    std::vector<int64_t> ends;
    for (auto& up : parts_dev_) {
      int64_t mx = -1;
      for (uint32_t nd : up->view.row_node) mx = std::max<int64_t>(mx, nd);
      ends.push_back(mx + 1);
    }
    std::vector<int64_t> b = ends;
    b.push_back(n_nodes_);
    std::sort(b.begin(), b.end());
    b.erase(std::unique(b.begin(), b.end()), b.end());
    feat_bounds_.assign(1, 0);
    for (int64_t x : b)
      if (x > feat_bounds_.back()) feat_bounds_.push_back(x);
    ev_feat_.assign(feat_bounds_.size() - 1, nullptr);
    for (auto& e : ev_feat_) QGNN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    part_chunk_.clear();
    for (int64_t e : ends) {
      int c = 0;
      while (c + 1 < int(ev_feat_.size()) && feat_bounds_[c + 1] < e) ++c;
      part_chunk_.push_back(c);
    }
  }
  phase("device state / hubs");
  set_features(features);
  if (feat_pending_) {  // construction consumes the features right away
    for (auto& up : parts_dev_) gather_features(*up);
    QGNN_CUDA(cudaEventRecord(ev_feat_free_, s_main_));
    feat_pending_ = false;
  }

  // weights: GnnModel::init (model.hpp:27-41), replicated on every rank
  woff_.assign(L_ + 1, 0);
  for (int64_t l = 0; l < L_; ++l) woff_[l + 1] = woff_[l] + dims_[l] * dims_[l + 1];
  nparams_ = woff_[L_];
  {
    std::vector<T> w(nparams_);
    for (int64_t l = 0; l < L_; ++l) {
      const double a = std::sqrt(6.0 / static_cast<double>(dims_[l] + dims_[l + 1]));
      const uint64_t key = rng_fork(rng_fork(rng_seed_key(s.seed), 0x77), uint64_t(l));
      for (int64_t i = 0; i < dims_[l] * dims_[l + 1]; ++i) {
        const double u = static_cast<double>(rng_u53(key, uint64_t(i) + 1)) * 0x1.0p-53;
        w[woff_[l] + i] = static_cast<T>((2.0 * u - 1.0) * a);
      }
    }
    w_.upload(w);
  }
  adam_m_.alloc(nparams_);
  adam_v_.alloc(nparams_);
  wgrad_all_.alloc(P_ * nparams_);
  wsum_.alloc(nparams_);

  plan_version_ = s.bit_mode == kAdaptive ? 1 : 0;
  phase("features / weights");
  {  // per-epoch key uploads and loss / hit-count readbacks: one copy each
    const size_t np = parts_dev_.size();
    keys_all_.alloc(std::max<size_t>(1, keys_.size() * np * size_t(P_)), true);
    QGNN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&keys_host_),
                            std::max<size_t>(1, keys_.size() * np * size_t(P_)) * sizeof(uint64_t),
                            cudaHostAllocDefault));
    epoch_out_.alloc(std::max<size_t>(1, 3 * np), true);
    QGNN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&epoch_out_host_),
                            std::max<size_t>(1, 3 * np) * sizeof(uint64_t), cudaHostAllocDefault));
    for (size_t i = 0; i < np; ++i) {
      parts_dev_[i]->loss = reinterpret_cast<double*>(epoch_out_.p + i);
      parts_dev_[i]->correct = reinterpret_cast<unsigned long long*>(epoch_out_.p + np + 2 * i);
    }
  }
  build_messages();
  if (p2p_) p2p_connect();
  phase("message lists");
  for (size_t k = 0; k < keys_.size(); ++k) upload_key_meta(int(k));
  phase("message metadata");
  QGNN_CUDA(cudaDeviceSynchronize());
  negotiate_sizes();
  if (s_.bit_mode == kAdaptive) {  // the re-solve's pinned window buffer
    std::vector<int64_t> stride, koff;
    window_layout(stride, koff);
  }
  phase("sync / negotiate");
}

// negotiate_buffers (plan.hpp:140-154) across ranks: every rank derives every
// pair's wire bytes from its own copy of the plan; the senders' figures are
// all-gathered and each receiver checks its incoming pairs against them
// (ProtocolError "negotiated buffer size mismatch", engine.hpp:546-547).  Runs
// at construction and after every plan adoption, never inside an epoch.
template <typename T>
void Engine<T>::negotiate_sizes() {
  if (s_.world == 1) return;
  const int64_t K = int64_t(keys_.size()), ppr = P_ / s_.world;
  const int64_t slice = K * ppr * P_ + 1;  // + the plan version
  std::vector<uint64_t> all(size_t(slice * s_.world), 0);
  uint64_t* mine = all.data() + s_.rank * slice;
  for (int64_t k = 0; k < K; ++k)
    for (int64_t p = p0_; p < p1_; ++p)
      for (int64_t q = 0; q < P_; ++q)
        if (q != p) mine[(k * ppr + (p - p0_)) * P_ + q] = msgs_[k][p][q].bytes;
  mine[slice - 1] = plan_version_;
  if (const char* e = std::getenv("QGNN_TEST_NEGOTIATE"))  // test hook: rank 1 disagrees
    if (std::atoi(e) == 1 && s_.rank == 1) mine[0] += 16;
  neg_.alloc(size_t(slice * s_.world), false);
  QGNN_CUDA(cudaMemcpyAsync(neg_.p, all.data(), all.size() * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, s_main_));
  allgather_dev(neg_.p, slice, s_main_);
  QGNN_CUDA(cudaStreamSynchronize(s_main_));
  QGNN_CUDA(cudaMemcpy(all.data(), neg_.p, all.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  bool ok = true;
  for (int r = 0; r < s_.world; ++r) {
    const uint64_t* theirs = all.data() + r * slice;
    ok &= theirs[slice - 1] == plan_version_;
    for (int64_t k = 0; k < K; ++k)
      for (int64_t p = r * ppr; p < (r + 1) * ppr; ++p)
        for (int64_t q = p0_; q < p1_; ++q)
          if (q != p) ok &= theirs[(k * ppr + (p - r * ppr)) * P_ + q] == msgs_[k][p][q].bytes;
  }
  // every rank learns every rank's verdict, so all of them fail together
  // (a lone failing rank would leave its peers waiting in the next exchange)
  std::vector<uint64_t> verdict(s_.world, 0);
  verdict[s_.rank] = ok ? 1 : 0;
  QGNN_CUDA(cudaMemcpyAsync(neg_.p, verdict.data(), verdict.size() * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, s_main_));
  allgather_dev(neg_.p, 1, s_main_);
  QGNN_CUDA(cudaStreamSynchronize(s_main_));
  QGNN_CUDA(cudaMemcpy(verdict.data(), neg_.p, verdict.size() * sizeof(uint64_t),
                       cudaMemcpyDeviceToHost));
  for (uint64_t v : verdict) ok &= v == 1;
  QGNN_REQUIRE(ok, QGNN_EPROTOCOL, "exchange: negotiated buffer size mismatch");
}

template <typename T>
Engine<T>::~Engine() {
  cudaDeviceSynchronize();
  if (drop_keys_host_) cudaFreeHost(drop_keys_host_);
  parts_dev_.clear();
  for (auto& e : ev_pool_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  // captured graphs may hold NCCL kernels of comm_: release them first
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec), g.exec = nullptr;
  if (comm_) nccl().CommDestroy(comm_);
  if (loop_) {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    loop_->engines[s_.rank] = nullptr;
    bool empty = true;
    for (void* e : loop_->engines) empty &= e == nullptr;
    if (empty)
      for (auto it = g_loops.begin(); it != g_loops.end(); ++it)
        if (it->second == loop_) {
          g_loops.erase(it);
          break;
        }
  }
  if (ev_c_) cudaEventDestroy(ev_c_);
  if (ev_d_) cudaEventDestroy(ev_d_);
  if (ev_a_) cudaEventDestroy(ev_a_);
  if (ev_b_) cudaEventDestroy(ev_b_);
  for (size_t r = 0; r < ipc_opened_.size(); ++r)
    if (ipc_opened_[r]) cudaIpcCloseMemHandle(peer_arena_[r]);
  if (keys_host_) cudaFreeHost(keys_host_);
  if (epoch_out_host_) cudaFreeHost(epoch_out_host_);
  if (ev_x_) cudaEventDestroy(ev_x_);
  if (ev_q_) cudaEventDestroy(ev_q_);
  if (s_main_) cudaStreamDestroy(s_main_);
  if (s_comm_) cudaStreamDestroy(s_comm_);
  if (s_copy_) cudaStreamDestroy(s_copy_);
  for (auto& g : graphs_)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (adam_bc_host_) cudaFreeHost(adam_bc_host_);
  if (win_host_) cudaFreeHost(win_host_);
  for (auto e : ev_feat_)
    if (e) cudaEventDestroy(e);
  if (ev_feat_free_) cudaEventDestroy(ev_feat_free_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (ctx_) qgnn_ctx_destroy(ctx_);
}

// h0[g] = feats[row_node[g]] for every partition row (zero padding untouched)
template <typename T>
__global__ void k_gather_rows(const T* __restrict__ feats, int64_t F, const int32_t* __restrict__ node,
                              int64_t n, T* __restrict__ out, int64_t ld) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t g = t / F;
  if (g >= n) return;
  const int64_t j = t - g * F;
  out[g * ld + j] = feats[int64_t(node[g]) * F + j];
}

template <typename T>
void Engine<T>::set_features(const void* f) {
  const int64_t F = dims_[0];
  const T* src = static_cast<const T*>(f);
  cudaPointerAttributes attr{};
  const bool pinned = cudaPointerGetAttributes(&attr, f) == cudaSuccess &&
                      (attr.type == cudaMemoryTypeHost || attr.type == cudaMemoryTypeDevice);
  cudaGetLastError();
  // node-range chunks copied asynchronously on s_copy_ (after the previous
  // epoch's readers of feat_all_); the epoch's first layer gathers partition
  // p into row order as soon as p's chunk has landed (gather_features), so
  // the upload overlaps the first layer's work.  A pinned `f` must stay alive
  // until the next run_epoch returns; a pageable one is consumed before
  // set_features returns (the copies from it are synchronous).
  if (!feat_all_.p || feat_all_.n < size_t(n_nodes_ * F)) feat_all_.alloc(n_nodes_ * F, false);
  // the staging matrix is free once the last epoch's gathers have read it
  // (ev_feat_free_ is recorded after them), so this copy may overlap the
  // rest of an epoch that is still in flight
  QGNN_CUDA(cudaStreamWaitEvent(s_copy_, ev_feat_free_, 0));
  for (size_t c = 0; c + 1 < feat_bounds_.size(); ++c) {
    const int64_t a = feat_bounds_[c], b = feat_bounds_[c + 1];
    QGNN_CUDA(cudaMemcpyAsync(feat_all_.p + a * F, src + a * F, size_t(b - a) * F * sizeof(T),
                              cudaMemcpyDefault, s_copy_));
    QGNN_CUDA(cudaEventRecord(ev_feat_[c], s_copy_));
  }
  if (!pinned) QGNN_CUDA(cudaStreamSynchronize(s_copy_));
  feat_pending_ = true;
}

// warp per row, 16-byte vectors (rows of F % 4 == 0 fp32 features)
__global__ void k_gather_rows4(const float4* __restrict__ feats, int64_t f4,
                               const int32_t* __restrict__ node, int64_t n, float4* __restrict__ out,
                               int64_t ld4) {
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < n; g += wstride) {
    const float4* src = feats + int64_t(node[g]) * f4;
    for (int64_t j = lane; j < f4; j += 32) out[g * ld4 + j] = __ldg(src + j);
  }
}

template <typename T>
void Engine<T>::gather_features(PartDev& D) {
  const int64_t F = dims_[0], ld = ld_of(F), no = D.view.num_owned;
  // inside a captured epoch the chunk events are recorded outside the graph
  QGNN_CUDA(cudaStreamWaitEvent(s_main_, ev_feat_[part_chunk_[D.id - p0_]],
                                capturing_ ? cudaEventWaitExternal : 0));
  if (sizeof(T) == 4 && F % 4 == 0)
    k_gather_rows4<<<unsigned(std::min<int64_t>(ceil_div(no, 8), int64_t(ctx_->num_sms) * 16)), 256,
                     0, s_main_>>>(reinterpret_cast<const float4*>(feat_all_.p), F / 4,
                                   D.row_node_d.p, no, reinterpret_cast<float4*>(D.h[0].p), ld / 4);
  else
    k_gather_rows<T><<<unsigned(ceil_div(no * F, 256)), 256, 0, s_main_>>>(feat_all_.p, F,
                                                                          D.row_node_d.p, no,
                                                                          D.h[0].p, ld);
  check_launch("k_gather_rows");
  ++launches_;
}

template <typename T>
void Engine<T>::recount_bits() {
  msgs_b_[0] = msgs_b_[1] = msgs_b_[2] = msgs_b_[3] = 0;
  for (size_t k = 0; k < keys_.size(); ++k)
    for (int64_t p = 0; p < P_; ++p)
      for (int64_t q = 0; q < P_; ++q) {
        if (p == q) continue;
        for (uint8_t b : msgs_[k][p][q].bits) ++msgs_b_[b == 0 ? 3 : b == 2 ? 0 : b == 4 ? 1 : 2];
      }
  bits_dirty_ = false;
}

// Message lists of every ordered pair and key (engine.hpp:142-143, 585-587, 683-687);
// bit widths from the mode, offsets from the codec wire order.
template <typename T>
void Engine<T>::build_messages() {
  msgs_.assign(keys_.size(), std::vector<std::vector<PairMsgs>>(P_, std::vector<PairMsgs>(P_)));
  // (key, source) rows of the pair table on host threads
  auto rows = [&](auto&& f) {
    std::vector<std::future<void>> jobs;
    for (size_t k = 0; k < keys_.size(); ++k)
      for (int64_t p = 0; p < P_; ++p) jobs.push_back(std::async(std::launch::async, f, k, p));
    for (auto& j : jobs) j.get();
  };
  rows([&](size_t k, int64_t p) {
    for (int64_t q = 0; q < P_; ++q) {
      if (p == q) continue;
      PairMsgs& m = msgs_[k][p][q];
      m.ids = keys_[k].bwd ? parts_[p].remote_in[q] : parts_[p].remote_out[q];
      const uint8_t b = s_.bit_mode == kFp ? 0 : s_.bit_mode == kFixed ? uint8_t(s_.fixed_bits) : 8;
      m.bits.assign(m.ids.size(), b);  // adaptive: initial all-8 plan (plan.hpp:104-126)
    }
  });
  if (s_.bit_mode == kUniform) compute_bits_uniform();
  rows([&](size_t k, int64_t p) {
    for (int64_t q = 0; q < P_; ++q)
      if (p != q) layout_pair(int(k), int(p), int(q));
  });
  arena_layout();
  bits_dirty_ = true;
}

template <typename T>
void Engine<T>::layout_pair(int k, int p, int q) {
  PairMsgs& m = msgs_[k][p][q];
  const int64_t n = int64_t(m.ids.size());
  const int64_t dim = keys_[k].dim;
  m.off.assign(n, 0);
  uint64_t off = 0, ref = 0;
  for (int b : {0, 2, 4, 8}) {
    for (int64_t i = 0; i < n; ++i) {
      if (m.bits[i] != b) continue;
      m.off[i] = off;
      off += qgnn_chunk_wire_bytes(dim, b, s_.layout, dtype_);
      ref += b == 0 ? uint64_t(dim) * 8 : qgnn_chunk_wire_bytes(dim, b, QGNN_WIRE_REF, QGNN_F64);
    }
  }
  m.bytes = off;
  m.ref_bytes = ref;
}

// engine.hpp:443-446: a random width per message per epoch
template <typename T>
void Engine<T>::compute_bits_uniform() {
  for (size_t k = 0; k < keys_.size(); ++k)
    for (int64_t p = 0; p < P_; ++p)
      for (int64_t q = 0; q < P_; ++q) {
        if (p == q) continue;
        PairMsgs& m = msgs_[k][p][q];
        for (size_t i = 0; i < m.ids.size(); ++i) {
          uint64_t key = root_;
          for (uint64_t c : {uint64_t(0x3), epoch_, keys_[k].code, uint64_t(p), uint64_t(q),
                             uint64_t(m.ids[i])})
            key = rng_fork(key, c);
          uint64_t ctr = 0;
          m.bits[i] = uint8_t(kChoices[rng_next_below(key, ctr, 3)]);
        }
      }
  bits_dirty_ = true;
}

// Arena: per key, send regions of hosted senders (per destination) followed by
// receive regions of hosted receivers for remote sources.  All keys reuse the
// same arena (they are processed one after another on the same streams).
template <typename T>
void Engine<T>::arena_layout() {
  if (p2p_) {
    p2p_layout();
    return;
  }
  send_base_.assign(keys_.size(), std::vector<std::vector<uint64_t>>(P_, std::vector<uint64_t>(P_, 0)));
  recv_base_ = send_base_;
  size_t need = 0;
  for (size_t k = 0; k < keys_.size(); ++k) {
    uint64_t o = 0;
    auto al = [](uint64_t x) { return (x + 255) / 256 * 256; };
    for (int64_t p = p0_; p < p1_; ++p)
      for (int64_t q = 0; q < P_; ++q) {
        if (q == p) continue;
        send_base_[k][p][q] = o;
        o = al(o + msgs_[k][p][q].bytes);
      }
    for (int64_t q = p0_; q < p1_; ++q)
      for (int64_t p = 0; p < P_; ++p) {
        if (p == q) continue;
        if (p >= p0_ && p < p1_ && !self_xfer_)
          recv_base_[k][q][p] = send_base_[k][p][q];  // zero copy on the same GPU
        else {
          recv_base_[k][q][p] = o;
          o = al(o + msgs_[k][p][q].bytes);
        }
      }
    need = std::max<size_t>(need, o);
  }
  if (need > arena_bytes_ || !arena_.p) {
    arena_.alloc(std::max<size_t>(need, 256), true);
    arena_bytes_ = std::max<size_t>(need, 256);
  }
}

// Peer-store layout, identical on every rank: per rank r, send regions of its
// same-rank pairs (zero copy) then receive regions of remote sources, all keys
// sharing one region (exchanges are sequential and the consumed flags order
// reuse), each pair sized for its widest possible plan so no plan change moves or
// grows an arena; then 2 * world flag words.
template <typename T>
void Engine<T>::p2p_layout() {
  const int64_t K = int64_t(keys_.size()), ppr = P_ / s_.world;
  const int wb = s_.bit_mode == kFp ? 0 : s_.bit_mode == kFixed ? s_.fixed_bits : 8;
  auto worst = [&](int64_t k, int64_t p, int64_t q) {
    return uint64_t(msgs_[k][p][q].ids.size()) *
           qgnn_chunk_wire_bytes(uint64_t(keys_[k].dim), wb, s_.layout, dtype_);
  };
  auto al = [](uint64_t x) { return (x + 255) / 256 * 256; };
  send_base_.assign(K, std::vector<std::vector<uint64_t>>(P_, std::vector<uint64_t>(P_, 0)));
  recv_base_ = send_base_;
  p2p_recv_ = send_base_;
  flags_off_.assign(s_.world, 0);
  for (int r = 0; r < s_.world; ++r) {
    const int64_t a = r * ppr, b = a + ppr;
    uint64_t need = 0;
    for (int64_t k = 0; k < K; ++k) {
      uint64_t o = 0;
      for (int64_t p = a; p < b; ++p)
        for (int64_t q = a; q < b; ++q) {
          if (q == p) continue;
          if (r == s_.rank) send_base_[k][p][q] = recv_base_[k][q][p] = o;
          o = al(o + worst(k, p, q));
        }
      for (int64_t q = a; q < b; ++q)
        for (int64_t p = 0; p < P_; ++p) {
          if (p >= a && p < b) continue;
          p2p_recv_[k][q][p] = o;
          if (r == s_.rank) recv_base_[k][q][p] = o;
          o = al(o + worst(k, p, q));
        }
      need = std::max(need, o);
    }
    flags_off_[r] = al(need);
  }
  const size_t bytes = flags_off_[s_.rank] + size_t(2 * s_.world) * sizeof(uint64_t);
  if (!arena_.p) {  // zeroed: all flags start at 0
    arena_.alloc(bytes, true);
    arena_bytes_ = bytes;
  }
  QGNN_REQUIRE(bytes <= arena_bytes_, QGNN_EPROTOCOL, "peer-store arena cannot grow");
}

// Map every peer's arena: the loopback group's engines directly, other processes
// through CUDA IPC handles all-gathered over NCCL.  Then the flag words this rank
// signals: slot `rank` of every peer's ready block and of its consumed block.
template <typename T>
void Engine<T>::p2p_connect() {
  const int W = s_.world;
  peer_arena_.assign(W, nullptr);
  ipc_opened_.assign(W, false);
  peer_arena_[s_.rank] = arena_.p;
  if (loop_) {
    LoopGroup& G = *loop_;
    G.barrier();  // every rank's arena exists
    for (int r = 0; r < W; ++r) peer_arena_[r] = static_cast<Engine<T>*>(G.engines[r])->arena_.p;
    G.barrier();
  } else {
    cudaIpcMemHandle_t h;
    QGNN_CUDA(cudaIpcGetMemHandle(&h, arena_.p));
    constexpr int64_t kH = sizeof(cudaIpcMemHandle_t);
    DBuf<uint8_t> hs;
    hs.alloc(size_t(kH * W), true);
    QGNN_CUDA(cudaMemcpy(hs.p + kH * s_.rank, &h, kH, cudaMemcpyHostToDevice));
    allgather_dev(hs.p, kH, s_main_);
    QGNN_CUDA(cudaStreamSynchronize(s_main_));
    std::vector<cudaIpcMemHandle_t> all(W);
    QGNN_CUDA(cudaMemcpy(all.data(), hs.p, size_t(kH * W), cudaMemcpyDeviceToHost));
    for (int r = 0; r < W; ++r) {
      if (r == s_.rank) continue;
      void* p = nullptr;
      QGNN_CUDA(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
      peer_arena_[r] = static_cast<uint8_t*>(p);
      ipc_opened_[r] = true;
    }
  }
  std::vector<uint64_t*> rd(W, nullptr), cs(W, nullptr);
  for (int r = 0; r < W; ++r) {
    if (r == s_.rank) continue;
    auto* f = reinterpret_cast<uint64_t*>(peer_arena_[r] + flags_off_[r]);
    rd[r] = f + s_.rank;
    cs[r] = f + W + s_.rank;
  }
  sig_ready_.upload(rd);
  sig_cons_.upload(cs);
}

// Before this rank's first K1 store of the next exchange: publish that every
// earlier exchange has been read here (the consumers precede this in stream
// order), then wait until every peer has read the previous one out of the
// regions these stores overwrite.
template <typename T>
void Engine<T>::p2p_begin_send() {
  const int W = s_.world;
  k_p2p_signal<<<1, 32 * unsigned(ceil_div(W, 32)), 0, s_main_>>>(sig_cons_.p, W, xseq_);
  check_launch("k_p2p_signal");
  auto* flags = reinterpret_cast<const uint64_t*>(arena_.p + flags_off_[s_.rank]);
  k_p2p_wait<<<1, 32 * unsigned(ceil_div(W, 32)), 0, s_main_>>>(flags + W, W, s_.rank, xseq_,
                                                                  p2p_timeout_ns(), ctx_->d_err);
  check_launch("k_p2p_wait");
  launches_ += 2;
  send_open_ = true;
}

template <typename T>
void Engine<T>::upload_key_meta(int k) {
  // message lists never change: rows / ids / destinations (and the windows)
  // are uploaded once; widths and wire offsets follow every plan
  const KeyInfo& K = keys_[k];
  par_parts([&](size_t ip) {
    PartDev& D = *parts_dev_[ip];
    const int64_t p = D.id;
    const View& V = D.view;
    auto& S = D.snd[k];
    std::vector<uint8_t> bits;
    std::vector<uint64_t> off;
    const bool fresh = !S.rows.p;
    std::vector<int32_t> rows;
    std::vector<uint32_t> ids;
    std::vector<uint16_t> set;
    S.q_begin.assign(P_ + 1, 0);
    for (int64_t q = 0; q < P_; ++q) {
      S.q_begin[q] = int64_t(bits.size());
      if (q == p) continue;
      const PairMsgs& m = msgs_[k][p][q];
      for (size_t i = 0; i < m.ids.size(); ++i) {
        if (fresh) {
          rows.push_back(K.bwd ? int32_t(V.device_slot_offset[q] + int64_t(i))
                               : V.gpu_row(m.ids[i]));
          ids.push_back(m.ids[i]);
          set.push_back(uint16_t(q));
        }
        bits.push_back(m.bits[i]);
        const int64_t rq = q / (P_ / s_.world);
        if (p2p_ && rq != s_.rank)  // straight into the receiver's arena (64-bit wrap)
          off.push_back(uint64_t(reinterpret_cast<uintptr_t>(peer_arena_[rq])) +
                        p2p_recv_[k][q][p] + m.off[i] -
                        uint64_t(reinterpret_cast<uintptr_t>(arena_.p)));
        else
          off.push_back(send_base_[k][p][q] + m.off[i]);
      }
    }
    S.q_begin[P_] = int64_t(bits.size());
    S.n = int64_t(bits.size());
    if (fresh) {
      S.rows.upload(rows);
      S.ids.upload(ids);
      S.set.upload(set);
      S.keys = keys_all_.p + (size_t(k) * parts_dev_.size() + size_t(p - p0_)) * size_t(P_);
      S.wlo.alloc(std::max<int64_t>(1, S.n), false);
      S.whi.alloc(std::max<int64_t>(1, S.n), false);
      if (S.n)
        k_fill2<T><<<unsigned(ceil_div(S.n, 256)), 256, 0, s_main_>>>(
            S.wlo.p, T(INFINITY), S.whi.p, T(-INFINITY), S.n);
    }
    S.bits.upload(bits);
    S.off.upload(off);

    auto& R = D.rcv[k];
    const bool rfresh = !R.dst.p;
    std::vector<int32_t> dst;
    std::vector<uint8_t> rb;
    std::vector<uint64_t> ro;
    std::vector<uint32_t> env;
    const bool gpu_layout = s_.layout == QGNN_WIRE_GPU;
    R.p_begin.assign(P_ + 1, 0);
    for (int64_t src = 0; src < P_; ++src) {
      R.p_begin[src] = int64_t(rb.size());
      if (src == p) continue;
      const PairMsgs& m = msgs_[k][src][p];
      for (size_t i = 0; i < m.ids.size(); ++i) {
        if (rfresh)
          dst.push_back(K.bwd ? V.gpu_row(m.ids[i])
                              : int32_t(V.device_slot_offset[src] + int64_t(i)));
        rb.push_back(m.bits[i]);
        ro.push_back(recv_base_[k][p][src] + m.off[i]);
        if (gpu_layout)  // the receiver's expectation: (src, this partition, its plan version)
          env.push_back((uint32_t(src) & 0xffu) | (uint32_t(p) & 0xffu) << 8 |
                        (uint32_t(plan_version_) & 0xffu) << 16);
      }
    }
    R.p_begin[P_] = int64_t(rb.size());
    R.n = int64_t(rb.size());
    if (rfresh) {
      if (K.bwd) {  // destination rows with their messages in ascending source order
        std::vector<int32_t> order(dst.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t a, int32_t b) { return dst[a] < dst[b]; });
        std::vector<int32_t> rws, ptr{0};
        for (size_t i = 0; i < order.size(); ++i) {
          if (i == 0 || dst[order[i]] != dst[order[i - 1]]) {
            if (i) ptr.push_back(int32_t(i));
            rws.push_back(dst[order[i]]);
          }
        }
        ptr.push_back(int32_t(order.size()));
        if (rws.empty()) ptr.assign(1, 0);
        R.acc_rows.upload(rws);
        R.acc_ptr.upload(ptr);
        R.acc_msg.upload(order);
        R.n_acc_rows = int64_t(rws.size());
      }
      R.dst.upload(dst.empty() ? std::vector<int32_t>{0} : dst);
    }
    R.bits.upload(rb);
    R.off.upload(ro);
    if (gpu_layout) R.env.upload(env);
    if constexpr (sizeof(T) == 4) {
      // chunk words hold offset / 16 in 30 bits: arenas up to 16 GiB
      const bool words = gpu_layout && direct_words_enabled() && arena_bytes_ <= (size_t(1) << 34);
      if (words && !K.bwd && V.remote_nnz() > 0) {
        if (!R.words.p) R.words.alloc(size_t(V.remote_nnz()), false);
        encode_chunk_words(D.rslot.p, V.remote_nnz(), R.off.p, R.bits.p, R.words.p, s_main_);
      } else if (words && K.bwd && R.n > 0 && k3_words_enabled()) {  // per scatter-add entry
        if (!R.words.p) R.words.alloc(size_t(R.n), false);
        encode_chunk_words(R.acc_msg.p, R.n, R.off.p, R.bits.p, R.words.p, s_main_);
      } else {
        R.words.release();  // slot-indexed gathers / message-indexed scatter-add
      }
    }
  });
}

template <typename T>
void Engine<T>::prepare_epoch() {
  if (s_.bit_mode == kUniform) {
    compute_bits_uniform();
    for (size_t k = 0; k < keys_.size(); ++k)
      for (int64_t p = 0; p < P_; ++p)
        for (int64_t q = 0; q < P_; ++q)
          if (p != q) layout_pair(int(k), int(p), int(q));
    arena_layout();
    for (size_t k = 0; k < keys_.size(); ++k) upload_key_meta(int(k));
  }
  // RNG stream of each encoded set: root.fork({0x2, epoch, key_code, src, dst}) (engine.hpp:497),
  // every key x hosted partition x destination staged in pinned memory, one copy (the
  // previous epoch, and with it its copy, has finished: finish_epoch waited for it)
  {
    const size_t np = parts_dev_.size();
    for (size_t k = 0; k < keys_.size(); ++k)
      for (size_t i = 0; i < np; ++i)
        for (int64_t q = 0; q < P_; ++q) {
          uint64_t key = root_;
          for (uint64_t c : {uint64_t(0x2), epoch_, keys_[k].code, uint64_t(parts_dev_[i]->id),
                             uint64_t(q)})
            key = rng_fork(key, c);
          keys_host_[(k * np + i) * size_t(P_) + size_t(q)] = key;
        }
    QGNN_CUDA(cudaMemcpyAsync(keys_all_.p, keys_host_, keys_.size() * np * P_ * sizeof(uint64_t),
                              cudaMemcpyHostToDevice, s_main_));
  }
  if (bits_dirty_) recount_bits();  // widths change only with the plan (or per epoch, uniform)
}

// ------------------------------------------------------------ data path ---
template <typename T>
void Engine<T>::quantize(PartDev& D, int k, const T* src, int64_t ld, cudaStream_t sq) {
  if (p2p_ && !send_open_) p2p_begin_send();
  auto& S = D.snd[k];
  if (S.n == 0) return;
  if (!sq) sq = s_main_;
  const int64_t dim = keys_[k].dim;
  kbegin(QGNN_K_QUANT, sq);
  const int st = qgnn_quantize_pack(ctx_, src, dtype_, ld, dim, S.n, S.rows.p, S.ids.p, S.bits.p,
                                    S.off.p, S.set.p, S.keys, s_.layout, arena_.p, S.wlo.p,
                                    S.whi.p, envelope(D.id), sq);
  if (st) throw Status(st, qgnn_last_error());
  // algorithmic bytes: rows read once per message + packed chunks + metadata
  double bytes = 0;
  for (int64_t q = 0; q < P_; ++q)
    if (q != D.id) bytes += double(msgs_[k][D.id][q].bytes);
  bytes += double(S.n) * (double(dim) * sizeof(T) + 4 + 4 + 1 + 8 + 2 + 2 * sizeof(T));
  kend(QGNN_K_QUANT, bytes, sq);
}

// receive (engine.hpp:607-618): decode every source straight into the halo
template <typename T>
void Engine<T>::decode_halo(int k, int64_t din, int64_t ldi, cudaStream_t st) {
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    auto& R = D.rcv[k];
    if (!R.n) continue;
    kbegin(QGNN_K_DEQUANT, st);
    const int rc = qgnn_dequant_scatter(ctx_, arena_.p, R.n, din, R.bits.p, R.off.p, s_.layout,
                                        R.dst.p, 0, D.halo.p, dtype_, ldi, R.env.p, st);
    if (rc) throw Status(rc, qgnn_last_error());
    double bytes = double(R.n) * (din * sizeof(T) + 4 + 1 + 8);
    for (int64_t src = 0; src < P_; ++src)
      if (src != D.id) bytes += double(msgs_[k][src][D.id].bytes);
    kend(QGNN_K_DEQUANT, bytes, st);
  }
}

// Grouped point-to-point exchange of the remote pairs on the comm stream.
template <typename T>
void Engine<T>::exchange(int k) {
  if (zero_copy()) return;  // every pair is on this GPU: zero-copy
  if (p2p_) {  // the stores are done: tell every peer (no bytes move here)
    if (!send_open_) p2p_begin_send();
    ++xseq_;
    // test hook (QGNN_TEST_P2P_DROP=r): rank r never publishes its first exchange
    const char* de = std::getenv("QGNN_TEST_P2P_DROP");
    const int drop = de ? std::atoi(de) : -1;
    if (!(drop == s_.rank && xseq_ == 1))
      k_p2p_signal<<<1, 32 * unsigned(ceil_div(s_.world, 32)), 0, s_main_>>>(sig_ready_.p,
                                                                            s_.world, xseq_);
    check_launch("k_p2p_signal");
    ++launches_;
    send_open_ = false;
    if (s_.overlap == 0) wait_exchange();
    return;
  }
  QGNN_CUDA(cudaEventRecord(ev_q_, s_main_));
  QGNN_CUDA(cudaStreamWaitEvent(s_comm_, ev_q_, 0));
  const int64_t ppr = P_ / s_.world;
  if (s_.kstats) {
    kbegin(QGNN_K_EXCHANGE);
    QGNN_CUDA(cudaEventRecord(ev_pool_[ev_next_].first, s_comm_));
  }
  // Grouped p2p schedule.  Inside one NCCL group the i-th send A->B is matched
  // with the i-th receive B<-A, so both sides enumerate a rank pair's messages in
  // the same (source partition p, destination partition q) order.
  std::vector<std::array<int64_t, 4>> sends, recvs;  // (peer rank, p, q, bytes)
  // self_xfer_ (one GPU, QGNN transport "nccl"): same-GPU pairs go through NCCL
  // self send/receive too, into their own receive regions
  for (int64_t p = p0_; p < p1_; ++p)
    for (int64_t q = 0; q < P_; ++q) {
      if (q == p || (q >= p0_ && q < p1_ && !self_xfer_)) continue;
      const uint64_t nb = msgs_[k][p][q].bytes;
      if (nb) sends.push_back({q / ppr, p, q, int64_t(nb)});
    }
  for (int64_t p = 0; p < P_; ++p) {
    if (p >= p0_ && p < p1_ && !self_xfer_) continue;
    for (int64_t q = p0_; q < p1_; ++q) {
      if (q == p) continue;
      const uint64_t nb = msgs_[k][p][q].bytes;
      if (nb) recvs.push_back({p / ppr, p, q, int64_t(nb)});
    }
  }
  double bytes = 0;
  for (const auto& e : sends) bytes += double(e[3]);
  if (loop_) {
    LoopGroup& G = *loop_;
    G.ev[s_.rank] = ev_q_;
    G.sends[s_.rank] = sends;
    G.recvs[s_.rank] = recvs;
    G.barrier();  // every rank's K1 enqueued; its receive regions free after ev_q_
    // the NCCL matching rule, checked for every rank pair (by every rank, so all
    // ranks agree on the outcome): b's receives from a, in order, are exactly
    // a's sends to b, in order
    bool match = true;
    for (int a = 0; a < s_.world; ++a)
      for (int b = 0; b < s_.world; ++b) {
        if (a == b) continue;
        std::vector<std::array<int64_t, 4>> sent, got;
        for (const auto& e : G.sends[a])
          if (e[0] == b) sent.push_back({e[1], e[2], e[3], 0});
        for (const auto& e : G.recvs[b])
          if (e[0] == a) got.push_back({e[1], e[2], e[3], 0});
        match &= sent == got;
      }
    for (int r = 0; r < s_.world; ++r)
      if (r != s_.rank) QGNN_CUDA(cudaStreamWaitEvent(s_comm_, G.ev[r], 0));
    for (const auto& e : sends) {
      auto* peer = static_cast<Engine<T>*>(G.engines[e[0]]);
      QGNN_CUDA(cudaMemcpyAsync(peer->arena_.p + peer->recv_base_[k][e[2]][e[1]],
                                arena_.p + send_base_[k][e[1]][e[2]], size_t(e[3]),
                                cudaMemcpyDeviceToDevice, s_comm_));
    }
    QGNN_CUDA(cudaEventRecord(ev_x_, s_comm_));
    G.ev2[s_.rank] = ev_x_;
    G.barrier();  // all copies enqueued (and every rank done reading G.sends)
    QGNN_REQUIRE(match, QGNN_EPROTOCOL,
                 "exchange: grouped send/receive order differs between ranks");
    peer_x_.clear();
    for (int r = 0; r < s_.world; ++r)
      if (r != s_.rank) peer_x_.push_back(G.ev2[r]);
    kend(QGNN_K_EXCHANGE, bytes, s_comm_, 0);
    if (s_.overlap == 0) wait_exchange();
    return;
  }
  QGNN_NCCL(nccl().GroupStart());
  for (const auto& e : sends)
    QGNN_NCCL(nccl().Send(arena_.p + send_base_[k][e[1]][e[2]], size_t(e[3]), ncclUint8,
                          int(e[0]), comm_, s_comm_));
  for (const auto& e : recvs)
    QGNN_NCCL(nccl().Recv(arena_.p + recv_base_[k][e[2]][e[1]], size_t(e[3]), ncclUint8,
                          int(e[0]), comm_, s_comm_));
  QGNN_NCCL(nccl().GroupEnd());
  kend(QGNN_K_EXCHANGE, bytes, s_comm_, 0);
  QGNN_CUDA(cudaEventRecord(ev_x_, s_comm_));
  if (s_.overlap == 0) wait_exchange();  // serialized schedule: nothing overlaps the exchange
}

// Receivers wait for the exchange of the current key: NCCL completes on our comm
// stream; loopback copies were issued on the senders' comm streams.
template <typename T>
void Engine<T>::wait_exchange() {
  if (zero_copy()) return;
  if (p2p_) {  // every peer's stores of this exchange have landed here
    auto* flags = reinterpret_cast<const uint64_t*>(arena_.p + flags_off_[s_.rank]);
    k_p2p_wait<<<1, 32 * unsigned(ceil_div(s_.world, 32)), 0, s_main_>>>(
        flags, s_.world, s_.rank, xseq_, p2p_timeout_ns(), ctx_->d_err);
    check_launch("k_p2p_wait");
    ++launches_;
    return;
  }
  if (loop_) {
    for (cudaEvent_t e : peer_x_) QGNN_CUDA(cudaStreamWaitEvent(s_main_, e, 0));
    // and for this rank's own outgoing copies: every key's send regions start at
    // arena offset 0, so the next K1 on s_main_ must not overwrite them while
    // s_comm_ is still reading them
    QGNN_CUDA(cudaStreamWaitEvent(s_main_, ev_x_, 0));
    return;
  }
  QGNN_CUDA(cudaStreamWaitEvent(s_main_, ev_x_, 0));
}

// In-place all-gather: rank r contributes base[r * slice, (r + 1) * slice).
template <typename T>
template <typename X>
void Engine<T>::allgather_dev(X* base, int64_t slice, cudaStream_t st) {
  if (s_.world == 1 || slice == 0) return;
  if (!loop_) {
    ncclDataType_t dt = ncclUint8;
    size_t count = size_t(slice) * sizeof(X);
    QGNN_NCCL(nccl().AllGather(base + s_.rank * slice, base, count, dt, comm_, st));
    return;
  }
  LoopGroup& G = *loop_;
  QGNN_CUDA(cudaEventRecord(ev_c_, st));
  G.ptr[s_.rank] = base;
  G.ev[s_.rank] = ev_c_;
  G.barrier();
  for (int r = 0; r < s_.world; ++r)
    if (r != s_.rank) QGNN_CUDA(cudaStreamWaitEvent(s_comm_, G.ev[r], 0));
  QGNN_CUDA(cudaStreamWaitEvent(s_comm_, ev_c_, 0));
  for (int r = 0; r < s_.world; ++r)
    if (r != s_.rank)
      QGNN_CUDA(cudaMemcpyAsync(static_cast<X*>(G.ptr[r]) + s_.rank * slice, base + s_.rank * slice,
                                size_t(slice) * sizeof(X), cudaMemcpyDeviceToDevice, s_comm_));
  QGNN_CUDA(cudaEventRecord(ev_d_, s_comm_));
  G.ev2[s_.rank] = ev_d_;
  G.barrier();
  for (int r = 0; r < s_.world; ++r)
    if (r != s_.rank) QGNN_CUDA(cudaStreamWaitEvent(st, G.ev2[r], 0));
  QGNN_CUDA(cudaStreamWaitEvent(st, ev_d_, 0));  // our own slice has been read out
}

#define QGNN_CALL(x)                                 \
  do {                                               \
    const int st_ = (x);                             \
    if (st_) throw Status(st_, qgnn_last_error());   \
  } while (0)

template <typename T>
bool Engine<T>::packed_fwd(int k, int64_t din, int64_t ldi) {
  if constexpr (sizeof(T) != 4) {
    return false;
  } else {
    static const bool on = [] {
      const char* e = std::getenv("QGNN_PACKED_HALO");  // 0: K3 into the fp32 halo (round 1)
      return !e || std::atoi(e) != 0;
    }();
    if (!on || s_.layout != QGNN_WIRE_GPU || keys_[k].bwd) return false;
    for (auto& up : parts_dev_)
      if (up->view.n_marginal &&
          !spmm_packed_ok(int(round_up(din, 4)), &up->hub_fm.plan, up->h[k].p, ldi))
        return false;
    return true;
  }
}

template <typename T>
PackedHalo Engine<T>::packed_halo(PartDev& D, int k, int64_t din) {
  auto& R = D.rcv[k];
  PackedHalo pk;
  pk.arena = arena_.p;
  pk.off = R.off.p;
  pk.bits = R.bits.p;
  pk.env = R.env.p;
  pk.dim = int(din);
  pk.err = ctx_->d_err;
  pk.direct = R.words.p != nullptr;
  if (pk.direct)  // the entries are chunk words: the headers are checked here, once each
    check_chunk_headers(arena_.p, R.off.p, R.bits.p, R.env.p, R.n, int(din), ctx_->d_err,
                        s_main_);
  return pk;
}

template <typename T>
void Engine<T>::forward_layer(int l) {
  const int t = l - 1;
  const int k = t;  // forward key index
  const int64_t din = dims_[t], dout = dims_[l];
  const int64_t ldi = ld_of(din), ldo = ld_of(dout);
  const int relu = l < L_ ? 1 : 0;
  // One GPU, in-line schedule: nothing overlaps the central rows, so each
  // partition's transform runs once over central + marginal rows (contiguous in
  // hagg) after its marginal aggregation: one GEMM launch instead of two.
  const bool one_gemm = zero_copy() && !side_overlap() && merge_gemm_enabled();
  // layer_forward_rows (model.hpp:90-124) for rows [r0, r0 + n): the GEMM with the
  // ReLU epilogue, or (LayerNorm / dropout) z -> act[t], then the chain -> h[l]
  const bool chain = chain_layer(l);
  // the next layer's ReLU-backward mask as bits (hbits)
  const bool bits = relu_fused() && l < L_ && relu && !chain && mask_bits_enabled();
  for (auto& up : parts_dev_)  // this epoch's bits of h[l] are valid once every row is written
    if (!up->hbits_rows.empty()) up->hbits_rows[l] = 0;
  auto transform = [&](PartDev& D, int64_t r0, int64_t n) {
    kbegin(QGNN_K_GEMM_FWD);
    bool done = false;
    if constexpr (sizeof(T) == 4) {
      if (bits) {
        if (dense_forward_bits_f32(ctx_, D.hagg[t].p, ldi, w_.p + woff_[t], din, dout, r0, n,
                                   D.h[l].p, ldo, D.hbits[l].p, hbits_ld(l), s_main_))
          D.hbits_rows[l] += n;
        done = true;
      }
    }
    if (!done)
      QGNN_CALL(qgnn_dense_forward(ctx_, dtype_, D.hagg[t].p, ldi, w_.p + woff_[t], din, dout,
                                   nullptr, r0, n, chain ? 0 : relu,
                                   chain ? D.act[t].p : D.h[l].p, ldo, s_main_));
    kend(QGNN_K_GEMM_FWD, double(n) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(n), din, dout));
    if (!chain) return;
    kbegin(QGNN_K_ELEMWISE);
    chain_forward<T>(D.act[t].p, D.act[t].p, ldo, D.h[l].p, ldo,
                     s_.layer_norm ? D.istd[t].p : nullptr, int(dout), r0, n, chain_args(D, l),
                     s_main_);
    kend(QGNN_K_ELEMWISE, double(n) * dout * sizeof(T) * 3, s_main_);
  };
  // central rows (engine.hpp:598-605): during the exchange
  auto central = [&](PartDev& D) {
    const int64_t nc = D.view.n_central;
    if (!nc) return;
    kbegin(QGNN_K_SPMM_FWD);
    const int nk = spmm(din, D.h[t].p, ldi, nullptr, 0, D.self_alpha.p, D.lptr.p, D.lcol.p,
                        D.lafwd.p, nullptr, nullptr, nullptr, 0, nc, D.hagg[t].p, ldi, &D.hub_fc.plan);
    const double nnz = double(D.view.local_ptr[nc]);
    kend(QGNN_K_SPMM_FWD, nc * (16.0 + din * sizeof(T)) + nnz * (4 + sizeof(T)) +
                              double(D.view.src_rows_central) * din * sizeof(T), s_main_, nk,
         (nnz + nc) * din * sizeof(T));
    if (one_gemm) return;
    transform(D, 0, nc);
  };
  // With features still in flight (first layer after set_features) or with no
  // remote exchange (one GPU), each partition's encode and central rows run as
  // soon as its rows exist; otherwise every encode precedes the exchange, which
  // the central rows then overlap.
  const bool feats = t == 0 && feat_pending_;
  const bool pkd = packed_fwd(k, din, ldi);  // no K3: the marginal SpMM decodes in registers
  if (side_overlap() && !feats) {
    // one GPU: encode + decode on the side stream while the central rows run
    fork_side();
    for (auto& up : parts_dev_) quantize(*up, k, up->h[t].p, ldi, s_comm_);  // fwd_send
    if (!pkd) decode_halo(k, din, ldi, s_comm_);
    for (auto& up : parts_dev_) central(*up);
    join_side();
  } else {
    if (feats || zero_copy()) {
      for (auto& up : parts_dev_) {
        if (feats) gather_features(*up);
        if (feats && up.get() == parts_dev_.back().get())
          QGNN_CUDA(cudaEventRecordWithFlags(ev_feat_free_, s_main_,  // staging matrix consumed
                                             capturing_ ? cudaEventRecordExternal : 0));
        quantize(*up, k, up->h[t].p, ldi);  // fwd_send (engine.hpp:566-588)
        central(*up);
      }
      feat_pending_ = false;
      exchange(k);
    } else {
      for (auto& up : parts_dev_) quantize(*up, k, up->h[t].p, ldi);  // fwd_send
      exchange(k);
      for (auto& up : parts_dev_) central(*up);
    }
    wait_exchange();
    if (!pkd) decode_halo(k, din, ldi, s_main_);
  }
  // marginal rows (engine.hpp:622-623)
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t nc = D.view.n_central, nm = D.view.n_marginal;
    if (one_gemm && !nm && nc) transform(D, 0, nc);  // all rows central: deferred transform
    if (!nm) continue;
    kbegin(QGNN_K_SPMM_FWD);
    const PackedHalo pk = pkd ? packed_halo(D, k, din) : PackedHalo{};
    const int nk = spmm(din, D.h[t].p, ldi, pkd ? nullptr : D.halo.p, ldi, D.self_alpha.p, D.lptr.p,
                        D.lcol.p, D.lafwd.p, D.rptr.p,
                        pkd && pk.direct ? D.rcv[k].words.p : D.rslot.p, D.ralpha.p, nc, nm,
                        D.hagg[t].p, ldi, &D.hub_fm.plan, nullptr, 0, pkd ? &pk : nullptr);
    const double nnz = double(D.view.local_ptr[nc + nm] - D.view.local_ptr[nc]) +
                       double(D.view.remote_nnz());
    // remote source rows: fp32 halo rows, or their packed chunks (+ offset, width)
    double slot_bytes = double(din * sizeof(T));
    if (pkd && D.rcv[k].n) {
      double in = 0;
      for (int64_t src = 0; src < P_; ++src)
        if (src != D.id) in += double(msgs_[k][src][D.id].bytes);
      slot_bytes = in / double(D.rcv[k].n) + 9;
    }
    kend(QGNN_K_SPMM_FWD, nm * (24.0 + din * sizeof(T)) + nnz * (4 + sizeof(T)) +
                              double(D.view.src_rows_marginal) * din * sizeof(T) +
                              double(D.view.src_slots_marginal) * slot_bytes, s_main_, nk,
         (nnz + nm) * din * sizeof(T));
    const int64_t g0 = one_gemm ? 0 : nc, gn = one_gemm ? nc + nm : nm;
    transform(D, g0, gn);
  }
}

// loss_phase (engine.hpp:647-659)
template <typename T>
void Engine<T>::loss_phase() {
  const int64_t C = dims_[L_], ldc = ld_of(C);
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    QGNN_CUDA(cudaMemsetAsync(D.dh.p, 0, D.view.num_owned * ldc * sizeof(T), s_main_));
    QGNN_CUDA(cudaMemsetAsync(D.loss, 0, sizeof(double), s_main_));
    QGNN_CUDA(cudaMemsetAsync(D.correct, 0, 2 * sizeof(unsigned long long), s_main_));
    kbegin(QGNN_K_ELEMWISE);
    if constexpr (sizeof(T) == 4) {
      loss_f32(ctx_, D.h[L_].p, ldc, int(C), D.labels.p, D.loss_rows.p, D.n_train, D.n_val,
               D.n_test, 1.0 / double(global_train_), D.dh.p, ldc, D.loss, D.correct, s_main_);
      kend(QGNN_K_ELEMWISE, double(D.view.num_owned) * C * sizeof(T) * 2, s_main_, 2);
      continue;
    }
    if (D.n_train)
      QGNN_CALL(qgnn_masked_ce(ctx_, dtype_, D.h[L_].p, ldc, C, D.labels.p, D.train_rows.p,
                               D.n_train, 1.0 / double(global_train_), D.dh.p, ldc, D.loss,
                               s_main_));
    if (D.n_val)
      QGNN_CALL(qgnn_count_correct(ctx_, dtype_, D.h[L_].p, ldc, C, D.labels.p, D.val_rows.p,
                                   D.n_val, D.correct, s_main_));
    if (D.n_test)
      QGNN_CALL(qgnn_count_correct(ctx_, dtype_, D.h[L_].p, ldc, C, D.labels.p, D.test_rows.p,
                                   D.n_test, D.correct + 1, s_main_));
    kend(QGNN_K_ELEMWISE, double(D.view.num_owned) * C * sizeof(T) * 2, s_main_,
         (D.n_train ? 2 : 0) + (D.n_val ? 1 : 0) + (D.n_test ? 1 : 0));
  }
}

template <typename T>
void Engine<T>::backward_layer(int l) {
  const int t = l - 1;
  const int k = int(L_) + t - 1;  // backward key index (keys: fwd 0..L-1, bwd 1..L-1)
  const int64_t din = dims_[t], dout = dims_[l];
  const int64_t ldi = ld_of(din), ldo = ld_of(dout);
  // fp32: the ReLU backward of this layer was folded into whoever produced dh,
  // and this layer's producers of dh_next are masked by h[t] (relu_mask4)
  const bool relu = l < L_ && !dh_masked_;
  const bool mk = relu_fused() && t >= 1;
  // LayerNorm / dropout: layer_backward_rows as chain.cu (dz from dh, act_in, h, inv_std)
  const bool chain = chain_layer(l);
  auto chain_bwd = [&](PartDev& D, int64_t r0, int64_t n) {
    kbegin(QGNN_K_ELEMWISE);
    chain_backward<T>(D.dh.p, ldo, D.act[t].p, ldo, D.h[l].p, ldo,
                      s_.layer_norm ? D.istd[t].p : nullptr, D.dz.p, ldo, int(dout), r0, n,
                      chain_args(D, l), s_main_);
    kend(QGNN_K_ELEMWISE, double(n) * dout * sizeof(T) * 4, s_main_);
  };
  const T* W = w_.p + woff_[t];
  // One GPU, in-line schedule (nothing overlaps the exchange): the input gradient of
  // the central rows runs in the same GEMM launch as the marginal rows' (bit-identical)
  const bool one_dgrad = zero_copy() && !side_overlap() && merge_gemm_enabled() && !chain &&
                         !relu && one_dgrad_enabled();
  // bwd_send (engine.hpp:661-688): marginal chain, remote partials, encode
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t nc = D.view.n_central, nm = D.view.n_marginal;
    const int64_t g0 = one_dgrad ? 0 : nc, gn = one_dgrad ? nc + nm : nm;
    const T* dz = D.dh.p;
    if (chain) {
      chain_bwd(D, nc, nm);
      dz = D.dz.p;
    } else if (relu) {
      kbegin(QGNN_K_ELEMWISE);
      QGNN_CALL(qgnn_relu_backward(ctx_, dtype_, D.h[l].p, ldo, D.dh.p, ldo, dout, nc, nm, D.dz.p,
                                   ldo, s_main_));
      kend(QGNN_K_ELEMWISE, double(nm) * dout * sizeof(T) * 3, s_main_);
      dz = D.dz.p;
    }
    kbegin(QGNN_K_GEMM_DGRAD);
    QGNN_CALL(qgnn_dense_input_grad(ctx_, dtype_, dz, ldo, W, din, dout, nullptr, g0, gn, D.gbar.p,
                                    ldi, s_main_));
    kend(QGNN_K_GEMM_DGRAD, double(gn) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(gn), din, dout));
    if (D.view.num_remote) {
      kbegin(QGNN_K_PARTIALS);
      const int nk = spmm(din, D.gbar.p, ldi, nullptr, 0, nullptr, D.sptr.p, D.srow.p, D.salpha.p,
                          nullptr, nullptr, nullptr, 0, D.view.num_remote, D.partials.p, ldi,
                          &D.hub_part.plan);
      kend(QGNN_K_PARTIALS, double(D.view.num_remote) * (8 + din * sizeof(T)) +
                                double(D.view.remote_nnz()) * (4 + sizeof(T)) +
                                double(D.view.n_marginal) * din * sizeof(T),
           s_main_, nk, double(D.view.remote_nnz()) * din * sizeof(T));
    }
    if (!side_overlap()) quantize(D, k, D.partials.p, ldi);
  }
  if (side_overlap()) {  // one GPU: encode on the side stream during bwd_finish
    fork_side();
    for (auto& up : parts_dev_) quantize(*up, k, up->partials.p, ldi, s_comm_);
  } else {
    exchange(k);
  }
  // bwd_finish (engine.hpp:690-740)
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t nc = D.view.n_central, no = D.view.num_owned;
    const T* dz = D.dh.p;
    if (chain) {
      chain_bwd(D, 0, nc);
      dz = D.dz.p;
    } else if (relu) {
      kbegin(QGNN_K_ELEMWISE);
      QGNN_CALL(qgnn_relu_backward(ctx_, dtype_, D.h[l].p, ldo, D.dh.p, ldo, dout, 0, nc, D.dz.p,
                                   ldo, s_main_));
      kend(QGNN_K_ELEMWISE, double(nc) * dout * sizeof(T) * 3, s_main_);
      dz = D.dz.p;
    }
    if (!one_dgrad) {
      kbegin(QGNN_K_GEMM_DGRAD);
      QGNN_CALL(qgnn_dense_input_grad(ctx_, dtype_, dz, ldo, W, din, dout, nullptr, 0, nc,
                                      D.gbar.p, ldi, s_main_));
      kend(QGNN_K_GEMM_DGRAD, double(nc) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
           gemm_flops(double(nc), din, dout));
    }
    kbegin(QGNN_K_GEMM_WGRAD);
    T* wg = wgrad_all_.p + D.id * nparams_ + woff_[t];
    QGNN_CALL(qgnn_dense_weight_grad(ctx_, dtype_, D.hagg[t].p, ldi, dz, ldo, din, dout,
                                     dtype_ == QGNN_F64 ? D.ref_order.p : nullptr, 0, no, 0, wg,
                                     s_main_));
    kend(QGNN_K_GEMM_WGRAD, double(no) * (din + dout) * sizeof(T), s_main_,
         dtype_ == QGNN_F64 ? 1 : 2, gemm_flops(double(no), din, dout));
    kbegin(QGNN_K_SPMM_BWD);
    const int nk = spmm(din, D.gbar.p, ldi, nullptr, 0, D.self_alpha.p, D.lptr.p, D.lcol.p,
                        D.labwd.p, nullptr, nullptr, nullptr, 0, no, D.dh_next.p, ldi, &D.hub_bwd.plan,
                        mk ? relu_mask(D, t, ldi).first : nullptr,
                        mk ? relu_mask(D, t, ldi).second : 0);
    kend(QGNN_K_SPMM_BWD, no * (16.0 + (mk ? 2 : 1) * din * sizeof(T)) +
                              double(D.view.local_nnz()) * (4 + sizeof(T)) +
                              double(D.view.src_rows_all) * din * sizeof(T), s_main_, nk,
         double(D.view.local_nnz() + no) * din * sizeof(T));
  }
  if (side_overlap())
    join_side();
  else
    wait_exchange();
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    scatter_add_all(D, k, din, ldi, mk ? relu_mask(D, t, ldi).first : nullptr,
                    mk ? relu_mask(D, t, ldi).second : ldi);
    std::swap(D.dh, D.dh_next);
  }
  dh_masked_ = mk;
}

// Last layer, transform first (fp32 engine, dout < din): y = h W on owned and
// halo rows, then z = A y (dout-wide gathers).  Messages: the same quantized
// rows of h as forward_layer (engine.hpp:566-588).
template <typename T>
void Engine<T>::forward_last_tf(int l) {
  const int t = l - 1;
  const int k = t;
  const int64_t din = dims_[t], dout = dims_[l];
  const int64_t ldi = ld_of(din), ldo = ld_of(dout);
  const T* W = w_.p + woff_[t];
  const bool side = side_overlap();
  // LayerNorm on the last layer: the aggregation lands in act[t] = z, the chain
  // writes h[l] = LN(z) (model.hpp:108-112; linear, no dropout on the last layer)
  const bool chain = chain_layer(l);
  if (side) {  // one GPU: encode + decode on the side stream during the owned-row work
    fork_side();
    for (auto& up : parts_dev_) quantize(*up, k, up->h[t].p, ldi, s_comm_);
    decode_halo(k, din, ldi, s_comm_);
  } else {
    for (auto& up : parts_dev_) quantize(*up, k, up->h[t].p, ldi);
    exchange(k);
  }
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t no = D.view.num_owned, nc = D.view.n_central;
    kbegin(QGNN_K_GEMM_FWD);
    QGNN_CALL(qgnn_dense_forward(ctx_, dtype_, D.h[t].p, ldi, W, din, dout, nullptr, 0, no, 0,
                                 D.dz.p, ldo, s_main_));
    kend(QGNN_K_GEMM_FWD, double(no) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(no), din, dout));
    if (!nc) continue;
    kbegin(QGNN_K_SPMM_FWD);
    const int nk = spmm(dout, D.dz.p, ldo, nullptr, 0, D.self_alpha.p, D.lptr.p, D.lcol.p,
                        D.lafwd.p, nullptr, nullptr, nullptr, 0, nc,
                        chain ? D.act[t].p : D.h[l].p, ldo, &D.hub_fc.plan);
    kend(QGNN_K_SPMM_FWD, nc * (16.0 + dout * sizeof(T)) +
                              double(D.view.local_ptr[nc]) * (4 + sizeof(T)) +
                              double(D.view.src_rows_central) * dout * sizeof(T), s_main_, nk,
         double(D.view.local_ptr[nc] + nc) * dout * sizeof(T));
  }
  if (side) {
    join_side();
  } else {
    wait_exchange();
    decode_halo(k, din, ldi, s_main_);
  }
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t nc = D.view.n_central, nm = D.view.n_marginal, nr = D.view.num_remote;
    if (!nm) continue;
    if (nr) {
      kbegin(QGNN_K_GEMM_FWD);
      QGNN_CALL(qgnn_dense_forward(ctx_, dtype_, D.halo.p, ldi, W, din, dout, nullptr, 0, nr, 0,
                                   D.partials.p, ldo, s_main_));
      kend(QGNN_K_GEMM_FWD, double(nr) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(nr), din, dout));
    }
    kbegin(QGNN_K_SPMM_FWD);
    const int nk = spmm(dout, D.dz.p, ldo, D.partials.p, ldo, D.self_alpha.p, D.lptr.p, D.lcol.p,
                        D.lafwd.p, D.rptr.p, D.rslot.p, D.ralpha.p, nc, nm,
                        chain ? D.act[t].p : D.h[l].p, ldo, &D.hub_fm.plan);
    const double nnz = double(D.view.local_ptr[nc + nm] - D.view.local_ptr[nc]) +
                       double(D.view.remote_nnz());
    kend(QGNN_K_SPMM_FWD, nm * (24.0 + dout * sizeof(T)) + nnz * (4 + sizeof(T)) +
                              double(D.view.src_rows_marginal + D.view.src_slots_marginal) *
                                  dout * sizeof(T), s_main_, nk,
         (nnz + nm) * dout * sizeof(T));
  }
  if (chain)
    for (auto& up : parts_dev_) {
      PartDev& D = *up;
      kbegin(QGNN_K_ELEMWISE);
      chain_forward<T>(D.act[t].p, D.act[t].p, ldo, D.h[l].p, ldo, D.istd[t].p, int(dout), 0,
                       D.view.num_owned, chain_args(D, l), s_main_);
      kend(QGNN_K_ELEMWISE, double(D.view.num_owned) * dout * sizeof(T) * 3, s_main_);
    }
}

// Backward of the transform-first last layer: g = A^T dz (dout-wide), then
// partials = g_halo W^T (the same rows backward_remote_partials(dz W^T) gives,
// aggregate.hpp:152-165), dh_next = g_local W^T, dW = h^T g_local + halo^T g_halo.
template <typename T>
void Engine<T>::backward_last_tf(int l) {
  const int t = l - 1;
  const int k = int(L_) + t - 1;
  const int64_t din = dims_[t], dout = dims_[l];
  const int64_t ldi = ld_of(din), ldo = ld_of(dout);
  const T* W = w_.p + woff_[t];
  const bool mk = relu_fused() && t >= 1;  // ReLU backward of layer t folded into dh_next's producers
  // LayerNorm on the last layer: dz = LN'(dh) first (dropout is never on the last layer)
  const bool chain = chain_layer(l);
  if (chain)
    for (auto& up : parts_dev_) {
      PartDev& D = *up;
      kbegin(QGNN_K_ELEMWISE);
      chain_backward<T>(D.dh.p, ldo, D.act[t].p, ldo, D.h[l].p, ldo, D.istd[t].p, D.dz.p, ldo,
                        int(dout), 0, D.view.num_owned, chain_args(D, l), s_main_);
      kend(QGNN_K_ELEMWISE, double(D.view.num_owned) * dout * sizeof(T) * 4, s_main_);
    }
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t nr = D.view.num_remote;
    if (nr) {
      kbegin(QGNN_K_PARTIALS);
      const int nk = spmm(dout, chain ? D.dz.p : D.dh.p, ldo, nullptr, 0, nullptr, D.sptr.p,
                          D.srow.p, D.salpha.p, nullptr, nullptr, nullptr, 0, nr, D.gpart.p, ldo,
                          &D.hub_part.plan);
      kend(QGNN_K_PARTIALS, double(nr) * (8 + dout * sizeof(T)) +
                                double(D.view.remote_nnz()) * (4 + sizeof(T)) +
                                double(D.view.n_marginal) * dout * sizeof(T),
           s_main_, nk, double(D.view.remote_nnz()) * dout * sizeof(T));
      kbegin(QGNN_K_GEMM_DGRAD);
      QGNN_CALL(qgnn_dense_input_grad(ctx_, dtype_, D.gpart.p, ldo, W, din, dout, nullptr, 0, nr,
                                      D.partials.p, ldi, s_main_));
      kend(QGNN_K_GEMM_DGRAD, double(nr) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(nr), din, dout));
    }
    if (!side_overlap()) quantize(D, k, D.partials.p, ldi);
  }
  if (side_overlap()) {  // one GPU: encode on the side stream during bwd_finish
    fork_side();
    for (auto& up : parts_dev_) quantize(*up, k, up->partials.p, ldi, s_comm_);
  } else {
    exchange(k);
  }
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t no = D.view.num_owned, nr = D.view.num_remote;
    kbegin(QGNN_K_SPMM_BWD);
    const int nk = spmm(dout, chain ? D.dz.p : D.dh.p, ldo, nullptr, 0, D.self_alpha.p, D.lptr.p,
                        D.lcol.p, D.labwd.p, nullptr, nullptr, nullptr, 0, no, D.gbar.p, ldo,
                        &D.hub_bwd.plan);
    kend(QGNN_K_SPMM_BWD, no * (16.0 + dout * sizeof(T)) +
                              double(D.view.local_nnz()) * (4 + sizeof(T)) +
                              double(D.view.src_rows_all) * dout * sizeof(T), s_main_, nk,
         double(D.view.local_nnz() + no) * dout * sizeof(T));
    kbegin(QGNN_K_GEMM_DGRAD);
    if constexpr (sizeof(T) == 4)
      input_grad_masked_f32(ctx_, D.gbar.p, ldo, W, din, dout, 0, no, D.dh_next.p, ldi,
                            mk ? D.h[t].p : nullptr, ldi, s_main_,
                            mk && relu_mask(D, t, ldi).second < 0 ? D.hbits[t].p : nullptr,
                            mk ? hbits_ld(t) : 0);
    else
      QGNN_CALL(qgnn_dense_input_grad(ctx_, dtype_, D.gbar.p, ldo, W, din, dout, nullptr, 0, no,
                                      D.dh_next.p, ldi, s_main_));
    kend(QGNN_K_GEMM_DGRAD, double(no) * (din + dout) * sizeof(T), s_main_, gemm_nk(),
         gemm_flops(double(no), din, dout));
    kbegin(QGNN_K_GEMM_WGRAD);
    T* wg = wgrad_all_.p + D.id * nparams_ + woff_[t];
    QGNN_CALL(qgnn_dense_weight_grad(ctx_, dtype_, D.h[t].p, ldi, D.gbar.p, ldo, din, dout, nullptr,
                                     0, no, 0, wg, s_main_));
    if (nr)
      QGNN_CALL(qgnn_dense_weight_grad(ctx_, dtype_, D.halo.p, ldi, D.gpart.p, ldo, din, dout,
                                       nullptr, 0, nr, 1, wg, s_main_));
    kend(QGNN_K_GEMM_WGRAD, double(no + nr) * (din + dout) * sizeof(T), s_main_,
         (dtype_ == QGNN_F64 ? 1 : 2) * (nr ? 2 : 1), gemm_flops(double(no + nr), din, dout));
  }
  if (side_overlap())
    join_side();
  else
    wait_exchange();
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    scatter_add_all(D, k, din, ldi, mk ? relu_mask(D, t, ldi).first : nullptr,
                    mk ? relu_mask(D, t, ldi).second : ldi);
    std::swap(D.dh, D.dh_next);
  }
  dh_masked_ = mk;
}

// bwd_last (engine.hpp:743-765): layer-1 weight gradient only
template <typename T>
void Engine<T>::backward_last() {
  const int64_t din = dims_[0], dout = dims_[1];
  const int64_t ldi = ld_of(din), ldo = ld_of(dout);
  const bool relu = L_ > 1 && !dh_masked_;  // fp32: usually folded into dh's producers
  for (auto& up : parts_dev_) {
    PartDev& D = *up;
    const int64_t no = D.view.num_owned;
    const T* dz = D.dh.p;
    if (chain_layer(1)) {  // LayerNorm / dropout of layer 1 (chain.cu)
      kbegin(QGNN_K_ELEMWISE);
      chain_backward<T>(D.dh.p, ldo, D.act[0].p, ldo, D.h[1].p, ldo,
                        s_.layer_norm ? D.istd[0].p : nullptr, D.dz.p, ldo, int(dout), 0, no,
                        chain_args(D, 1), s_main_);
      kend(QGNN_K_ELEMWISE, double(no) * dout * sizeof(T) * 4, s_main_);
      dz = D.dz.p;
    } else if (relu) {
      kbegin(QGNN_K_ELEMWISE);
      QGNN_CALL(qgnn_relu_backward(ctx_, dtype_, D.h[1].p, ldo, D.dh.p, ldo, dout, 0, no, D.dz.p,
                                   ldo, s_main_));
      kend(QGNN_K_ELEMWISE, double(no) * dout * sizeof(T) * 3, s_main_);
      dz = D.dz.p;
    }
    kbegin(QGNN_K_GEMM_WGRAD);
    QGNN_CALL(qgnn_dense_weight_grad(ctx_, dtype_, D.hagg[0].p, ldi, dz, ldo, din, dout,
                                     dtype_ == QGNN_F64 ? D.ref_order.p : nullptr, 0, no, 0,
                                     wgrad_all_.p + D.id * nparams_ + woff_[0], s_main_));
    kend(QGNN_K_GEMM_WGRAD, double(no) * (din + dout) * sizeof(T), s_main_,
         dtype_ == QGNN_F64 ? 1 : 2, gemm_flops(double(no), din, dout));
  }
}

// allreduce_and_step (engine.hpp:782-801): fixed-order sum, then Adam
template <typename T>
void Engine<T>::step() {
  kbegin(QGNN_K_ELEMWISE);
  allgather_dev(wgrad_all_.p, (P_ / s_.world) * nparams_, s_main_);
  k_sum_parts<T><<<unsigned(ceil_div(nparams_, 256)), 256, 0, s_main_>>>(wgrad_all_.p, int(P_),
                                                                         nparams_, wsum_.p);
  // bias corrections of step adam_t_ were staged by launch_epoch (adam_bc_)
  adam_step_devbc(dtype_, w_.p, adam_m_.p, adam_v_.p, wsum_.p, nparams_, s_.lr, 0.9, 0.999, 1e-8,
                  adam_bc_.p, s_main_);
  ++ctx_->wgen;  // the next GEMM re-splits the updated weights
  kend(QGNN_K_ELEMWISE, double(nparams_) * sizeof(T) * (P_ + 6), s_main_, 2);
}

// launch_epoch enqueues the whole epoch on the engine's streams and returns;
// finish_epoch waits for it and reads the loss / accuracy back.  Between the
// two the host may stage the next epoch's inputs (set_features).
template <typename T>
void Engine<T>::launch_epoch() {
  QGNN_REQUIRE(!in_flight_, QGNN_EPROTOCOL, "launch_epoch: previous epoch not finished");
  ++epoch_;
  QGNN_CUDA(cudaSetDevice(s_.device));
  launches_ = 0;
  ++ctx_->wgen;  // replayed graphs update the weights without running step() on the host
  prepare_epoch();
  // Adam step t = epoch: bias corrections staged through pinned memory
  ++adam_t_;
  if (!adam_bc_host_) {
    QGNN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&adam_bc_host_), 2 * sizeof(double),
                            cudaHostAllocDefault));
    adam_bc_.alloc(2);
  }
  QGNN_CUDA(cudaStreamSynchronize(s_main_));  // the pinned slot is free (previous epoch done)
  adam_bc_host_[0] = 1.0 - std::pow(0.9, double(adam_t_));
  adam_bc_host_[1] = 1.0 - std::pow(0.999, double(adam_t_));
  QGNN_CUDA(cudaMemcpyAsync(adam_bc_.p, adam_bc_host_, 2 * sizeof(double), cudaMemcpyHostToDevice,
                            s_main_));
  if (s_.dropout > 0.0) {  // dropout streams root.fork({0x4, epoch, l, device}) (engine.hpp:600)
    const int64_t nloc = p1_ - p0_;
    if (!drop_keys_host_) {
      QGNN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&drop_keys_host_),
                              nloc * L_ * sizeof(uint64_t), cudaHostAllocDefault));
      drop_keys_.alloc(nloc * L_);
    }
    for (int64_t p = p0_; p < p1_; ++p)
      for (int64_t l = 0; l < L_; ++l) {
        uint64_t key = root_;
        for (uint64_t c : {uint64_t(0x4), epoch_, uint64_t(l), uint64_t(p)}) key = rng_fork(key, c);
        drop_keys_host_[(p - p0_) * L_ + l] = key;
      }
    QGNN_CUDA(cudaMemcpyAsync(drop_keys_.p, drop_keys_host_, nloc * L_ * sizeof(uint64_t),
                              cudaMemcpyHostToDevice, s_main_));
  }
  // peer-store ranks sharing one GPU (loopback tests): the host-side uploads above
  // synchronize the whole device, so no rank may queue a flag wait of this epoch
  // until every rank is past them (separate GPUs need no such barrier)
  if (p2p_ && loop_) loop_->barrier();
  QGNN_CUDA(cudaEventRecord(ev_a_, s_main_));
  const bool graph = graphs_enabled() && epoch_ > 1;
  EpochGraph& graph_ = graphs_[feat_pending_ ? 1 : 0];
  if (graph && graph_.exec && graph_.plan == plan_version_ && graph_.arena == arena_.p &&
      graph_.scratch == ctx_->scratch && graph_.gemm_b == ctx_->gemm_b) {
    QGNN_CUDA(cudaGraphLaunch(graph_.exec, s_main_));  // replay: restore the host-side records
    ev_used_ = graph_.ev_used;
    launches_ = graph_.launches;
    feat_pending_ = false;
    if (s_.kstats)
      for (int c = 0; c < QGNN_K_COUNT; ++c) kst_[c].gbytes += graph_.gbytes[c];
  } else if (graph) {
    if (graph_.exec) QGNN_CUDA(cudaGraphExecDestroy(graph_.exec));
    graph_ = EpochGraph{};
    double gb0[QGNN_K_COUNT];
    for (int c = 0; c < QGNN_K_COUNT; ++c) gb0[c] = kst_[c].gbytes;
    cudaGraph_t g = nullptr;
    QGNN_CUDA(cudaStreamBeginCapture(s_main_, cudaStreamCaptureModeRelaxed));
    capturing_ = true;
    try {
      epoch_body();
    } catch (...) {
      capturing_ = false;
      cudaStreamEndCapture(s_main_, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    capturing_ = false;
    QGNN_CUDA(cudaStreamEndCapture(s_main_, &g));
    QGNN_CUDA(cudaGraphInstantiate(&graph_.exec, g, 0));
    QGNN_CUDA(cudaGraphDestroy(g));
    graph_.plan = plan_version_;
    graph_.arena = arena_.p;
    graph_.scratch = ctx_->scratch;
    graph_.gemm_b = ctx_->gemm_b;
    graph_.ev_used = ev_used_;
    graph_.launches = launches_;
    for (int c = 0; c < QGNN_K_COUNT; ++c) graph_.gbytes[c] = kst_[c].gbytes - gb0[c];
    QGNN_CUDA(cudaGraphLaunch(graph_.exec, s_main_));
  } else {
    epoch_body();
  }
  QGNN_CUDA(cudaEventRecord(ev_b_, s_main_));
  in_flight_ = true;
}

template <typename T>
void Engine<T>::epoch_body() {
  for (int64_t l = 1; l <= L_; ++l) {
    NvtxRange r("qgnn fwd layer", l);
    if (l == L_ && tf_last_)
      forward_last_tf(int(l));
    else
      forward_layer(int(l));
  }
  {
    NvtxRange r("qgnn loss", 0);
    loss_phase();
  }
  for (int64_t l = L_; l >= 2; --l) {
    NvtxRange r("qgnn bwd layer", l);
    if (l == L_ && tf_last_)
      backward_last_tf(int(l));
    else
      backward_layer(int(l));
  }
  NvtxRange r("qgnn bwd layer 1 + allreduce/Adam", 1);
  backward_last();
  step();
}

// Watchdog: wait for the epoch's end event by polling, checking the
// NCCL communicator's asynchronous error state; after QGNN_WATCHDOG_S (600 s) or on
// an NCCL error the communicator is aborted (releasing the peers' collectives) and
// the epoch fails with ProtocolError / NCCL error instead of hanging the process.
template <typename T>
void Engine<T>::watchdog_wait(cudaEvent_t ev) {
  static const double limit_s = [] {
    const char* e = std::getenv("QGNN_WATCHDOG_S");
    return e ? std::max(0.001, std::atof(e)) : 600.0;
  }();
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0;; ++spin) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) QGNN_CUDA(q);
    if ((spin & 255) != 0) {
      std::this_thread::yield();
      continue;
    }
    if (comm_) {
      ncclResult_t ar = ncclSuccess;
      if (nccl().CommGetAsyncError(comm_, &ar) == ncclSuccess && ar != ncclSuccess &&
          ar != ncclInProgress) {
        nccl().CommAbort(comm_);
        comm_ = nullptr;
        throw Status(QGNN_ENCCL, std::string("watchdog: NCCL error: ") + nccl().GetErrorString(ar));
      }
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > limit_s) {
      if (comm_) {
        nccl().CommAbort(comm_);
        comm_ = nullptr;
      }
      throw Status(QGNN_EPROTOCOL, "watchdog: epoch " + std::to_string(epoch_) +
                                       " did not complete within " + std::to_string(limit_s) + " s");
    }
    // spin like cudaEventSynchronize's default (epoch-end latency enters the e2e
    // wall time); after a second, back off to 100 us naps
    if (el > 1.0)
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    else
      std::this_thread::yield();
  }
}

template <typename T>
void Engine<T>::finish_epoch(qgnn_epoch_metrics* m) {
  QGNN_REQUIRE(in_flight_, QGNN_EPROTOCOL, "finish_epoch: no epoch in flight");
  in_flight_ = false;
  watchdog_wait(ev_b_);
  float ms = 0;
  QGNN_CUDA(cudaEventElapsedTime(&ms, ev_a_, ev_b_));
  // device-detected errors: with world > 1 every rank learns every rank's status
  // before anyone throws (a lone failing rank would leave its peers waiting in the
  // loss all-gather and the next exchange)
  const int st = qgnn_ctx_check(ctx_, s_main_);
  const std::string st_msg = st ? qgnn_last_error() : "";
  if (s_.world > 1) {
    std::vector<uint64_t> all(s_.world, 0);
    all[s_.rank] = uint64_t(st);
    if (!dstat_.p) dstat_.alloc(s_.world);
    QGNN_CUDA(cudaMemcpyAsync(dstat_.p, all.data(), all.size() * sizeof(uint64_t),
                              cudaMemcpyHostToDevice, s_main_));
    allgather_dev(dstat_.p, 1, s_main_);
    QGNN_CUDA(cudaStreamSynchronize(s_main_));
    QGNN_CUDA(cudaMemcpy(all.data(), dstat_.p, all.size() * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost));
    if (st) throw Status(st, st_msg);
    for (int r = 0; r < s_.world; ++r)
      if (all[r])
        throw Status(QGNN_EPROTOCOL, "exchange: peer rank " + std::to_string(r) +
                                         " failed this epoch (status " + std::to_string(all[r]) + ")");
  } else if (st) {
    throw Status(st, st_msg);
  }
  double kms0[QGNN_K_COUNT];
  for (int c = 0; c < QGNN_K_COUNT; ++c) kms0[c] = kst_[c].ms;
  flush_kstats();
  double kms[QGNN_K_COUNT];
  for (int c = 0; c < QGNN_K_COUNT; ++c) kms[c] = kst_[c].ms - kms0[c];
  launches_last_ = launches_;

  // loss / accuracy (engine.hpp:393-397, 803-849)
  std::vector<double> loss(P_, 0.0);
  std::vector<unsigned long long> corr(2 * P_, 0);
  {  // one readback of every hosted partition's loss and hit counts
    const size_t np = parts_dev_.size();
    QGNN_CUDA(cudaMemcpyAsync(epoch_out_host_, epoch_out_.p, 3 * np * sizeof(uint64_t),
                              cudaMemcpyDeviceToHost, s_main_));
    QGNN_CUDA(cudaStreamSynchronize(s_main_));
    for (size_t i = 0; i < np; ++i) {
      const int id = parts_dev_[i]->id;
      std::memcpy(&loss[id], epoch_out_host_ + i, sizeof(double));
      std::memcpy(&corr[2 * id], epoch_out_host_ + np + 2 * i, 2 * sizeof(unsigned long long));
    }
  }
  if (s_.world > 1) {  // every rank fills its partitions' slots, then all-gather
    if (!dloss_.p) {
      dloss_.alloc(P_);
      dcorr_.alloc(2 * P_);
    }
    QGNN_CUDA(cudaMemcpyAsync(dloss_.p, loss.data(), P_ * sizeof(double), cudaMemcpyHostToDevice,
                              s_main_));
    QGNN_CUDA(cudaMemcpyAsync(dcorr_.p, corr.data(), 2 * P_ * sizeof(unsigned long long),
                              cudaMemcpyHostToDevice, s_main_));
    const int64_t ppr = P_ / s_.world;
    allgather_dev(dloss_.p, ppr, s_main_);
    allgather_dev(dcorr_.p, 2 * ppr, s_main_);
    QGNN_CUDA(cudaStreamSynchronize(s_main_));
    QGNN_CUDA(cudaMemcpy(loss.data(), dloss_.p, P_ * sizeof(double), cudaMemcpyDeviceToHost));
    QGNN_CUDA(cudaMemcpy(corr.data(), dcorr_.p, 2 * P_ * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost));
  }
  double total = 0.0;
  unsigned long long vc = 0, tc = 0;
  for (int64_t p = 0; p < P_; ++p) {
    total += loss[p];
    vc += corr[2 * p];
    tc += corr[2 * p + 1];
  }
  if (!std::isfinite(total))
    throw Status(QGNN_EDIVERGED, "epoch " + std::to_string(epoch_) + ": loss diverged");
  qgnn_epoch_metrics em{};
  em.epoch = epoch_;
  em.train_loss = total;
  em.val_acc = global_val_ ? double(vc) / double(global_val_) : 0.0;
  em.test_acc = global_test_ ? double(tc) / double(global_test_) : 0.0;
  for (size_t k = 0; k < keys_.size(); ++k)
    for (int64_t p = 0; p < P_; ++p)
      for (int64_t q = 0; q < P_; ++q)
        if (p != q) {
          em.bytes_total += msgs_[k][p][q].bytes;
          em.ref_bytes_total += msgs_[k][p][q].ref_bytes;
        }
  em.msgs_b2 = msgs_b_[0];
  em.msgs_b4 = msgs_b_[1];
  em.msgs_b8 = msgs_b_[2];
  em.msgs_fp = msgs_b_[3];
  em.ms_total = ms;
  em.ms_quant = kms[QGNN_K_QUANT];
  em.ms_exchange = kms[QGNN_K_EXCHANGE];
  em.ms_dequant = kms[QGNN_K_DEQUANT];
  em.ms_spmm = kms[QGNN_K_SPMM_FWD] + kms[QGNN_K_SPMM_BWD] + kms[QGNN_K_PARTIALS];
  em.ms_gemm = kms[QGNN_K_GEMM_FWD] + kms[QGNN_K_GEMM_DGRAD] + kms[QGNN_K_GEMM_WGRAD];
  em.ms_other = kms[QGNN_K_ELEMWISE];
  resolve_seconds_ = 0;
  if (s_.bit_mode == kAdaptive) adaptive_round(&em);
  em.plan_version = plan_version_;
  em.resolve_seconds = resolve_seconds_;
  *m = em;
}

// Host layout of the trace windows the re-solve reads (every sender partition,
// all ranks): key k's lo values of partition p at win_host_[koff[k] + p *
// stride[k] + i], its hi values half a buffer later.  The message lists are
// fixed after setup, so the pinned buffer is allocated once, at construction.
template <typename T>
size_t Engine<T>::window_layout(std::vector<int64_t>& stride, std::vector<int64_t>& koff) {
  stride.assign(keys_.size(), 0);
  koff.assign(keys_.size() + 1, 0);
  for (size_t k = 0; k < keys_.size(); ++k) {
    int64_t maxn = 0;
    for (int64_t p = 0; p < P_; ++p) {
      int64_t n = 0;
      for (int64_t q = 0; q < P_; ++q)
        if (q != p) n += int64_t(msgs_[k][p][q].ids.size());
      maxn = std::max(maxn, n);
    }
    stride[k] = std::max<int64_t>(1, maxn);
    koff[k + 1] = koff[k] + P_ * stride[k];
  }
  const size_t half = size_t(koff[keys_.size()]);
  if (win_cap_ < 2 * half) {
    if (win_host_) QGNN_CUDA(cudaFreeHost(win_host_));
    QGNN_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&win_host_), 2 * half * sizeof(T),
                            cudaHostAllocDefault));
    if (s_.world > 1) win_dev_.alloc(2 * half, false);
    win_cap_ = 2 * half;
  }
  return half;
}

// gather_stats (engine.hpp:135-165) + reassignment_round (solve.hpp:337-363) + adopt_plan (:851-861)
template <typename T>
void Engine<T>::adaptive_round(qgnn_epoch_metrics*) {
  NvtxRange nv("qgnn adaptive re-solve, epoch", int64_t(epoch_));
  if (s_.period <= 0 || epoch_ % uint64_t(s_.period) != 0) return;
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int64_t> stride, koff;
  const size_t half = window_layout(stride, koff);
  for (size_t k = 0; k < keys_.size(); ++k) {
    const int64_t ppr = P_ / s_.world;
    for (auto& up : parts_dev_) {
      auto& S = up->snd[k];
      if (!S.n) continue;
      const size_t o = size_t(koff[k] + up->id * stride[k]);
      if (s_.world == 1) {  // straight into the pinned host copy
        QGNN_CUDA(cudaMemcpyAsync(win_host_ + o, S.wlo.p, S.n * sizeof(T), cudaMemcpyDeviceToHost,
                                  s_main_));
        QGNN_CUDA(cudaMemcpyAsync(win_host_ + half + o, S.whi.p, S.n * sizeof(T),
                                  cudaMemcpyDeviceToHost, s_main_));
      } else {
        QGNN_CUDA(cudaMemcpyAsync(win_dev_.p + o, S.wlo.p, S.n * sizeof(T),
                                  cudaMemcpyDeviceToDevice, s_main_));
        QGNN_CUDA(cudaMemcpyAsync(win_dev_.p + half + o, S.whi.p, S.n * sizeof(T),
                                  cudaMemcpyDeviceToDevice, s_main_));
      }
    }
    if (s_.world > 1) {
      allgather_dev(win_dev_.p + koff[k], ppr * stride[k], s_main_);
      allgather_dev(win_dev_.p + half + koff[k], ppr * stride[k], s_main_);
    }
  }
  if (s_.world > 1)
    QGNN_CUDA(cudaMemcpyAsync(win_host_, win_dev_.p, 2 * half * sizeof(T), cudaMemcpyDeviceToHost,
                              s_main_));
  QGNN_CUDA(cudaStreamSynchronize(s_main_));
  const auto t_win = std::chrono::steady_clock::now();
  // per key: stats -> group_and_order -> solve_assignment, concurrently (solve.hpp:343-350)
  Cost cm;
  cm.n = P_;
  cm.theta.assign(P_ * P_, s_.theta);
  cm.gamma.assign(P_ * P_, s_.gamma);
  std::vector<std::future<SolveResult>> jobs(keys_.size());
  std::vector<char> has(keys_.size(), 0);
  for (size_t k = 0; k < keys_.size(); ++k) {
    for (int64_t p = 0; p < P_ && !has[k]; ++p)
      for (int64_t q = 0; q < P_; ++q)
        if (p != q && !msgs_[k][p][q].ids.empty()) has[k] = 1;
    if (!has[k]) continue;
    // stats (engine.hpp:135-165) -> group_and_order -> solve_assignment, one thread per key
    jobs[k] = std::async(std::launch::async, [&, k]() {
      const auto a = std::chrono::steady_clock::now();
      std::vector<PairStat> pairs;
      for (int64_t p = 0; p < P_; ++p) {
        int64_t mb = 0;  // first message of pair (p, q) in p's send order
        for (int64_t q = 0; q < P_; ++q) {
          if (p == q) continue;
          const PairMsgs& m = msgs_[k][p][q];
          PairStat ps;
          ps.src = uint32_t(p);
          ps.dst = uint32_t(q);
          ps.msgs.reserve(m.ids.size());
          for (size_t i = 0; i < m.ids.size(); ++i) {
            const size_t w = size_t(koff[k] + p * stride[k] + mb + int64_t(i));
            const double lo = double(win_host_[w]);
            const double hi = double(win_host_[half + w]);
            if (!(hi >= lo)) continue;  // traced (trace.hpp:93)
            MsgStat st;
            st.id = m.ids[i];
            st.dim = uint64_t(keys_[k].dim);
            st.lo = lo;
            st.hi = hi;
            st.asq = keys_[k].bwd ? 1.0 : rx_asq_[p][q][i];
            st.pos = uint32_t(i);
            ps.msgs.push_back(st);
          }
          mb += int64_t(m.ids.size());
          if (!ps.msgs.empty()) pairs.push_back(std::move(ps));
        }
      }
      if (pairs.empty()) return SolveResult{};
      const auto b = std::chrono::steady_clock::now();
      SolveResult r = group_and_order(pairs, s_.group_size);
      const auto c = std::chrono::steady_clock::now();
      solve_exact(r, cm, s_.lambda);
      if (std::getenv("QGNN_RESOLVE_PROFILE")) {
        const auto d = std::chrono::steady_clock::now();
        size_t ng = 0;
        for (const auto& pp : r.pairs) ng += pp.groups.size();
        std::fprintf(stderr,
                     "[resolve] key %zu: stats %.3f s, group %.3f s, solve %.3f s, %zu pairs %zu "
                     "groups\n",
                     k, std::chrono::duration<double>(b - a).count(),
                     std::chrono::duration<double>(c - b).count(),
                     std::chrono::duration<double>(d - c).count(), r.pairs.size(), ng);
      }
      return r;
    });
  }
  // adopt: new bits for every message (all-8 default for untraced / absent pairs),
  // one host thread per key; then the wire layout and the device metadata
  ++plan_version_;
  std::vector<std::future<void>> adopt(keys_.size());
  for (size_t k = 0; k < keys_.size(); ++k)
    adopt[k] = std::async(std::launch::async, [&, k] {
      for (int64_t p = 0; p < P_; ++p)
        for (int64_t q = 0; q < P_; ++q)
          if (p != q)
            std::fill(msgs_[k][p][q].bits.begin(), msgs_[k][p][q].bits.end(), uint8_t(8));
      if (has[k]) {
        SolveResult r = jobs[k].get();
        for (const PlanPairG& pp : r.pairs) {
          PairMsgs& m = msgs_[k][pp.src][pp.dst];
          for (const Group& g : pp.groups)
            for (uint32_t i : g.pos) m.bits[i] = uint8_t(g.bits);  // stats carried positions
        }
      }
      for (int64_t p = 0; p < P_; ++p)
        for (int64_t q = 0; q < P_; ++q)
          if (p != q) layout_pair(int(k), int(p), int(q));
    });
  for (auto& f : adopt) f.get();
  const auto t_adopt = std::chrono::steady_clock::now();
  bits_dirty_ = true;
  arena_layout();
  const auto t_arena = std::chrono::steady_clock::now();
  std::vector<std::future<void>> meta(keys_.size());
  for (size_t k = 0; k < keys_.size(); ++k)
    meta[k] = std::async(std::launch::async, [&, k] {
      QGNN_CUDA(cudaSetDevice(s_.device));
      upload_key_meta(int(k));
    });
  for (auto& f : meta) f.get();
  negotiate_sizes();
  const auto t_meta = std::chrono::steady_clock::now();
  for (size_t k = 0; k < keys_.size(); ++k) {
    for (auto& up : parts_dev_) {  // reset windows (engine.hpp:855-860)
      auto& S = up->snd[k];
      if (S.n)
        k_fill2<T><<<unsigned(ceil_div(S.n, 256)), 256, 0, s_main_>>>(S.wlo.p, T(INFINITY), S.whi.p,
                                                                      T(-INFINITY), S.n);
    }
  }
  QGNN_CUDA(cudaStreamSynchronize(s_main_));
  resolve_seconds_ =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (std::getenv("QGNN_RESOLVE_PROFILE"))
    std::fprintf(stderr,
                 "[resolve] windows %.3f s, solve+adopt %.3f s, arena %.3f s, upload %.3f s, "
                 "total %.3f s (%u host threads)\n",
                 std::chrono::duration<double>(t_win - t0).count(),
                 std::chrono::duration<double>(t_adopt - t_win).count(),
                 std::chrono::duration<double>(t_arena - t_adopt).count(),
                 std::chrono::duration<double>(t_meta - t_arena).count(), resolve_seconds_,
                 std::thread::hardware_concurrency());
}

template <typename T>
void Engine<T>::get_weights(int l, void* out) {
  QGNN_REQUIRE(!in_flight_, QGNN_EPROTOCOL, "get_weights: an epoch is in flight");
  QGNN_REQUIRE(l >= 0 && l < L_, QGNN_EINVAL, "get_weights: bad layer");
  QGNN_CUDA(cudaMemcpy(out, w_.p + woff_[l], dims_[l] * dims_[l + 1] * sizeof(T),
                       cudaMemcpyDeviceToHost));
}

template <typename T>
void Engine<T>::set_weights(int l, const void* in) {
  QGNN_REQUIRE(!in_flight_, QGNN_EPROTOCOL, "set_weights: an epoch is in flight");
  QGNN_REQUIRE(l >= 0 && l < L_, QGNN_EINVAL, "set_weights: bad layer");
  QGNN_CUDA(cudaMemcpy(w_.p + woff_[l], in, dims_[l] * dims_[l + 1] * sizeof(T),
                       cudaMemcpyHostToDevice));
  ++ctx_->wgen;
}

template <typename T>
void Engine<T>::info(int64_t* out) {
  int64_t msgs = 0, max_owned = 0, max_halo = 0;
  for (int64_t p = 0; p < P_; ++p)
    for (int64_t q = 0; q < P_; ++q)
      if (p != q) msgs += int64_t(parts_[p].remote_out[q].size());
  for (auto& up : parts_dev_) {
    max_owned = std::max(max_owned, up->view.num_owned);
    max_halo = std::max(max_halo, up->view.num_remote);
  }
  out[0] = msgs;
  out[1] = P_;
  out[2] = p1_ - p0_;
  out[3] = max_owned;
  out[4] = max_halo;
  out[5] = launches_last_;
}

template <typename T>
int Engine<T>::kernel_stats(double* out, int n) {
  // 3 doubles per class (ms, launches, algorithmic bytes); with room for 4 per
  // class the SpMM gathered-row bytes follow as the 4th
  const int w = n >= 4 * QGNN_K_COUNT ? 4 : 3;
  const int m = std::min<int>(n / w, QGNN_K_COUNT);
  for (int c = 0; c < m; ++c) {
    out[w * c] = kst_[c].ms;
    out[w * c + 1] = kst_[c].launches;
    out[w * c + 2] = kst_[c].bytes;
    if (w == 4) out[w * c + 3] = kst_[c].gbytes;
    kst_[c] = KStat{};
  }
  return m;
}

}  // namespace qgnn_b200

using namespace qgnn_b200;

struct qgnn_engine {
  std::unique_ptr<EngineBase> impl;
};

extern "C" {

int qgnn_engine_create(const qgnn_settings* s, int64_t n_nodes, const int64_t* adj_ptr,
                       const int32_t* adj, const void* features, const int32_t* labels,
                       const uint8_t* train, const uint8_t* val, const uint8_t* test,
                       const uint32_t* owner, const void* nccl_unique_id, qgnn_engine** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(s && out && adj_ptr && adj && features, QGNN_EINVAL, "engine: null argument");
  int count = 0;
  QGNN_REQUIRE(cudaGetDeviceCount(&count) == cudaSuccess && count > 0, QGNN_ECUDA,
               "no CUDA device: the B200 path has no CPU fallback");
  auto* e = new qgnn_engine;
  try {
    if (s->dtype == QGNN_F64)
      e->impl = std::make_unique<Engine<double>>(*s, n_nodes, adj_ptr, adj, features, labels, train,
                                                 val, test, owner, nccl_unique_id);
    else
      e->impl = std::make_unique<Engine<float>>(*s, n_nodes, adj_ptr, adj, features, labels, train,
                                                val, test, owner, nccl_unique_id);
  } catch (...) {
    delete e;
    throw;
  }
  *out = e;
  QGNN_API_END
}

int qgnn_engine_destroy(qgnn_engine* e) {
  QGNN_API_BEGIN
  delete e;
  QGNN_API_END
}

int qgnn_engine_run_epoch(qgnn_engine* e, qgnn_epoch_metrics* m) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(e && m, QGNN_EINVAL, "null engine");
  e->impl->run_epoch(m);
  QGNN_API_END
}

int qgnn_engine_set_kstats(qgnn_engine* e, int on) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(e, QGNN_EINVAL, "null engine");
  e->impl->set_kstats(on != 0);
  QGNN_API_END
}

int qgnn_engine_launch_epoch(qgnn_engine* e) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(e, QGNN_EINVAL, "null engine");
  e->impl->launch_epoch();
  QGNN_API_END
}

int qgnn_engine_finish_epoch(qgnn_engine* e, qgnn_epoch_metrics* m) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(e && m, QGNN_EINVAL, "null engine");
  e->impl->finish_epoch(m);
  QGNN_API_END
}

int qgnn_engine_set_features(qgnn_engine* e, const void* f) {
  QGNN_API_BEGIN
  e->impl->set_features(f);
  QGNN_API_END
}

int qgnn_engine_get_weights(qgnn_engine* e, int layer, void* out) {
  QGNN_API_BEGIN
  e->impl->get_weights(layer, out);
  QGNN_API_END
}

int qgnn_engine_set_weights(qgnn_engine* e, int layer, const void* in) {
  QGNN_API_BEGIN
  e->impl->set_weights(layer, in);
  QGNN_API_END
}

int qgnn_engine_info(qgnn_engine* e, int64_t* out5) {
  QGNN_API_BEGIN
  e->impl->info(out5);
  QGNN_API_END
}

int qgnn_engine_kernel_stats(qgnn_engine* e, double* out, int n) {
  try {
    return e->impl->kernel_stats(out, n);
  } catch (...) {
    return -status_from_exception();
  }
}

int qgnn_loopback_id(uint64_t group, void* out128) {
  QGNN_API_BEGIN
  std::memset(out128, 0, 128);
  std::memcpy(out128, kLoopMagic, 8);
  std::memcpy(static_cast<char*>(out128) + 8, &group, 8);
  QGNN_API_END
}

int qgnn_nccl_unique_id(void* out128) {
  QGNN_API_BEGIN
  ncclUniqueId id;
  QGNN_NCCL(nccl().GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  QGNN_API_END
}

// ---- production SpMM plan (aggregate.hpp:94-165 at scale) ----------------------
struct qgnn_spmm_plan {
  qgnn_ctx* ctx = nullptr;
  int64_t row_begin = 0, n_rows = 0, max_dim = 0;
  qgnn_b200::Hubs hubs;
};

int qgnn_spmm_plan_create(qgnn_ctx* ctx, const int64_t* ptr_a, const int64_t* ptr_b,
                          int64_t row_begin, int64_t n_rows, int64_t max_dim, int64_t hub_deg,
                          qgnn_spmm_plan** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(ctx && out && ptr_a, QGNN_EINVAL, "spmm_plan_create: null argument");
  QGNN_REQUIRE(row_begin >= 0 && n_rows >= 0 && max_dim > 0 && hub_deg >= 1, QGNN_EINVAL,
               "spmm_plan_create: bad sizes");
  auto* p = new qgnn_spmm_plan;
  p->ctx = ctx;
  p->row_begin = row_begin;
  p->n_rows = n_rows;
  p->max_dim = round_up(max_dim, 8);
  try {
    build_hub_plan(p->hubs, ptr_a, ptr_b, row_begin, row_begin + n_rows, p->max_dim, hub_deg);
  } catch (...) {
    delete p;
    throw;
  }
  *out = p;
  QGNN_API_END
}

int qgnn_spmm_plan_destroy(qgnn_spmm_plan* p) {
  delete p;
  return QGNN_OK;
}

int qgnn_spmm_plan_run(qgnn_spmm_plan* p, int64_t dim, const float* x, int64_t ld_x,
                       const float* y, int64_t ld_y, const float* self_alpha,
                       const int64_t* ptr_a, const int32_t* col_a, const float* alpha_a,
                       const int64_t* ptr_b, const int32_t* col_b, const float* alpha_b,
                       const float* mask, int64_t ld_mask, float* out, int64_t ld_out,
                       void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(p, QGNN_EINVAL, "spmm_plan_run: null plan");
  QGNN_REQUIRE(dim > 0 && dim <= p->max_dim, QGNN_EINVAL, "spmm_plan_run: dim exceeds the plan");
  const int64_t d4 = round_up(dim, 4);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  QGNN_REQUIRE(ld_x % 4 == 0 && ld_out % 4 == 0 && d4 <= ld_x && d4 <= ld_out && al16(x) &&
                   al16(out) && (!ptr_b || (ld_y % 4 == 0 && d4 <= ld_y && al16(y))) &&
                   (!mask || (ld_mask % 4 == 0 && d4 <= ld_mask && al16(mask))),
               QGNN_EINVAL,
               "spmm_plan_run: fp32 rows must be 16-byte aligned with ld a multiple of 4 "
               "columns covering round_up(dim, 4) (zero padded)");
  if (p->n_rows == 0) return QGNN_OK;
  spmm_f32(p->ctx, int(d4), x, ld_x, y, ld_y, self_alpha, ptr_a, col_a, alpha_a, ptr_b, col_b,
           alpha_b, p->row_begin, p->n_rows, out, ld_out, &p->hubs.plan,
           static_cast<cudaStream_t>(stream), mask, ld_mask);
  QGNN_API_END
}

// ---- standalone exchange (exchange.hpp:45-78; engine.hpp:502, :528-529) ----------
struct qgnn_comm {
  int world = 1, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  std::shared_ptr<qgnn_b200::LoopGroup> loop;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
};

int qgnn_comm_create(const void* id128, int world, int rank, int device, qgnn_comm** out) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(out && world >= 1 && rank >= 0 && rank < world, QGNN_EINVAL,
               "comm_create: bad rank / world");
  QGNN_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<qgnn_comm>();
  c->world = world;
  c->rank = rank;
  c->device = device;
  QGNN_CUDA(cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming));
  QGNN_CUDA(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
  if (id128 && std::memcmp(id128, kLoopMagic, 8) == 0) {
    uint64_t key;
    std::memcpy(&key, static_cast<const char*>(id128) + 8, 8);
    key ^= 0x636f6d6d00000000ull;  // separate namespace from engine loopback groups
    std::lock_guard<std::mutex> lk(g_loop_mu);
    auto& g = g_loops[key];
    if (!g) {
      g = std::make_shared<LoopGroup>();
      g->world = world;
      g->engines.assign(world, nullptr);
      g->ptr.assign(world, nullptr);
      g->ev.assign(world, nullptr);
      g->ev2.assign(world, nullptr);
      g->sends.assign(world, {});
      g->recvs.assign(world, {});
    }
    QGNN_REQUIRE(g->world == world && !g->engines[rank], QGNN_EPROTOCOL,
                 "comm_create: loopback world mismatch or rank already registered");
    g->engines[rank] = c.get();
    c->loop = g;
  } else {
    if (id128) {
      ncclUniqueId id;
      std::memcpy(&id, id128, sizeof(id));
      QGNN_NCCL(nccl().CommInitRank(&c->nccl, world, id, rank));
    } else {
      QGNN_REQUIRE(world == 1, QGNN_EINVAL, "comm_create: world > 1 needs an id");
      QGNN_NCCL(nccl().CommInitAll(&c->nccl, 1, &device));
    }
  }
  *out = c.release();
  QGNN_API_END
}

int qgnn_comm_destroy(qgnn_comm* c) {
  if (!c) return QGNN_OK;
  if (c->nccl) nccl().CommDestroy(c->nccl);
  if (c->loop) {
    std::lock_guard<std::mutex> lk(g_loop_mu);
    c->loop->engines[c->rank] = nullptr;
    bool empty = true;
    for (void* e : c->loop->engines) empty &= e == nullptr;
    if (empty)
      for (auto it = g_loops.begin(); it != g_loops.end(); ++it)
        if (it->second == c->loop) {
          g_loops.erase(it);
          break;
        }
  }
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  delete c;
  return QGNN_OK;
}

int qgnn_exchange(qgnn_comm* c, const void* send, const uint64_t* send_off,
                  const uint64_t* send_bytes, void* recv, const uint64_t* recv_off,
                  const uint64_t* recv_bytes, void* stream) {
  QGNN_API_BEGIN
  QGNN_REQUIRE(c && send_off && send_bytes && recv_off && recv_bytes, QGNN_EINVAL,
               "exchange: null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const auto* sb = static_cast<const uint8_t*>(send);
  auto* rb = static_cast<uint8_t*>(recv);
  const int W = c->world, me = c->rank;
  if (c->nccl) {
    // one NCCL group: every pair's send and receive posted together, so the
    // transfers to all peers proceed concurrently over NVLink / NVSwitch
    QGNN_NCCL(nccl().GroupStart());
    for (int r = 0; r < W; ++r)
      if (send_bytes[r])
        QGNN_NCCL(nccl().Send(sb + send_off[r], size_t(send_bytes[r]), ncclUint8, r, c->nccl, st));
    for (int r = 0; r < W; ++r)
      if (recv_bytes[r])
        QGNN_NCCL(nccl().Recv(rb + recv_off[r], size_t(recv_bytes[r]), ncclUint8, r, c->nccl, st));
    QGNN_NCCL(nccl().GroupEnd());
    return QGNN_OK;
  }
  // in-process loopback: receivers pull from the senders' buffers (device copies)
  LoopGroup& G = *c->loop;
  std::vector<std::array<int64_t, 4>> mine(W);
  for (int r = 0; r < W; ++r)
    mine[r] = {int64_t(send_off[r]), int64_t(send_bytes[r]), int64_t(recv_off[r]),
               int64_t(recv_bytes[r])};
  QGNN_CUDA(cudaEventRecord(c->ev_ready, st));
  G.ptr[me] = const_cast<uint8_t*>(sb);
  G.ev[me] = c->ev_ready;
  G.sends[me] = mine;
  G.barrier();
  // ProtocolError (engine.hpp:546-550): negotiated sizes must agree pairwise
  bool match = true;
  for (int a = 0; a < W; ++a)
    for (int b = 0; b < W; ++b) match &= G.sends[a][b][1] == G.sends[b][a][3];
  if (match)
    for (int r = 0; r < W; ++r) {
      const int64_t nb = G.sends[r][me][1];
      if (!nb) continue;
      if (r != me) QGNN_CUDA(cudaStreamWaitEvent(st, G.ev[r], 0));
      QGNN_CUDA(cudaMemcpyAsync(rb + recv_off[r], static_cast<uint8_t*>(G.ptr[r]) + G.sends[r][me][0],
                                size_t(nb), cudaMemcpyDeviceToDevice, st));
    }
  QGNN_CUDA(cudaEventRecord(c->ev_done, st));
  G.ev2[me] = c->ev_done;
  G.barrier();  // every rank's pulls enqueued
  // our send buffer may be reused once every receiver has copied out of it
  for (int r = 0; r < W; ++r)
    if (r != me && G.sends[me][r][1]) QGNN_CUDA(cudaStreamWaitEvent(st, G.ev2[r], 0));
  G.barrier();  // nobody reads G.* of this call after here
  QGNN_REQUIRE(match, QGNN_EPROTOCOL,
               "exchange: send/receive sizes disagree between ranks (negotiate_buffers)");
  QGNN_API_END
}

}  // extern "C"
