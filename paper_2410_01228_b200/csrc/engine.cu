// cs_engine: the C-ABI (include/conserve_b200.h) over the block pool, the
// layer forward and the checkpoint/restore data movement.
//
// Streams: compute (forward), d2h (checkpoint gather), h2d (restore). The
// whole forward is enqueued at once (or replayed as a CUDA graph); a
// layer-wise preemption is applied on the device: the safepoint kernel
// between layers truncates the iteration descriptor to the online prefix and
// every later kernel -- the K8 GEMMs included -- reads the truncated counts,
// so no host thread paces the launches.
#include <cublasLt.h>
#include <cublas_v2.h>
#include <cuda.h>
#include <nccl.h>
#include <time.h>

#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <chrono>
#include <cmath>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <fstream>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/conserve_b200.h"
#include "block_pool.h"
#include "common.cuh"

namespace csk {
void init_matrix(__nv_bfloat16* w, int64_t rows, int64_t cols, int64_t global_cols, int64_t col_off,
                 const RowMap& map, uint64_t seed, uint64_t tensor, float scale, float offset, cudaStream_t s);
void embed(__nv_bfloat16* x, const __nv_bfloat16* emb, const int32_t* tok_ids, int hidden, const IterDesc* desc,
           int grid, cudaStream_t s);
void add_rmsnorm(__nv_bfloat16* x, const __nv_bfloat16* add, const __nv_bfloat16* w, __nv_bfloat16* xn, int hidden,
                 float eps, const IterDesc* desc, const int32_t* row_idx, int grid, cudaStream_t s,
                 const SafepointArg& sp = SafepointArg{}, unsigned long long* zero_keys = nullptr);
void silu_mul(const __nv_bfloat16* gu, __nv_bfloat16* act, int ffn, const IterDesc* desc, int grid_rows,
              cudaStream_t s, bool interleave);
void rope_append(__nv_bfloat16* qkv, const int32_t* tok_pos, const int32_t* tok_slot, __nv_bfloat16* pool, int hq,
                 int hkv, int D, int num_layers, int layer, float theta, const IterDesc* desc, int grid,
                 cudaStream_t s);
void argmax_rows(const float* logits, int vocab, unsigned long long* keys, const IterDesc* desc, int grid,
                 cudaStream_t s, bool zero = true);
void safepoint_vote(__nv_bfloat16* tail, const IterDesc* desc, const PreemptMailbox* mb, cudaStream_t s);
void read_globaltimer(uint64_t* mapped_out, cudaStream_t s);
void calib_clock(volatile uint64_t* mb, cudaStream_t s);
void kv_move(bool to_host, __nv_bfloat16* pool, __nv_bfloat16* host_mapped, const void* segs_mapped, int n_segs,
             int runs_per_seg, int D, int sms, cudaStream_t s);
void kv_pack(bool to_stage, __nv_bfloat16* pool, __nv_bfloat16* stage, const void* segs, const int64_t* stage_off,
             int n_segs, int runs_per_seg, int D, int sms, cudaStream_t s);
void fill_pool(__nv_bfloat16* pool, size_t n, uint64_t seed, cudaStream_t s);
int decode_sk_ctas_per_sm(int head_dim, int group, int ns);
bool launch_attention(const AttnParams& p, const CUtensorMap* kv_map, int head_dim, int group, int n_dec_grid,
                      int n_pt_grid, cudaStream_t s);
int prefill_tile_rows();
int prefill_tc2_tile_rows();
int prefill_tile_keys();
int wgemm_stages(int Mp, size_t budget);
int wgemm_max_clusters(int Mp, int stages, int splits);
bool wgemm_supported(int M, int N, int K);
void wgemm_sk(const CUtensorMap* wmap, const CUtensorMap* xmap, void* y, float* ws, int32_t* cnt, int M, int Mp,
              int N, int K, bool f32_out, int ctas, cudaStream_t s);
void wgemm_tc(const CUtensorMap* wmap, const CUtensorMap* xmap, void* y, int M, int Mp, int N, int K, int splits,
              int stages, bool f32_out, cudaStream_t s);
void p2p_allreduce(const P2PArgs& a, __nv_bfloat16* out, int64_t count, int blocks, cudaStream_t s);
void p2p_allreduce2(const P2PArgs& a, __nv_bfloat16* out, int64_t count, int blocks, cudaStream_t s);
bool gemm_pf_supported(int N, int K);
void gemm_pf(const CUtensorMap* xmap, const CUtensorMap* wmap, void* y, int M, const int32_t* m_dev, int N, int K,
             bool f32_out, int sms, cudaStream_t s, bool swiglu = false, const PfExtra* ex = nullptr);
void rope_table(float2* tab, const int32_t* tok_pos, int D, float theta, const IterDesc* desc, int grid,
                cudaStream_t s);
void sm_copy(void* dst, const void* src, size_t bytes, cudaStream_t s);
void out_copy(void* h_out, const IterDesc* desc, const void* keys, int E, cudaStream_t s);
}  // namespace csk

namespace {

thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CK(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__)); \
  } while (0)
#define CKB(x)                                                                                  \
  do {                                                                                          \
    cublasStatus_t s_ = (x);                                                                    \
    if (s_ != CUBLAS_STATUS_SUCCESS)                                                            \
      throw CudaError(std::string(#x) + ": cublas status " + std::to_string(static_cast<int>(s_))); \
  } while (0)
#define CKN(x)                                                                                  \
  do {                                                                                          \
    ncclResult_t r_ = (x);                                                                      \
    if (r_ != ncclSuccess) throw CudaError(std::string(#x) + ": " + ncclGetErrorString(r_));    \
  } while (0)

template <typename F>
int guard(F&& f) {
  try {
    f();
    return CS_OK;
  } catch (const csb::PoolError& e) {
    g_err = e.what();
    return CS_ERR_POOL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return CS_ERR_CUDA;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return CS_ERR_CONFIG;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return CS_ERR_INVALID;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return CS_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return CS_ERR_RUNTIME;
  }
}

uint64_t host_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<uint64_t>(ts.tv_nsec);
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared ownership of a job's event pair: the descriptor ring and the job
// record may release it in either order.
struct EventPair {
  cudaEvent_t start = nullptr, end = nullptr;
  EventPair() {
    CK(cudaEventCreate(&start));
    CK(cudaEventCreate(&end));
  }
  ~EventPair() {
    cudaEventDestroy(start);
    cudaEventDestroy(end);
  }
};

// Pinned, device-mapped FIFO ring for per-job segment descriptors; the move
// kernel reads them over the host link directly (no extra H2D copy).
struct DescRing {
  uint8_t* host = nullptr;
  uint8_t* dev = nullptr;
  size_t cap = 0, head = 0;
  struct Live {
    size_t off, len;
    std::shared_ptr<EventPair> ev;
  };
  std::deque<Live> live;
  size_t alloc(size_t n, const std::shared_ptr<EventPair>& ev) {
    if (n > cap) throw std::runtime_error("descriptor ring too small for one job");
    if (head + n > cap) head = 0;
    auto overlaps = [&](const Live& l) { return head < l.off + l.len && l.off < head + n; };
    while (!live.empty() && std::any_of(live.begin(), live.end(), overlaps)) {
      CK(cudaEventSynchronize(live.front().ev->end));
      live.pop_front();
    }
    const size_t off = head;
    live.push_back({off, n, ev});
    head += align_up(n, 256);
    return off;
  }
};

}  // namespace

struct cs_engine;

namespace {

struct DeviceMover : csb::Mover {
  cs_engine* e;
  struct Rec {
    int64_t ord;
    std::shared_ptr<EventPair> ev;
  };
  std::deque<Rec> live[2];          // launched, not yet seen complete (issue order)
  int64_t issued[2] = {0, 0}, done[2] = {0, 0};
  std::map<int64_t, float> ms_of[2];  // device ms of recently completed jobs (cs_job_poll)
  explicit DeviceMover(cs_engine* eng) : e(eng) {}
  int64_t launch(int dir, const std::vector<csb::Segment>& segs, int64_t after_other);
  int64_t gather_to_host(const std::vector<csb::Segment>& segs, int64_t after_h2d) override {
    return launch(CS_D2H, segs, after_h2d);
  }
  int64_t scatter_from_host(const std::vector<csb::Segment>& segs, int64_t after_d2h) override {
    return launch(CS_H2D, segs, after_d2h);
  }
  int64_t done_prefix(int32_t dir) override {
    poll(dir);
    return done[dir];
  }
  void poll(int dir);
  // end event of job `ord` of `dir`, or null once it completed
  cudaEvent_t pending_event(int dir, int64_t ord) {
    for (const Rec& r : live[dir])
      if (r.ord == ord) return r.ev->end;
    return nullptr;
  }
};

}  // namespace

struct Weights {
  __nv_bfloat16 *emb = nullptr, *final_norm = nullptr, *lm_head = nullptr;
  std::vector<__nv_bfloat16*> attn_norm, mlp_norm, wqkv, wo, wgu, wd;
};

struct cs_engine {
  cs_config cfg{};
  bool host_only = false, no_model = false;
  bool dry = false;  // replay fast-forward: bookkeeping only, no kernels
  int L = 0, hidden = 0, hq = 0, hkv = 0, D = 0, ffn = 0, vocab = 0, G = 0, tp = 1, rank = 0;
  int64_t block_elems = 0;  // per rank, all layers
  int64_t max_tok = 0, max_ent = 0;
  int sms = 148;

  std::unique_ptr<csb::BlockPool> pool;
  std::unique_ptr<DeviceMover> mover;

  // device memory
  __nv_bfloat16* kv = nullptr;
  alignas(64) CUtensorMap kv_map{};  // TMA view of the pool as [rows][D] bf16, 64x16 boxes, 128-B swizzle
  __nv_bfloat16* host_kv = nullptr;      // pinned
  __nv_bfloat16* host_kv_dev = nullptr;  // mapped alias
  size_t host_kv_bytes = 0;
  int host_numa_node = -1;               // node the pool is bound to, -1 = cudaHostAlloc
  void* weight_mem = nullptr;
  Weights w;
  __nv_bfloat16 *x = nullptr, *xn = nullptr, *qkv = nullptr, *attn = nullptr, *tmp = nullptr, *gu = nullptr,
                *act = nullptr, *xl = nullptr;
  float* logits = nullptr;
  float* ws = nullptr;
  size_t ws_floats = 0;
  float* ws2 = nullptr;  // K2 split-K partials
  int32_t* dec_cnt = nullptr;  // K1 split-K arrival counters
  float* ws_sk = nullptr;      // K1 stream-K partials
  int sk_ctas = 0;             // K1 stream-K grid (0: split-K kernel)
  int sk_resident = 0;         // K1 stream-K CTAs resident at once
  int sk_pairs_max = 0;        // K1 kernel choice: stream-K below this many pairs
  int sk_stages = 2;           // K1 stream-K per-warp ring depth (CS_K1_STAGES=3 for A/B)
  // host time per forward (CS_HOST_TIMERS=1 prints the totals at cs_destroy)
  double host_prep_ms = 0, host_enq_ms = 0, host_wait_ms = 0, host_post_ms = 0;
  int64_t host_launches = 0;
  bool k2_pair = false;        // K2 on CTA pairs (head_dim 128; opt-in CS_K2_PAIR=1)
  size_t ws2_floats = 0;
  uint8_t* d_meta = nullptr;
  uint8_t* h_meta = nullptr;
  uint8_t* h_meta_dev = nullptr;  // mapped alias (the SM metadata copy reads it)
  size_t meta_cap = 0;
  uint8_t* d_out = nullptr;  // IterDesc + out ids
  uint8_t* h_out = nullptr;
  uint8_t* h_out_dev = nullptr;   // mapped alias (the output copy kernel writes it)
  csk::PreemptMailbox* mailbox = nullptr;  // mapped pinned
  csk::PreemptMailbox* mailbox_dev = nullptr;
  int64_t clock_offset_ns = 0;  // gpu globaltimer - host CLOCK_MONOTONIC

  cudaStream_t s_compute = nullptr, s_d2h = nullptr, s_h2d = nullptr;
  cudaEvent_t ev_start = nullptr, ev_end = nullptr, ev_fwd_done = nullptr;
  bool any_forward = false;
  cublasHandle_t blas = nullptr;
  void* blas_ws = nullptr;
  // cuBLASLt plans autotuned per decode-graph bucket (few-row GEMMs are
  // latency/bandwidth bound and the default heuristic is not always the
  // fastest there); key = M | N << 12 | K << 32 | f32 << 63
  struct LtPlan {
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
    cublasLtMatmulAlgo_t algo{};
  };
  cublasLtHandle_t lt = nullptr;
  std::map<uint64_t, LtPlan> lt_plans;
  std::map<int, bool> lt_tuned;
  void tune_gemms(int M);
  bool lt_gemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32);
  // K7 (csrc/gemm_tc.cu): the M <= 256 projections on our own tcgen05
  // weight-streaming kernel; TMA maps per (tensor, rows, K, box rows)
  // 0 never (CS_WGEMM=0), 1 always for M <= 256 (CS_WGEMM=1), 2 (default) where tune_gemms
  // timed it faster than the best cuBLAS plan
  int wgemm_mode = 2;
  std::map<uint64_t, bool> k7_pick;
  std::map<std::pair<int, int>, int> k7_clusters;  // (Mp, K split) -> co-resident clusters (per engine: no shared state)
  std::map<std::tuple<const void*, int, int, int>, CUtensorMap> tmaps;
  const CUtensorMap* tmap(const void* p, int rows, int K, int box_rows);
  bool wgemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32);
  bool wgemm_launch(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32);
  bool k7_sk = false;           // K7 in stream-K mode (CS_K7_SK=1; default: the cluster split-K kernel)
  float* k7_ws = nullptr;       // stream-K partials
  int32_t* k7_cnt = nullptr;    // stream-K per-tile arrival counters
  ncclComm_t comm = nullptr;
  DescRing ring[2];
  // K4/K5 DMA path: per-direction device staging (token-major, like a host
  // slot) between the pack/unpack kernel and the copy-engine transfer
  __nv_bfloat16* stage[2] = {nullptr, nullptr};
  size_t stage_elems = 0;
  bool kv_zerocopy = false;  // CS_KV_ZEROCOPY=1: SM zero-copy kernel instead (A/B)
  bool kv_small_zc = true;  // short-run chunks as one zero-copy kernel (CS_KV_SMALL_ZC=0: off)
  double moved_ms[2] = {0, 0};
  std::atomic<int64_t> launches{0};  // hand-written kernel launches (not cuBLAS/NCCL)

  // iteration state
  struct Iter {
    bool active = false;
    uint64_t epoch = 0;
    int n_tok = 0, n_tok_on = 0, n_ent = 0, n_ent_on = 0, n_dec = 0, n_pt = 0;
    bool has_offline = false;
    int splits = 1, pps = 1;
    bool k1_sk = false;  // K1 runs the stream-K kernel this iteration
    int k2_splits = 1, k2_tps = 1 << 30;
    bool graph = false;  // decode-only plan replayed from a captured CUDA graph
    int bucket = 0;      // graph bucket: token rows / entries / decode rows (padded)
    std::vector<cs_batch_entry> entries;
    std::vector<std::array<int64_t, 3>> writes;  // (id, w0, w1) per entry (w0<0: none)
    csk::AttnParams ap{};
    const int32_t* d_tok_ids = nullptr;
    const int32_t* d_tok_slot = nullptr;
    const int32_t* d_ent_last = nullptr;
    bool device_m = false;  // every layer GEMM is K8 (reads the device row count)
    int64_t wait_h2d = 0;  // last restore writing a block this plan reads
    uint64_t signal_ns = 0;
    int64_t meta_bytes = 0;
    double k1_bytes = 0, k2_flops = 0;  // algorithmic work per layer
    int32_t retro_layer = -1;  // host-decided drop after the device finished (cs_iter_retro_drop)
  } it;

  void enqueue_layers();
  int enqueue_body(int Tg, int Eg, bool graph);
  // CUDA graphs of decode-only forwards, keyed by (bucket, safepoints, gen);
  // gen bumps whenever a buffer baked into the graphs is reallocated
  struct GraphExec {
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
  };
  std::map<uint64_t, GraphExec> graphs;
  uint64_t graph_gen = 0;
  bool graphs_enabled = true;
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
    ++graph_gen;
  }
  int gemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32,
           const int32_t* m_dev = nullptr, const csk::PfExtra* ex = nullptr);
  float2* rope_tab = nullptr;  // [max_tok][D/2] (cos, sin) of the iteration (K8 qkv epilogue)
  bool kt_layer = true;        // kernel timing on for the layer being enqueued
  bool fuse_epilogues = true;  // K8 RoPE / residual epilogues (CS_NO_FUSE=1: separate kernels, for A/B)
  // Per-kernel-class device timing (cs_set_kernel_timing; bench roofline):
  // event pairs on the launching stream around every non-graph launch of
  // K8 / K2 / K1, folded into the totals at cs_iter_wait (iterations the
  // safepoint cut are skipped: their algorithmic work is not the host's).
  struct KTime {
    int64_t launches = 0;
    double ms = 0, units = 0;
  };
  bool ktime_on = false;
  KTime ktime[CS_KT_N];
  std::vector<cudaEvent_t> kt_ev;
  // (class, algorithmic units, weight) per event pair; weight = the layer
  // stride of the timed launch, so class totals estimate every layer
  struct KtPending {
    int cls;
    double units;
    int weight;
  };
  std::vector<KtPending> kt_pending;
  int kt_weight = 1;  // weight of the launches being enqueued
  template <typename Fn>
  void timed(int cls, double units, Fn&& fn) {
    if (!ktime_on || it.graph || !kt_layer) {
      fn();
      return;
    }
    const size_t k = kt_pending.size();
    while (kt_ev.size() < 2 * k + 2) {
      cudaEvent_t ev;
      CK(cudaEventCreate(&ev));
      kt_ev.push_back(ev);
    }
    CK(cudaEventRecord(kt_ev[2 * k], s_compute));
    fn();
    CK(cudaEventRecord(kt_ev[2 * k + 1], s_compute));
    kt_pending.push_back({cls, units, kt_weight});
  }
  // K8 (csrc/gemm_pf.cu) for this layer GEMM? Prefill-sized M, or any
  // non-graph M > 256 when a safepoint may truncate the batch on the device
  bool use_pf(int M, int N, int K) const;
  int pf_min_rows = 2048;
  bool pf_enabled = true;
  // W_gate|up stored interleaved in 128-row blocks ([g 0..127 | u 0..127 |
  // g 128..255 | ...]) so a 256-column K8 tile holds matching gate and up
  // features and its epilogue writes silu(g) * u directly (ffn % 128 == 0)
  bool gu_interleave = false;
  void allreduce(__nv_bfloat16* buf, int64_t count);
  // ---- peer-memory all-reduce: exchange region =
  // [2 partial buffers of (max_tok*hidden + 64) bf16][flag u64][step u64][arrive i32]
  uint8_t* xchg = nullptr;
  size_t xchg_part_elems = 0;
  bool p2p = false;
  int p2p_blocks = 0;
  int p2p_mode = 0;                    // 0 auto, 1 one-shot, 2 two-shot (CS_P2P_ALLREDUCE)
  int part_slot = 0;                   // next partial buffer (same sequence on every rank)
  std::vector<uint8_t*> peer_xchg;     // exchange region of every rank, rank order
  std::vector<cudaIpcMemHandle_t> opened;  // (for cs_destroy) handles we opened
  std::vector<void*> opened_ptrs;
  __nv_bfloat16* xpart(uint8_t* base, int slot) const {
    return reinterpret_cast<__nv_bfloat16*>(base) + static_cast<size_t>(slot) * xchg_part_elems;
  }
  uint64_t* xflag(uint8_t* base) const {
    return reinterpret_cast<uint64_t*>(base + 2 * xchg_part_elems * sizeof(__nv_bfloat16));
  }
  // destination of a partial-sum GEMM: this rank's next exchange buffer when
  // the peer path is attached, else the all-reduce buffer itself (NCCL, g=1)
  __nv_bfloat16* partial_out(__nv_bfloat16* buf) { return p2p ? xpart(xchg, part_slot) : buf; }
  void reduce_into(__nv_bfloat16* buf, int64_t count);
};

namespace {

int64_t DeviceMover::launch(int dir, const std::vector<csb::Segment>& segs_in, int64_t after_other) {
  if (e->dry || segs_in.empty()) return 0;
  // Segments in host-address order (slot, then token): pages of one request
  // usually hold adjacent host slots (in either order after LIFO reuse), so
  // sorted they merge into a few long copy-engine runs instead of one
  // cudaMemcpyAsync per 2 MiB page on the host's critical path.
  std::vector<csb::Segment> segs(segs_in);
  std::sort(segs.begin(), segs.end(), [](const csb::Segment& a, const csb::Segment& b) {
    return a.slot != b.slot ? a.slot < b.slot : a.t0 < b.t0;
  });
  auto ev = std::make_shared<EventPair>();
  cudaStream_t st = dir == CS_D2H ? e->s_d2h : e->s_h2d;
  // a gather reads KV the last forward wrote; either direction may have to
  // follow a job of the other one that touches the same block / host slot
  if (dir == CS_D2H && e->any_forward) CK(cudaStreamWaitEvent(st, e->ev_fwd_done, 0));
  if (after_other > 0) {
    if (cudaEvent_t w = pending_event(1 - dir, after_other)) CK(cudaStreamWaitEvent(st, w, 0));
  }
  const int runs = e->L * 2 * e->hkv;
  const size_t tok_elems = static_cast<size_t>(runs) * e->D;  // one token of one page, all layers
  DescRing& ring = e->ring[dir];
  CK(cudaEventRecord(ev->start, st));
  if (e->kv_zerocopy) {
    const size_t n = segs.size() * sizeof(csb::Segment);
    const size_t off = ring.alloc(n, ev);
    std::memcpy(ring.host + off, segs.data(), n);
    csk::kv_move(dir == CS_D2H, e->kv, e->host_kv_dev, ring.dev + off, static_cast<int>(segs.size()), runs, e->D,
                 e->sms, st);
    e->launches += 1;
  } else {
    // chunks whose staging fits the buffer: pack (D2H) -> copy-engine DMA of
    // the merged host runs -> (H2D) unpack; in stream order on this stream
    const size_t seg_bytes = sizeof(csb::Segment) + sizeof(int64_t);
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    size_t i0 = 0;
    while (i0 < segs.size()) {
      size_t i1 = i0, used = 0;
      while (i1 < segs.size()) {
        const size_t need = static_cast<size_t>(segs[i1].t1 - segs[i1].t0) * tok_elems;
        if (i1 > i0 && used + need > e->stage_elems) break;
        used += need;
        ++i1;
      }
      const size_t n = i1 - i0;
      const size_t off = ring.alloc(n * seg_bytes, ev);
      std::memcpy(ring.host + off, segs.data() + i0, n * sizeof(csb::Segment));
      int64_t* so = reinterpret_cast<int64_t*>(ring.host + off + n * sizeof(csb::Segment));
      dsts.clear();
      srcs.clear();
      sizes.clear();
      size_t pos = 0;
      for (size_t k = i0; k < i1; ++k) {
        const csb::Segment& g = segs[k];
        so[k - i0] = static_cast<int64_t>(pos);
        const size_t len = static_cast<size_t>(g.t1 - g.t0) * tok_elems * 2;
        uint8_t* hp = reinterpret_cast<uint8_t*>(e->host_kv) +
                      (static_cast<size_t>(g.slot) * 16 + static_cast<size_t>(g.t0)) * tok_elems * 2;
        uint8_t* sp = reinterpret_cast<uint8_t*>(e->stage[dir] + pos);
        void* d = dir == CS_D2H ? static_cast<void*>(hp) : static_cast<void*>(sp);
        void* src = dir == CS_D2H ? static_cast<void*>(sp) : static_cast<void*>(hp);
        // merge with the previous run when both sides continue it
        if (!sizes.empty() && static_cast<uint8_t*>(dsts.back()) + sizes.back() == d &&
            static_cast<uint8_t*>(srcs.back()) + sizes.back() == src) {
          sizes.back() += len;
        } else {
          dsts.push_back(d);
          srcs.push_back(src);
          sizes.push_back(len);
        }
        pos += static_cast<size_t>(g.t1 - g.t0) * tok_elems;
      }
      const void* dseg = ring.dev + off;
      const int64_t* dso = reinterpret_cast<const int64_t*>(ring.dev + off + n * sizeof(csb::Segment));
      // many short host runs (decode deltas: one 128 KB token per request)
      // cost a DMA setup each; such a chunk moves as one zero-copy kernel
      // straight between the blocks and the mapped host slots instead
      if (e->kv_small_zc && sizes.size() >= 8 && pos * 2 / sizes.size() < (1u << 20)) {
        csk::kv_move(dir == CS_D2H, e->kv, e->host_kv_dev, dseg, static_cast<int>(n), runs, e->D, e->sms, st);
        e->launches += 1;
        i0 = i1;
        continue;
      }
      if (dir == CS_D2H) {
        csk::kv_pack(true, e->kv, e->stage[dir], dseg, dso, static_cast<int>(n), runs, e->D, e->sms, st);
        e->launches += 1;
      }
      // one copy-engine DMA per merged host run (host slots are token-major,
      // so adjacent slots of one job usually merge into a few long runs)
      for (size_t k = 0; k < sizes.size(); ++k) CK(cudaMemcpyAsync(dsts[k], srcs[k], sizes[k], cudaMemcpyDefault, st));
      if (dir == CS_H2D) {
        csk::kv_pack(false, e->kv, e->stage[dir], dseg, dso, static_cast<int>(n), runs, e->D, e->sms, st);
        e->launches += 1;
      }
      i0 = i1;
    }
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(ev->end, st));
  live[dir].push_back({++issued[dir], std::move(ev)});
  return issued[dir];
}

void DeviceMover::poll(int dir) {
  while (!live[dir].empty()) {
    const Rec& r = live[dir].front();
    const cudaError_t q = cudaEventQuery(r.ev->end);
    if (q == cudaErrorNotReady) break;
    CK(q);
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, r.ev->start, r.ev->end));
    e->moved_ms[dir] += ms;
    ms_of[dir][r.ord] = ms;
    if (ms_of[dir].size() > 4096) ms_of[dir].erase(ms_of[dir].begin());
    done[dir] = r.ord;
    live[dir].pop_front();
  }
}

constexpr uint64_t kTensorEmb = 1, kTensorLm = 2, kTensorFinalNorm = 3;
uint64_t tensor_id(int layer, int which) { return 1000ull + static_cast<uint64_t>(layer) * 16 + which; }
enum { kWAttnNorm = 0, kWQkv = 1, kWO = 2, kWMlpNorm = 3, kWGu = 4, kWD = 5 };

void validate(const cs_config& c) {
  if (c.page_tokens != 16) throw ConfigError("page_tokens is fixed at 16");
  if (c.num_layers < 1) throw ConfigError("num_layers must be >= 1");
  if (c.safepoint_interval_layers < 1) throw ConfigError("safepoint_interval_layers must be >= 1");
  if (c.tp_size < 1 || c.tp_rank < 0 || c.tp_rank >= c.tp_size) throw ConfigError("bad tp_rank/tp_size");
  if (c.n_kv_heads % c.tp_size || c.n_heads % c.tp_size || c.ffn % c.tp_size)
    throw ConfigError("heads and ffn must divide by tp_size (KV-head-group sharding)");
  if (c.n_heads % c.n_kv_heads) throw ConfigError("n_heads must be a multiple of n_kv_heads");
  if (c.head_dim != 64 && c.head_dim != 128) throw ConfigError("head_dim must be 64 or 128");
  if (c.hidden % 8 || (c.ffn / c.tp_size) % 8) throw ConfigError("hidden and ffn shard must be multiples of 8");
  const int64_t model_bpt = 2LL * c.num_layers * c.n_kv_heads * c.head_dim * 2;
  // Bookkeeping-only engines hold no KV bytes: the reference's accounting
  // unit may then be any value (its presets use 196608 B/token for every
  // model, coserve_cli.cpp:56,75,92).
  if (c.kv_bytes_per_token < 1) throw ConfigError("kv_bytes_per_token must be positive");
  if (c.kv_bytes_per_token != model_bpt && !(c.flags & CS_FLAG_HOST_ONLY))
    throw ConfigError("kv_bytes_per_token must equal 2*L*H_kv*d*2 = " + std::to_string(model_bpt));
  if (c.gpu_kv_capacity < 1 || c.host_kv_capacity < 1) throw ConfigError("KV capacities must be positive");
  if (c.d2h_bandwidth <= 0 || c.h2d_bandwidth <= 0) throw ConfigError("transfer bandwidths must be positive");
  if (c.max_batched_tokens < 1) throw ConfigError("max_batched_tokens must be >= 1");
}

// Pinned host KV pool on the GPU's own NUMA node (config 5: 8 ranks each
// checkpointing over their own host link). The node comes from sysfs for
// the device's PCI bus id; with more than one node the region is mmap'ed,
// bound to that node (mbind, MPOL_BIND) before any page is touched, then
// pinned and mapped for the device (cudaHostRegister). One node, an unknown
// node or CS_HOST_NUMA=0: plain cudaHostAlloc. *node = the bound node or -1.
int gpu_numa_node(int device) {
  char bus[64] = {0};
  if (cudaDeviceGetPCIBusId(bus, sizeof(bus), device) != cudaSuccess) return -1;
  std::string id(bus);
  for (char& c : id) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  if (id.size() > 12) id = id.substr(id.size() - 12);  // dddd:bb:dd.f
  std::ifstream f("/sys/bus/pci/devices/" + id + "/numa_node");
  int node = -1;
  if (!(f >> node)) return -1;
  return node;
}

int numa_node_count() {
  int n = 0;
  for (int i = 0; i < 1024; ++i) {
    std::ifstream f("/sys/devices/system/node/node" + std::to_string(i) + "/cpulist");
    if (!f) break;
    ++n;
  }
  return n;
}

void* alloc_host_pool(int device, size_t bytes, int* node) {
  *node = -1;
  const char* env = std::getenv("CS_HOST_NUMA");
  const int want = env && env[0] == '0' ? -1 : gpu_numa_node(device);
  if (want >= 0 && want < 64 && numa_node_count() > 1) {
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p != MAP_FAILED) {
      unsigned long mask = 1ul << want;
      constexpr int kMpolBind = 2;
      if (syscall(SYS_mbind, p, bytes, kMpolBind, &mask, 64, 0) == 0 &&
          cudaHostRegister(p, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable) == cudaSuccess) {
        *node = want;
        return p;
      }
      cudaGetLastError();  // clear a failed registration; fall back below
      munmap(p, bytes);
    }
  }
  void* p = nullptr;
  CK(cudaHostAlloc(&p, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  return p;
}

void free_host_pool(void* p, size_t bytes, int node) {
  if (!p) return;
  if (node >= 0) {
    cudaHostUnregister(p);
    munmap(p, bytes);
  } else {
    cudaFreeHost(p);
  }
}

// TMA descriptor for the KV pool viewed as [rows][D] bf16 (a page of one
// (block, layer, K|V, head) = 16 consecutive rows): 64-column x 16-row boxes,
// SWIZZLE_128B to match the UMMA operand layout (attn_tc.cu). The driver entry
// point is resolved through the runtime, so no -lcuda.
// 2D bf16 tensor map over [rows][cols] (row-major), SWIZZLE_128B, box
// 64 columns x box_rows rows; false when the driver rejects the shape.
bool make_2d_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);

void make_kv_tensor_map(CUtensorMap* map, void* pool, uint64_t rows, int D) {
  if (rows >= (1ull << 31)) throw ConfigError("KV pool too large for 32-bit TMA row coordinates");
  if (!make_2d_map(map, pool, rows, static_cast<uint64_t>(D), 16)) throw CudaError("cuTensorMapEncodeTiled failed");
}

bool make_2d_map(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  // resolved once (thread-safe static initialisation: engines may build maps concurrently)
  static const EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(fn);
  }();
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

// ------------------------------------------------------------------ GEMM ----
// Row-major Y[M,N] = X[M,K] * W[N,K]^T on cuBLAS (plain library GEMM).
static uint64_t lt_key(int M, int N, int K, bool f32) {
  return static_cast<uint64_t>(M) | (static_cast<uint64_t>(N) << 12) | (static_cast<uint64_t>(K) << 32) |
         (static_cast<uint64_t>(f32) << 63);
}

bool cs_engine::lt_gemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K,
                        bool out_f32) {
  auto f = lt_plans.find(lt_key(M, N, K, out_f32));
  if (f == lt_plans.end()) return false;
  const float alpha = 1.f, beta = 0.f;
  const LtPlan& pl = f->second;
  CKB(cublasLtMatmul(lt, pl.op, &alpha, W, pl.a, A, pl.b, &beta, C, pl.c, C, pl.c, &pl.algo, blas_ws, 64u << 20,
                     s_compute));
  return true;
}

// Times every heuristic candidate (up to 16) of the step's GEMM shapes at M
// rows -- and K7, our tcgen05 weight-streaming kernel -- on the live weights
// and activation buffers (outputs land in buffers the coming forward
// overwrites) and keeps the fastest; once per bucket, before its graph is
// captured. Each candidate runs over up to 8 layers' weights in turn, so the
// weights stream from HBM as in a decode step (one layer's set would sit in
// the 126 MB L2 and favour a different kernel).
void cs_engine::tune_gemms(int M) {
  if (lt_tuned[M]) return;
  lt_tuned[M] = true;
  if (!lt) CKB(cublasLtCreate(&lt));
  struct Shape {
    const __nv_bfloat16* A;
    std::vector<const __nv_bfloat16*> W;
    void* C;
    int N, K;
    bool f32;
  };
  const int qkv_cols = (hq + 2 * hkv) * D;
  std::vector<Shape> shapes(5);
  shapes[0] = {xn, {}, qkv, qkv_cols, hidden, false};
  shapes[1] = {attn, {}, tmp, hidden, hq * D, false};
  shapes[2] = {xn, {}, gu, 2 * ffn, hidden, false};
  shapes[3] = {act, {}, tmp, hidden, ffn, false};
  shapes[4] = {xl, {w.lm_head}, logits, vocab, hidden, true};
  for (int l = 0; l < std::min(L, 8); ++l) {  // 8 layers' weights exceed the L2 several times over
    shapes[0].W.push_back(w.wqkv[l]);
    shapes[1].W.push_back(w.wo[l]);
    shapes[2].W.push_back(w.wgu[l]);
    shapes[3].W.push_back(w.wd[l]);
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const float alpha = 1.f, beta = 0.f;
  const size_t wsz = 64u << 20;
  // ms per launch of `run` over every weight of the shape (after one warm pass)
  auto time_over = [&](const Shape& sh, const std::function<bool(const __nv_bfloat16*)>& run) {
    for (const __nv_bfloat16* W : sh.W)
      if (!run(W)) return 1e30f;
    CK(cudaEventRecord(e0, s_compute));
    for (const __nv_bfloat16* W : sh.W) run(W);
    CK(cudaEventRecord(e1, s_compute));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    return ms / static_cast<float>(sh.W.size());
  };
  for (const Shape& sh : shapes) {
    if (sh.f32 && M > max_ent) continue;
    LtPlan pl;
    CKB(cublasLtMatmulDescCreate(&pl.op, CUBLAS_COMPUTE_32F, CUDA_R_32F));
    const cublasOperation_t ta = CUBLAS_OP_T, tb = CUBLAS_OP_N;
    CKB(cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSA, &ta, sizeof(ta)));
    CKB(cublasLtMatmulDescSetAttribute(pl.op, CUBLASLT_MATMUL_DESC_TRANSB, &tb, sizeof(tb)));
    // column-major view: C[N, M] = W^T[N, K] * X^T[K, M]
    CKB(cublasLtMatrixLayoutCreate(&pl.a, CUDA_R_16BF, sh.K, sh.N, sh.K));
    CKB(cublasLtMatrixLayoutCreate(&pl.b, CUDA_R_16BF, sh.K, M, sh.K));
    CKB(cublasLtMatrixLayoutCreate(&pl.c, sh.f32 ? CUDA_R_32F : CUDA_R_16BF, sh.N, M, sh.N));
    cublasLtMatmulPreference_t pref;
    CKB(cublasLtMatmulPreferenceCreate(&pref));
    CKB(cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &wsz, sizeof(wsz)));
    cublasLtMatmulHeuristicResult_t res[16];
    int n = 0;
    const cublasStatus_t hs = cublasLtMatmulAlgoGetHeuristic(lt, pl.op, pl.a, pl.b, pl.c, pl.c, pref, 16, res, &n);
    cublasLtMatmulPreferenceDestroy(pref);
    float best = 1e30f;
    int bi = -1;
    // the lm_head runs replicated on every rank of a sharded engine: its
    // algorithm must not depend on per-rank timing noise, or the ranks'
    // logits (and sampled ids) could differ in the last bits
    const bool replicated = sh.f32 && tp > 1;
    for (int i = 0; hs == CUBLAS_STATUS_SUCCESS && i < n; ++i) {
      if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
      if (replicated) {
        bi = i;
        break;
      }
      const float ms = time_over(sh, [&](const __nv_bfloat16* W) {
        return cublasLtMatmul(lt, pl.op, &alpha, W, pl.a, sh.A, pl.b, &beta, sh.C, pl.c, sh.C, pl.c, &res[i].algo,
                              blas_ws, wsz, s_compute) == CUBLAS_STATUS_SUCCESS;
      });
      if (ms < best) {
        best = ms;
        bi = i;
      }
    }
    if (bi >= 0) {
      pl.algo = res[bi].algo;
      lt_plans[lt_key(M, sh.N, sh.K, sh.f32)] = pl;
    } else {
      cublasLtMatmulDescDestroy(pl.op);
      cublasLtMatrixLayoutDestroy(pl.a);
      cublasLtMatrixLayoutDestroy(pl.b);
      cublasLtMatrixLayoutDestroy(pl.c);
    }
    // K7 against the best cuBLAS plan (CS_WGEMM=2)
    if (wgemm_mode == 2 && !(sh.f32 && tp > 1) && csk::wgemm_supported(M, sh.N, sh.K)) {
      const float ms7 = time_over(sh, [&](const __nv_bfloat16* W) {
        return wgemm_launch(sh.A, W, sh.C, M, sh.N, sh.K, sh.f32);
      });
      k7_pick[lt_key(M, sh.N, sh.K, sh.f32)] = ms7 < best;
      static const bool verbose = std::getenv("CS_WGEMM_VERBOSE") != nullptr;
      if (verbose)
        std::fprintf(stderr, "tune M=%d N=%d K=%d: cuBLAS %.4f ms, K7 %.4f ms -> %s\n", M, sh.N, sh.K, best, ms7,
                     ms7 < best ? "K7" : "cuBLAS");
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  CK(cudaGetLastError());
}

const CUtensorMap* cs_engine::tmap(const void* p, int rows, int K, int box_rows) {
  const auto key = std::make_tuple(p, rows, K, box_rows);
  auto f = tmaps.find(key);
  if (f != tmaps.end()) return &f->second;
  CUtensorMap m;
  if (!make_2d_map(&m, p, static_cast<uint64_t>(rows), static_cast<uint64_t>(K), static_cast<uint32_t>(box_rows)))
    return nullptr;
  return &tmaps.emplace(key, m).first->second;
}

bool cs_engine::wgemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32) {
  if (wgemm_mode == 0) return false;
  if (wgemm_mode == 2) {  // tuned: only where it beat cuBLAS at this bucket
    auto f = k7_pick.find(lt_key(M, N, K, out_f32));
    if (f == k7_pick.end() || !f->second) return false;
  }
  return wgemm_launch(A, W, C, M, N, K, out_f32);
}

bool cs_engine::wgemm_launch(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K,
                             bool out_f32) {
  if (!csk::wgemm_supported(M, N, K)) return false;
  const int Mp = (M + 15) / 16 * 16;
  // X rows past M are out of the tensor: TMA fills them with zeros
  const CUtensorMap* wm = tmap(W, N, K, 128);
  const CUtensorMap* xm = tmap(A, M, K, Mp);
  if (!wm || !xm) return false;
  if (k7_sk) {  // stream-K mode: one persistent CTA per SM, equal weight ranges
    if (!k7_ws || N / 128 > 8192) return false;
    csk::wgemm_sk(wm, xm, C, k7_ws, k7_cnt, M, Mp, N, K, out_f32, sms, s_compute);
    return true;
  }
  // ONE wave of CTAs: >= one feature tile per SM -> two CTAs per SM, no
  // split; fewer tiles -> one deep-ring CTA per SM and the largest K split
  // (a cluster of <= 8, any size, uneven last split) with n_tiles x split <=
  // SMs whose clusters are all co-resident. A second wave would double the
  // prologue + epilogue the weight stream cannot hide (qkv at split 4: 192
  // CTAs on 148 SMs ran at 2 TB/s, profiles/r1/k7_gemm.md).
  const int n_tiles = N / 128;
  const bool two = n_tiles >= sms;
  const int stages = csk::wgemm_stages(Mp, two ? 112 * 1024 : 220 * 1024);
  int splits = 1;
  if (!two) {
    for (int sp = 8; sp >= 2; --sp) {
      if (n_tiles * sp > sms || K / 64 / sp < 4) continue;
      auto key = std::make_pair(Mp, sp);
      auto f = k7_clusters.find(key);
      if (f == k7_clusters.end()) f = k7_clusters.emplace(key, csk::wgemm_max_clusters(Mp, stages, sp)).first;
      if (f->second >= n_tiles) {
        splits = sp;
        break;
      }
    }
  }
  csk::wgemm_tc(wm, xm, C, M, Mp, N, K, splits, stages, out_f32, s_compute);
  return true;
}

bool cs_engine::use_pf(int M, int N, int K) const {
  if (!pf_enabled || !csk::gemm_pf_supported(N, K)) return false;
  if (M >= pf_min_rows) return true;
  // the device-side row count is what makes a layer-wise drop shrink the
  // GEMMs of the remaining layers: worth K8's small-M cost when one may come
  return M > 256 && cfg.instrumented != 0 && it.has_offline && !it.graph;
}

// Returns the number of hand-written kernels it launched (K7/K8: 1, cuBLAS: 0).
// m_dev: device row count (IterDesc.n_tok_cur) honoured by K8.
int cs_engine::gemm(const __nv_bfloat16* A, const __nv_bfloat16* W, void* C, int M, int N, int K, bool out_f32,
                    const int32_t* m_dev, const csk::PfExtra* ex) {
  if (M <= 0) return 0;
  // an epilogue fusion is only requested where K8 runs (use_pf checked by the caller)
  if (ex && !use_pf(M, N, K)) throw std::logic_error("K8 epilogue fusion requested off the K8 path");
  if (use_pf(M, N, K)) {
    const int rows = A == xl ? static_cast<int>(max_ent) : static_cast<int>(max_tok);
    const CUtensorMap* xm = tmap(A, rows, K, 128);
    const CUtensorMap* wm = tmap(W, N, K, 128);
    if (xm && wm) {
      timed(CS_KT_K8, 2.0 * M * N * K,
            [&] { csk::gemm_pf(xm, wm, C, M, m_dev, N, K, out_f32, sms, s_compute, false, ex); });
      return 1;
    }
  }
  if (ex) throw CudaError("K8 tensor maps unavailable for a fused epilogue");
  if (wgemm(A, W, C, M, N, K, out_f32)) return 1;
  timed(CS_KT_LIB, 2.0 * M * N * K, [&] {
    if (lt_gemm(A, W, C, M, N, K, out_f32)) return;
    const float alpha = 1.f, beta = 0.f;
    CKB(cublasGemmEx(blas, CUBLAS_OP_T, CUBLAS_OP_N, N, M, K, &alpha, W, CUDA_R_16BF, K, A, CUDA_R_16BF, K, &beta, C,
                     out_f32 ? CUDA_R_32F : CUDA_R_16BF, N, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT));
  });
  return 0;
}

void cs_engine::allreduce(__nv_bfloat16* buf, int64_t count) {
  if (tp <= 1 || count <= 0) return;
  if (!comm) throw std::logic_error("tp_size > 1 needs cs_nccl_init or cs_tp_attach_* before a forward");
  CKN(ncclAllReduce(buf, buf, static_cast<size_t>(count), ncclBfloat16, ncclSum, comm, s_compute));
}

// Sums the partial written by the preceding partial_out() GEMM over all ranks
// into buf (peer path) or reduces buf in place (NCCL).
void cs_engine::reduce_into(__nv_bfloat16* buf, int64_t count) {
  if (tp <= 1 || count <= 0) return;
  if (!p2p) {
    allreduce(buf, count);
    return;
  }
  csk::P2PArgs a{};
  for (int r = 0; r < tp; ++r) {
    a.part[r] = xpart(peer_xchg[static_cast<size_t>(r)], part_slot);
    a.flag[r] = xflag(peer_xchg[static_cast<size_t>(r)]);
    a.step[r] = xflag(peer_xchg[static_cast<size_t>(r)]) + 1;
    a.flag2[r] = xflag(peer_xchg[static_cast<size_t>(r)]) + 3;
  }
  a.arrive = reinterpret_cast<int*>(xflag(xchg) + 2);
  a.arrive2 = reinterpret_cast<int*>(xflag(xchg) + 4);
  a.rank = rank;
  a.g = tp;
  // two-shot (reduce-scatter + all-gather, 2(g-1)/g x payload over NVLink
  // per rank) for large payloads at g >= 4; one-shot ((g-1) x payload, one
  // barrier) otherwise. CS_P2P_ALLREDUCE=oneshot|twoshot forces either.
  const bool two = p2p_mode == 2 || (p2p_mode == 0 && tp >= 4 && count * 2 >= (512 << 10));
  if (two) {
    csk::p2p_allreduce2(a, buf, count, p2p_blocks, s_compute);
  } else {
    csk::p2p_allreduce(a, buf, count, p2p_blocks, s_compute);
  }
  part_slot ^= 1;
}

// Enqueues the layer stack and the head for Tg token rows / Eg entries (the
// plan's counts, or the graph bucket's); returns the kernels it launched.
int cs_engine::enqueue_body(int Tg, int Eg, bool graph) {
  int n_launch = 0;
  const auto* desc = reinterpret_cast<const csk::IterDesc*>(d_meta);
  // K8 GEMMs read the live row count: a safepoint drop shrinks them too
  const int32_t* m_dev = &desc->n_tok_cur;
  const bool instrumented = cfg.instrumented != 0 && it.has_offline;
  const int qkv_cols = (hq + 2 * hkv) * D;
  const int T = Tg;
  __nv_bfloat16* tail = tmp + static_cast<size_t>(max_tok) * hidden;  // vote slot
  auto is_sp = [&](int l) { return instrumented && l > 0 && l < L && l % cfg.safepoint_interval_layers == 0; };

  // K8 epilogue fusions (single rank, K8 path): RoPE + KV append in the qkv
  // projection, the residual add in o_proj / down
  const bool fuse_ok = !graph && tp == 1 && fuse_epilogues;
  const bool fuse_rope = fuse_ok && D == 128 && rope_tab && use_pf(static_cast<int>(Tg), qkv_cols, hidden);
  const bool fuse_o = fuse_ok && use_pf(static_cast<int>(Tg), hidden, hq * D);
  const bool fuse_down = fuse_ok && use_pf(static_cast<int>(Tg), hidden, ffn);
  // decode-only graphs: RoPE of q and the new token's K/V append inside K1
  const bool k1_rope = graph && fuse_epilogues && rope_tab;
  if (fuse_rope || k1_rope) {
    csk::rope_table(rope_tab, it.ap.tok_pos, D, cfg.rope_theta, desc, T, s_compute);
    ++n_launch;
  }
  // kernel-class timing (bench) on every kt_stride-th layer only: every
  // layer has the same shapes, and ~16 timed layers keep a deep model's
  // event records + launches inside the device launch queue (a full queue
  // blocks cs_forward_launch until the GPU drains it, which would delay the
  // caller's preemption signal by tens of layers)
  const int kt_stride = std::max(1, (L + 15) / 16);
  for (int l = 0; l < L; ++l) {
    const int64_t M = Tg;
    kt_layer = l % kt_stride == 0;
    kt_weight = std::min(kt_stride, L - l);  // this layer stands for itself and the untimed ones after it
    if (l == 0) {
      csk::embed(x, w.emb, it.d_tok_ids, hidden, desc, T, s_compute);
    }
    // K6 rides in the layer's first kernel: progress for the host monitor at
    // every layer of an instrumented plan, the drop check at safepoints
    csk::SafepointArg sp{};
    if (instrumented) {
      sp.mb = mailbox_dev;
      sp.layer = l;
      sp.mode = is_sp(l) ? (tp == 1 ? 1 : 2) : 0;
      sp.tail = tail;
    }
    csk::add_rmsnorm(x, (l == 0 || fuse_down) ? nullptr : tmp, w.attn_norm[l], xn, hidden, cfg.rms_eps, desc,
                     nullptr, T, s_compute, sp);
    if (fuse_rope) {
      csk::PfExtra ex;
      ex.rope_tab = rope_tab;
      ex.tok_slot = it.d_tok_slot;
      ex.pool = kv;
      ex.hq = hq;
      ex.hkv = hkv;
      ex.D = D;
      ex.num_layers = L;
      ex.layer = l;
      n_launch += gemm(xn, w.wqkv[l], qkv, static_cast<int>(M), qkv_cols, hidden, false, m_dev, &ex);
    } else {
      n_launch += gemm(xn, w.wqkv[l], qkv, static_cast<int>(M), qkv_cols, hidden, false, m_dev);
      if (!k1_rope)
        csk::rope_append(qkv, it.ap.tok_pos, it.d_tok_slot, kv, hq, hkv, D, L, l,
                         cfg.rope_theta, desc, T, s_compute);
    }
    csk::AttnParams ap = it.ap;
    ap.layer = l;
    ap.k1_rope = k1_rope ? 1 : 0;
    ap.rope_theta = cfg.rope_theta;
    ap.tok_slot = it.d_tok_slot;
    ap.rope_tab = rope_tab;
    bool ok = true;
    const int n_dec_grid = graph ? Tg : it.n_dec;
    if (n_dec_grid > 0)
      timed(CS_KT_K1, it.k1_bytes, [&] { ok &= csk::launch_attention(ap, &kv_map, D, G, n_dec_grid, 0, s_compute); });
    if (it.n_pt > 0)
      timed(CS_KT_K2, it.k2_flops, [&] { ok &= csk::launch_attention(ap, &kv_map, D, G, 0, it.n_pt, s_compute); });
    if (!ok) throw ConfigError("unsupported attention shape");
    if (fuse_o) {  // x += attn . Wo^T in K8's epilogue
      csk::PfExtra ex;
      ex.resid = x;
      n_launch += gemm(attn, w.wo[l], tmp, static_cast<int>(M), hidden, hq * D, false, m_dev, &ex);
    } else {
      __nv_bfloat16* part = partial_out(tmp);
      n_launch += gemm(attn, w.wo[l], part, static_cast<int>(M), hidden, hq * D, false, m_dev);
      if (part != tmp) ++n_launch;
      reduce_into(tmp, M * hidden);
    }
    csk::add_rmsnorm(x, fuse_o ? nullptr : tmp, w.mlp_norm[l], xn, hidden, cfg.rms_eps, desc, nullptr, T, s_compute);
    const CUtensorMap* gxm = nullptr;
    const CUtensorMap* gwm = nullptr;
    if (gu_interleave && use_pf(static_cast<int>(M), 2 * ffn, hidden)) {
      gxm = tmap(xn, static_cast<int>(max_tok), hidden, 128);
      gwm = tmap(w.wgu[l], 2 * ffn, hidden, 128);
    }
    if (gxm && gwm) {  // K8 with the SwiGLU epilogue: gate|up never round-trips through HBM
      timed(CS_KT_K8, 2.0 * M * 2 * ffn * hidden, [&] {
        csk::gemm_pf(gxm, gwm, act, static_cast<int>(M), m_dev, 2 * ffn, hidden, false, sms, s_compute, true);
      });
      n_launch += 1;
    } else {
      n_launch += gemm(xn, w.wgu[l], gu, static_cast<int>(M), 2 * ffn, hidden, false, m_dev);
      csk::silu_mul(gu, act, ffn, desc, T, s_compute, gu_interleave);
      n_launch += 1;
    }
    if (fuse_down) {  // x += act . Wd^T in K8's epilogue
      csk::PfExtra ex;
      ex.resid = x;
      n_launch += gemm(act, w.wd[l], tmp, static_cast<int>(M), hidden, ffn, false, m_dev, &ex);
    } else {
      __nv_bfloat16* part = partial_out(tmp);
      n_launch += gemm(act, w.wd[l], part, static_cast<int>(M), hidden, ffn, false, m_dev);
      if (tp > 1) {
        if (part != tmp) ++n_launch;
        if (is_sp(l + 1)) {
          // the safepoint vote rides in 8 extra elements of this all-reduce
          csk::safepoint_vote(part + M * hidden, desc, mailbox_dev, s_compute);
          reduce_into(tmp, M * hidden + 8);
          CK(cudaMemcpyAsync(tail, tmp + M * hidden, 16, cudaMemcpyDeviceToDevice, s_compute));
        } else {
          reduce_into(tmp, M * hidden);
        }
      }
    }
    n_launch += (l == 0 ? 1 : 0) + 3 - (fuse_rope || k1_rope ? 1 : 0) + (tp > 1 && is_sp(l + 1) ? 1 : 0) +
                (it.n_dec > 0 ? 1 : 0) + (it.n_pt > 0 ? (it.k2_splits > 1 ? 2 : 1) : 0);
    if ((cfg.flags & CS_FLAG_SYNC_DEBUG) && !graph) {
      CK(cudaStreamSynchronize(s_compute));
      CK(cudaGetLastError());
    }
  }
  // Final norm of each entry's last row -> lm_head -> argmax.
  kt_layer = true;
  kt_weight = 1;
  const int E = Eg;
  auto* keys = reinterpret_cast<unsigned long long*>(d_out + sizeof(csk::IterDesc));
  csk::add_rmsnorm(x, fuse_down ? nullptr : tmp, w.final_norm, xl, hidden, cfg.rms_eps, desc, it.d_ent_last, E,
                   s_compute, csk::SafepointArg{}, keys);
  n_launch += gemm(xl, w.lm_head, logits, E, vocab, hidden, true);
  csk::argmax_rows(logits, vocab, keys, desc, E, s_compute, /*zero=*/false);
  // descriptor + sampled-token keys straight into the mapped host outputs
  // (no copy-engine D2H queued behind checkpoint DMAs)
  csk::out_copy(h_out_dev, reinterpret_cast<const csk::IterDesc*>(d_meta), d_out + sizeof(csk::IterDesc), E,
                s_compute);
  n_launch += 3;
  return n_launch;
}

// Enqueues every layer of the current iteration.
// Decode-only plans run a CUDA graph captured once per bucket: all per-plan
// data (counts, split sizes, block tables) is read from the device metadata,
// so one graph serves every plan of its bucket and the ~350 launches of a
// decode step cost one cudaGraphLaunch.
void cs_engine::enqueue_layers() {
  if (it.graph) {
    const bool sp = cfg.instrumented != 0 && it.has_offline && L > 1;
    const uint64_t key = static_cast<uint64_t>(it.bucket) | (static_cast<uint64_t>(sp) << 16) |
                         (static_cast<uint64_t>(it.k1_sk) << 17) | (graph_gen << 20);
    auto f = graphs.find(key);
    if (f == graphs.end()) {
      static const bool no_tune = [] {
        const char* v = std::getenv("CS_NO_GEMM_TUNE");
        return v && v[0] == '1';
      }();
      if (!no_tune) tune_gemms(it.bucket);  // outside the capture: it times candidates
      GraphExec ge;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(s_compute, cudaStreamCaptureModeThreadLocal));
      try {
        ge.launches = enqueue_body(it.bucket, it.bucket, true);
      } catch (...) {
        cudaStreamEndCapture(s_compute, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CK(cudaStreamEndCapture(s_compute, &g));
      CK(cudaGraphInstantiate(&ge.exec, g, 0));
      CK(cudaGraphDestroy(g));
      f = graphs.emplace(key, ge).first;
    }
    CK(cudaGraphLaunch(f->second.exec, s_compute));
    launches += f->second.launches;
  } else {
    launches += enqueue_body(it.n_tok, it.n_ent, false);
  }
  CK(cudaEventRecord(ev_end, s_compute));
  CK(cudaEventRecord(ev_fwd_done, s_compute));
  CK(cudaGetLastError());
}

// Builds the iteration's device metadata into the pinned
// staging buffer and the attention parameters; false for bookkeeping-only.
static double host_ms_now() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static bool prepare_iteration(cs_engine* e, const cs_batch_entry* entries, int32_t n, uint64_t epoch) {
    if (e->it.active) throw std::logic_error("iterations overlap on the device");
    if (n < 1) throw std::invalid_argument("empty batch");
    if (n > e->max_ent) throw std::invalid_argument("plan has more entries than max_entries");
    auto& it = e->it;
    it = cs_engine::Iter{};
    it.epoch = epoch;
    it.entries.assign(entries, entries + n);
    csb::BlockPool& pool = *e->pool;

    // ---- host metadata: positions per 0.11 ----
    std::vector<int32_t> tok_ids, tok_pos, tok_slot, ent_q0(n), ent_qlen(n), ent_kvlen(n), ent_bt(n), ent_last(n);
    std::vector<int32_t> dec_ent, bt;
    std::vector<csk::PrefillTile> tiles;
    std::vector<int32_t> tile_keys;  // keys a tile's rows attend to (K2 work per KV head)
    bool seen_offline = false;
    int n_tok_on = 0, n_ent_on = 0, n_dec_on = 0, n_pt_on = 0, max_dec_pages = 0, max_pre_kv = 0;
    for (int i = 0; i < n; ++i) {
      const cs_batch_entry& be = entries[i];
      if (be.online && seen_offline) throw std::invalid_argument("online entries must form a prefix of the plan");
      if (!be.online) seen_offline = true;
      const csb::Req* r = pool.find(be.request_id);
      if (!r) throw std::logic_error("unknown request id in kv manager");
      std::vector<int32_t> pos;
      std::array<int64_t, 3> wr{be.request_id, -1, -1};
      if (be.kind == CS_DECODE) {
        if (be.compute_tokens != 1 || be.context_tokens < 1) throw std::invalid_argument("decode entry needs P=1, C>=1");
        pos.push_back(static_cast<int32_t>(be.context_tokens - 1));
        wr = {be.request_id, be.context_tokens - 1, be.context_tokens};
      } else if (be.kind == CS_PREFILL) {
        if (be.compute_tokens < 1) throw std::invalid_argument("prefill entry needs P>=1");
        for (int64_t p = 0; p < be.compute_tokens; ++p) pos.push_back(static_cast<int32_t>(be.context_tokens + p));
        wr = {be.request_id, be.context_tokens, be.context_tokens + be.compute_tokens};
      } else if (be.kind == CS_RECOMPUTE) {
        // Positions of the pages re-materialized by this build's allocation
        // (kv_cache.cpp:76-107), page order; BatchEntry.C is context_len.
        std::vector<size_t> pages;
        for (const csb::Growth& g : r->growth)
          if (g.was_discarded) pages.push_back(g.page);
        std::sort(pages.begin(), pages.end());
        for (size_t pg : pages)
          for (int64_t t = 0; t < r->pages[pg].tokens; ++t) pos.push_back(static_cast<int32_t>(pg * 16 + t));
        if (static_cast<int64_t>(pos.size()) != be.compute_tokens)
          throw std::logic_error("recompute entry does not match the re-materialized pages");
      } else {
        throw std::invalid_argument("unknown entry kind");
      }
      const int kv_len = pos.back() + 1;
      ent_q0[i] = static_cast<int32_t>(tok_pos.size());
      ent_qlen[i] = static_cast<int32_t>(pos.size());
      ent_kvlen[i] = kv_len;
      ent_bt[i] = static_cast<int32_t>(bt.size());
      const int n_pages = (kv_len + 15) / 16;
      pool.blocks_for_read(be.request_id, static_cast<size_t>(n_pages), bt, it.wait_h2d);
      for (int32_t p : pos) {
        tok_ids.push_back(csk::token_id(e->cfg.token_seed, be.request_id, p, e->vocab));
        tok_pos.push_back(p);
        tok_slot.push_back(bt[static_cast<size_t>(ent_bt[i] + p / 16)] * 16 + (p % 16));
      }
      ent_last[i] = static_cast<int32_t>(tok_pos.size()) - 1;
      if (pos.size() == 1) {
        dec_ent.push_back(i);
        max_dec_pages = std::max(max_dec_pages, n_pages);
      } else {
        // K2 work tiles: prefill_tile_rows() packed (token, head-in-group) rows
        const int rows = static_cast<int>(pos.size()) * e->G;
        max_pre_kv = std::max(max_pre_kv, kv_len);
        const int step = e->k2_pair ? csk::prefill_tc2_tile_rows() : csk::prefill_tile_rows();
        for (int r0 = 0; r0 < rows; r0 += step) {
          tiles.push_back({i, r0});
          const int last = std::min(r0 + step, rows) - 1;
          tile_keys.push_back(std::min(kv_len, pos[static_cast<size_t>(last / e->G)] + 1));
        }
      }
      if (be.online) {
        n_tok_on = static_cast<int>(tok_pos.size());
        n_ent_on = i + 1;
        n_dec_on = static_cast<int>(dec_ent.size());
        n_pt_on = static_cast<int>(tiles.size());
      }
      it.writes.push_back(wr);
    }
    const int T = static_cast<int>(tok_pos.size());
    if (T > e->max_tok) throw std::invalid_argument("plan exceeds max_batched_tokens");
    for (int i = 0; i < n; ++i) {
      const double q = ent_qlen[i], kv = ent_kvlen[i];
      if (ent_qlen[i] == 1) {
        it.k1_bytes += (kv * e->hkv + e->hq) * e->D * 2.0 * 2.0;
      } else {
        // causal pairs of a chunk whose last query sits at kv_len - 1
        it.k2_flops += (q * (kv - q) + q * (q + 1) / 2) * 4.0 * e->hq * e->D;
      }
    }
    it.n_tok = T;
    it.n_tok_on = n_tok_on;
    it.n_ent = n;
    it.n_ent_on = n_ent_on;
    it.n_dec = static_cast<int>(dec_ent.size());
    it.n_pt = static_cast<int>(tiles.size());
    it.has_offline = seen_offline;
    pool.on_forward_launched();
    it.active = true;  // from here on an error must end the iteration (cs_forward_launch)
    if (e->host_only || e->no_model || e->dry) return false;

    // ---- graph mode: decode-only plans of <= 256 rows replay a captured
    // CUDA graph of their bucket (sizes padded; kernels skip rows >= *_cur)
    static const bool no_graphs = [] {
      const char* v = std::getenv("CS_NO_GRAPHS");
      return v && v[0] == '1';
    }();
    it.graph = false;
    it.bucket = 0;
    if (e->graphs_enabled && !no_graphs && it.n_pt == 0 && it.n_dec == T && T <= 256) {
      int b = 8;
      while (b < T) b *= 2;
      if (b <= e->max_ent && b <= e->max_tok) {
        it.graph = true;
        it.bucket = b;
      }
    }
    const int Tcap = it.graph ? it.bucket : T;  // token-array stride
    const int Dcap = it.graph ? it.bucket : it.n_dec;

    // ---- split-K for K1: aim for ~4 CTAs per SM. The launch grid (and the
    // workspace stride) is SG; the active split count lives in the descriptor.
    int SG = 1, S = 1, pps = std::max(1, max_dec_pages);
    if (it.n_dec > 0) {
      const int target = 4 * e->sms;
      S = std::max(1, (target + it.n_dec * e->hkv - 1) / (it.n_dec * e->hkv));
      S = std::min(S, std::max(1, (max_dec_pages + 3) / 4));
      S = std::min(S, 128);  // attn_decode_combine_kernel stages <= 128 splits
      if (it.graph) {
        SG = std::min(128, std::max(1, (target + Dcap * e->hkv - 1) / (Dcap * e->hkv)));
        S = std::min(S, SG);
      }
      pps = (max_dec_pages + S - 1) / S;
      S = (max_dec_pages + pps - 1) / pps;
      if (!it.graph) SG = S;
      const size_t need = static_cast<size_t>(Dcap) * e->hkv * SG * e->G * (2 + e->D);
      if (SG > 1 && need > e->ws_floats) {
        if (e->ws) CK(cudaFree(e->ws));
        e->ws_floats = need * 2;
        CK(cudaMalloc(&e->ws, e->ws_floats * 4));
        e->drop_graphs();
      }
    }
    it.splits = SG;
    it.pps = pps;

    // ---- pack metadata: [desc | tok_ids | tok_pos | tok_slot | ent x5 (cap max_ent) | dec | tiles | bt] ----
    const size_t E = static_cast<size_t>(e->max_ent);
    size_t off = 0;
    auto region = [&](size_t bytes) {
      const size_t o = off;
      off = align_up(off + bytes, 16);
      return o;
    };
    const size_t o_desc = region(sizeof(csk::IterDesc));
    const size_t o_tok = region(sizeof(int32_t) * 3 * static_cast<size_t>(Tcap));
    const size_t o_ent = region(sizeof(int32_t) * 5 * E);
    const size_t o_dec = region(sizeof(int32_t) * (2 * static_cast<size_t>(Dcap) + 1) + 4);  // dec_ent | dec_pfx
    const size_t o_tiles = region((sizeof(csk::PrefillTile) + 4) * tiles.size() + 8);
    const size_t o_bt = region(sizeof(int32_t) * bt.size() + 4);
    const size_t total = off;
    if (total > e->meta_cap) {
      if (e->d_meta) CK(cudaFree(e->d_meta));
      if (e->h_meta) CK(cudaFreeHost(e->h_meta));
      e->meta_cap = align_up(total * 2, 1 << 20);
      CK(cudaMalloc(&e->d_meta, e->meta_cap));
      CK(cudaHostAlloc(&e->h_meta, e->meta_cap, cudaHostAllocMapped | cudaHostAllocPortable));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_meta_dev), e->h_meta, 0));
      e->drop_graphs();
    }
    uint8_t* h = e->h_meta;
    csk::IterDesc desc{};
    desc.n_tok_cur = desc.n_tok_all = T;
    desc.n_tok_on = n_tok_on;
    desc.n_ent_cur = desc.n_ent_all = n;
    desc.n_ent_on = n_ent_on;
    desc.n_dec_cur = desc.n_dec_all = it.n_dec;
    desc.n_dec_on = n_dec_on;
    desc.n_pt_cur = desc.n_pt_all = it.n_pt;
    desc.n_pt_on = n_pt_on;
    desc.dropped_at = -1;
    desc.dec_splits = S;
    desc.dec_pps = pps;
    desc.epoch = epoch;
    std::memcpy(h + o_desc, &desc, sizeof(desc));
    int32_t* ht = reinterpret_cast<int32_t*>(h + o_tok);
    std::memcpy(ht, tok_ids.data(), 4 * T);
    std::memcpy(ht + Tcap, tok_pos.data(), 4 * T);
    std::memcpy(ht + 2 * Tcap, tok_slot.data(), 4 * T);
    int32_t* he = reinterpret_cast<int32_t*>(h + o_ent);
    std::memcpy(he, ent_q0.data(), 4 * n);
    std::memcpy(he + E, ent_qlen.data(), 4 * n);
    std::memcpy(he + 2 * E, ent_kvlen.data(), 4 * n);
    std::memcpy(he + 3 * E, ent_bt.data(), 4 * n);
    std::memcpy(he + 4 * E, ent_last.data(), 4 * n);
    if (!dec_ent.empty()) {
      std::memcpy(h + o_dec, dec_ent.data(), 4 * dec_ent.size());
      // K1 stream-K: page-count prefix over the decode entries (online first)
      int32_t* pf = reinterpret_cast<int32_t*>(h + o_dec) + Dcap;
      pf[0] = 0;
      for (size_t k = 0; k < dec_ent.size(); ++k)
        pf[k + 1] = pf[k] + (ent_kvlen[static_cast<size_t>(dec_ent[k])] + 15) / 16;
    }
    if (!tiles.empty()) {
      // K2 launch order: heaviest tiles first (the block scheduler then runs a
      // longest-first list schedule over the SMs); ties keep plan order
      std::vector<int32_t> order(tiles.size());
      for (size_t k = 0; k < order.size(); ++k) order[k] = static_cast<int32_t>(k);
      std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return tile_keys[a] > tile_keys[b]; });
      std::memcpy(h + o_tiles, tiles.data(), sizeof(csk::PrefillTile) * tiles.size());
      std::memcpy(h + o_tiles + sizeof(csk::PrefillTile) * tiles.size(), order.data(), 4 * order.size());
    }
    std::memcpy(h + o_bt, bt.data(), 4 * bt.size());

    // split-K for K2 when the tile grid cannot fill the SMs (few prefill rows
    // over a long context): ctas x splits <= SMs (one wave), splits of >= 4
    // key tiles (512 keys), <= 64
    it.k2_splits = 1;
    it.k2_tps = 1 << 30;
    if (it.n_pt > 0) {
      const int ctas = it.n_pt * e->hkv * (e->k2_pair ? 2 : 1);  // SMs per unit: a CTA pair or one CTA
      const int kt = csk::prefill_tile_keys();
      const int max_kt = (max_pre_kv + kt - 1) / kt;
      if (ctas < e->sms && max_kt >= 8) {
        const int S2 = std::min({e->sms / ctas, max_kt / 4, 64});
        if (S2 > 1) {
          it.k2_tps = (max_kt + S2 - 1) / S2;
          it.k2_splits = (max_kt + it.k2_tps - 1) / it.k2_tps;
          const size_t need = static_cast<size_t>(it.n_pt) * e->hkv * it.k2_splits * (e->D + 2) *
                              (e->k2_pair ? csk::prefill_tc2_tile_rows() : csk::prefill_tile_rows());
          if (need > e->ws2_floats) {
            if (e->ws2) CK(cudaFree(e->ws2));
            e->ws2_floats = need * 2;
            CK(cudaMalloc(&e->ws2, e->ws2_floats * 4));
            e->drop_graphs();
          }
        }
      }
    }
    uint8_t* d = e->d_meta;
    csk::AttnParams& ap = it.ap;
    ap.qkv = e->qkv;
    ap.out = e->attn;
    ap.pool = e->kv;
    ap.desc = reinterpret_cast<const csk::IterDesc*>(d + o_desc);
    it.d_tok_ids = reinterpret_cast<const int32_t*>(d + o_tok);
    ap.tok_pos = it.d_tok_ids + Tcap;
    it.d_tok_slot = it.d_tok_ids + 2 * Tcap;
    it.d_ent_last = reinterpret_cast<const int32_t*>(d + o_ent) + 4 * E;
    ap.ent_q0 = reinterpret_cast<const int32_t*>(d + o_ent);
    ap.ent_qlen = ap.ent_q0 + E;
    ap.ent_kvlen = ap.ent_q0 + 2 * E;
    ap.ent_bt = ap.ent_q0 + 3 * E;
    ap.block_table = reinterpret_cast<const int32_t*>(d + o_bt);
    ap.dec_ent = reinterpret_cast<const int32_t*>(d + o_dec);
    ap.dec_pfx = reinterpret_cast<const int32_t*>(d + o_dec) + Dcap;
    ap.ws_sk = e->ws_sk;
    // K1 kernel choice: with fewer (entry, KV head) pairs than resident
    // stream-K CTAs every pair is split anyway and equal page ranges keep all
    // SMs streaming (39 x 4.2K: -3.3% step time); with more pairs the
    // per-pair split-K kernel has no segment overhead (128 x 2K: -5.5%)
    // (profiles/r2/k1_streamk_ab.md). Graphs are keyed by the choice.
    it.k1_sk = e->sk_ctas > 0 && it.n_dec * e->hkv < e->sk_pairs_max;
    ap.sk_ctas = it.k1_sk ? e->sk_ctas : 0;
    ap.sk_stages = e->sk_stages;
    ap.tiles = reinterpret_cast<const csk::PrefillTile*>(d + o_tiles);
    ap.tile_order = reinterpret_cast<const int32_t*>(d + o_tiles + sizeof(csk::PrefillTile) * tiles.size());
    ap.ws = e->ws;
    ap.dec_cnt = e->dec_cnt;
    ap.num_layers = e->L;
    ap.hq = e->hq;
    ap.hkv = e->hkv;
    ap.qkv_stride = (e->hq + 2 * e->hkv) * e->D;
    ap.n_splits = it.splits;
    ap.ws2 = e->ws2;
    ap.k2_splits = it.k2_splits;
    ap.k2_pair = e->k2_pair ? 1 : 0;
    ap.k2_tiles_per_split = it.k2_tps;
    ap.pages_per_split = it.pps;
    ap.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(e->D));
    it.meta_bytes = static_cast<int64_t>(total);

    return true;
}

extern "C" {

const char* cs_last_error(void) { return g_err.c_str(); }
const char* cs_version(void) { return "conserve_b200 0.1 (sm_100a)"; }

void cs_config_default(cs_config* c) {
  std::memset(c, 0, sizeof(*c));
  // tiny config-1 decoder: 2 layers, d_model 256, 4 heads
  c->num_layers = 2;
  c->hidden = 256;
  c->n_heads = 4;
  c->n_kv_heads = 4;
  c->head_dim = 64;
  c->ffn = 512;
  c->vocab = 1024;
  c->rope_theta = 10000.f;
  c->rms_eps = 1e-5f;
  c->weight_seed = 1;
  c->token_seed = 1;
  c->kv_bytes_per_token = 2048;
  c->gpu_kv_capacity = 64LL * 16 * 2048;
  c->host_kv_capacity = 4096LL * 16 * 2048;
  c->d2h_bandwidth = 38797312000.0;
  c->h2d_bandwidth = 38797312000.0;
  c->gather_cost_us = 500.0;
  c->page_tokens = 16;
  c->safepoint_interval_layers = 1;
  c->max_batched_tokens = 512;
  c->incremental = 1;
  c->instrumented = 1;
  c->extra_blocks = -1;
  c->extra_host_slots = -1;
  c->max_entries = 0;
  c->layer_lookahead = 0;
  c->tp_rank = 0;
  c->tp_size = 1;
  c->device = 0;
  c->flags = 0;
}

int cs_create(const cs_config* cfg, cs_engine** out) {
  return guard([&] {
    validate(*cfg);
    auto e = std::make_unique<cs_engine>();
    e->cfg = *cfg;
    e->host_only = (cfg->flags & CS_FLAG_HOST_ONLY) != 0;
    e->no_model = (cfg->flags & CS_FLAG_NO_MODEL) != 0;
    e->tp = cfg->tp_size;
    e->rank = cfg->tp_rank;
    e->L = cfg->num_layers;
    e->hidden = cfg->hidden;
    e->hq = cfg->n_heads / cfg->tp_size;
    e->hkv = cfg->n_kv_heads / cfg->tp_size;
    e->G = cfg->n_heads / cfg->n_kv_heads;
    e->D = cfg->head_dim;
    e->ffn = cfg->ffn / cfg->tp_size;
    e->vocab = cfg->vocab;
    e->block_elems = static_cast<int64_t>(e->L) * 2 * e->hkv * 16 * e->D;
    e->max_tok = cfg->max_batched_tokens;
    e->max_ent = cfg->max_entries > 0 ? cfg->max_entries : 1024;

    const int64_t page_bytes = 16LL * cfg->kv_bytes_per_token;
    const int64_t base_blocks = (cfg->gpu_kv_capacity + page_bytes - 1) / page_bytes;
    const int64_t extra_b = cfg->extra_blocks >= 0 ? cfg->extra_blocks
                                                   : 2 * (e->max_tok / 16 + e->max_ent) + 64;
    const int64_t base_slots = (cfg->host_kv_capacity + page_bytes - 1) / page_bytes;
    const int64_t extra_s = cfg->extra_host_slots >= 0 ? cfg->extra_host_slots : e->max_ent + 64;

    csb::PoolConfig pc;
    pc.page_tokens = 16;
    pc.kv_bytes_per_token = cfg->kv_bytes_per_token;
    pc.gpu_capacity = cfg->gpu_kv_capacity;
    pc.host_capacity = cfg->host_kv_capacity;
    pc.d2h_bw = cfg->d2h_bandwidth;
    pc.h2d_bw = cfg->h2d_bandwidth;
    pc.gather_us = cfg->gather_cost_us;
    pc.incremental = cfg->incremental != 0;
    pc.n_blocks = base_blocks + extra_b;
    pc.n_slots = base_slots + extra_s;
    pc.moved_bytes_per_token = cfg->kv_bytes_per_token / cfg->tp_size;
    pc.fwd_quarantine = (cfg->flags & CS_FLAG_NO_FWD_QUARANTINE) == 0;

    if (!e->host_only) {
      CK(cudaSetDevice(cfg->device));
      CK(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, cfg->device));
      // the forward gets the block scheduler first; the host-link-bound
      // checkpoint / restore copies fill in behind it
      int prio_low = 0, prio_high = 0;
      CK(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
      const char* np = std::getenv("CS_NO_STREAM_PRIORITY");
      if (np && np[0] == '1') prio_low = prio_high = 0;
      CK(cudaStreamCreateWithPriority(&e->s_compute, cudaStreamNonBlocking, prio_high));
      CK(cudaStreamCreateWithPriority(&e->s_d2h, cudaStreamNonBlocking, prio_low));
      CK(cudaStreamCreateWithPriority(&e->s_h2d, cudaStreamNonBlocking, prio_low));
      CK(cudaEventCreate(&e->ev_start));
      CK(cudaEventCreate(&e->ev_end));
      CK(cudaEventCreateWithFlags(&e->ev_fwd_done, cudaEventDisableTiming));

      const size_t blk_bytes = static_cast<size_t>(e->block_elems) * 2;
      // + 1: the scratch block (BlockPool::scratch_block)
      CK(cudaMalloc(&e->kv, static_cast<size_t>(pc.n_blocks + 1) * blk_bytes));
      CK(cudaMemset(e->kv, 0, static_cast<size_t>(pc.n_blocks + 1) * blk_bytes));  // finite everywhere
      make_kv_tensor_map(&e->kv_map, e->kv, static_cast<uint64_t>(pc.n_blocks + 1) * e->L * 2 * e->hkv * 16, e->D);
      e->host_kv_bytes = static_cast<size_t>(pc.n_slots) * blk_bytes;
      e->host_kv = static_cast<__nv_bfloat16*>(alloc_host_pool(cfg->device, e->host_kv_bytes, &e->host_numa_node));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->host_kv_dev), e->host_kv, 0));
      {
        const char* zc = std::getenv("CS_KV_ZEROCOPY");
        e->kv_zerocopy = zc && zc[0] == '1';
        const char* sz = std::getenv("CS_KV_SMALL_ZC");
        e->kv_small_zc = !(sz && sz[0] == '0');
        if (!e->kv_zerocopy) {
          // 256 MiB per direction (>= one page): a larger job runs as a
          // sequence of pack + DMA chunks on its stream
          e->stage_elems = std::max<size_t>(static_cast<size_t>(e->block_elems), (256u << 20) / 2);
          for (int d = 0; d < 2; ++d) CK(cudaMalloc(&e->stage[d], e->stage_elems * 2));
        }
      }
      for (int d = 0; d < 2; ++d) {
        e->ring[d].cap = 8u << 20;
        CK(cudaHostAlloc(&e->ring[d].host, e->ring[d].cap, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->ring[d].dev), e->ring[d].host, 0));
      }
      CK(cudaHostAlloc(&e->mailbox, sizeof(csk::PreemptMailbox), cudaHostAllocMapped | cudaHostAllocPortable));
      std::memset(e->mailbox, 0, sizeof(csk::PreemptMailbox));
      e->mailbox->seen_layer = -1;
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->mailbox_dev), e->mailbox, 0));
      e->mover = std::make_unique<DeviceMover>(e.get());

      if (!e->no_model) {
        // weights, one allocation
        const int64_t H = e->hidden, qkv_rows = static_cast<int64_t>(e->hq + 2 * e->hkv) * e->D;
        const int64_t per_layer = 2 * H + qkv_rows * H + H * e->hq * e->D + 2LL * e->ffn * H + H * e->ffn;
        const int64_t total = 2LL * e->vocab * H + H + per_layer * e->L;
        CK(cudaMalloc(&e->weight_mem, static_cast<size_t>(total) * 2));
        __nv_bfloat16* p = static_cast<__nv_bfloat16*>(e->weight_mem);
        auto take = [&](int64_t n) {
          __nv_bfloat16* r = p;
          p += n;
          return r;
        };
        e->w.emb = take(e->vocab * H);
        e->w.lm_head = take(e->vocab * H);
        e->w.final_norm = take(H);
        const uint64_t seed = cfg->weight_seed;
        const float wscale = 0.02f * 1.7320508f;  // uniform with std 0.02
        csk::RowMap ident{1, {0, 0, 0}, {0, 0, 0}};
        cudaStream_t s = e->s_compute;
        csk::init_matrix(e->w.emb, e->vocab, H, H, 0, ident, seed, kTensorEmb, wscale, 0.f, s);
        csk::init_matrix(e->w.lm_head, e->vocab, H, H, 0, ident, seed, kTensorLm, wscale, 0.f, s);
        csk::init_matrix(e->w.final_norm, 1, H, H, 0, ident, seed, kTensorFinalNorm, 0.1f, 1.f, s);
        const int64_t Hq_g = cfg->n_heads, Hkv_g = cfg->n_kv_heads, F_g = cfg->ffn;
        {
          const char* v = std::getenv("CS_NO_GU_INTERLEAVE");
          e->gu_interleave = e->ffn % 128 == 0 && !(v && v[0] == '1');
        }
        __nv_bfloat16* gu_tmp = nullptr;
        if (e->gu_interleave) CK(cudaMalloc(&gu_tmp, 2LL * e->ffn * H * 2));
        for (int l = 0; l < e->L; ++l) {
          e->w.attn_norm.push_back(take(H));
          e->w.wqkv.push_back(take(qkv_rows * H));
          e->w.wo.push_back(take(H * e->hq * e->D));
          e->w.mlp_norm.push_back(take(H));
          e->w.wgu.push_back(take(2LL * e->ffn * H));
          e->w.wd.push_back(take(H * e->ffn));
          csk::init_matrix(e->w.attn_norm[l], 1, H, H, 0, ident, seed, tensor_id(l, kWAttnNorm), 0.1f, 1.f, s);
          csk::init_matrix(e->w.mlp_norm[l], 1, H, H, 0, ident, seed, tensor_id(l, kWMlpNorm), 0.1f, 1.f, s);
          // qkv: global rows [q heads | k heads | v heads] x D; this rank's heads
          csk::RowMap qkv_map{3,
                              {0, e->hq * e->D, (e->hq + e->hkv) * e->D},
                              {static_cast<int64_t>(e->rank) * e->hq * e->D,
                               Hq_g * e->D + static_cast<int64_t>(e->rank) * e->hkv * e->D,
                               (Hq_g + Hkv_g) * e->D + static_cast<int64_t>(e->rank) * e->hkv * e->D}};
          csk::init_matrix(e->w.wqkv[l], qkv_rows, H, H, 0, qkv_map, seed, tensor_id(l, kWQkv), wscale, 0.f, s);
          // o_proj: row-parallel -> this rank's input columns
          csk::init_matrix(e->w.wo[l], H, e->hq * e->D, Hq_g * e->D, static_cast<int64_t>(e->rank) * e->hq * e->D,
                           ident, seed, tensor_id(l, kWO), wscale, 0.f, s);
          csk::RowMap gu_map{2, {0, e->ffn, 0}, {static_cast<int64_t>(e->rank) * e->ffn,
                                                 F_g + static_cast<int64_t>(e->rank) * e->ffn, 0}};
          if (e->gu_interleave) {
            // init in the gate | up order, then 128-row blocks interleaved
            const size_t blk = static_cast<size_t>(128) * H * 2;
            csk::init_matrix(gu_tmp, 2LL * e->ffn, H, H, 0, gu_map, seed, tensor_id(l, kWGu), wscale, 0.f, s);
            CK(cudaMemcpy2DAsync(e->w.wgu[l], 2 * blk, gu_tmp, blk, blk, e->ffn / 128, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpy2DAsync(reinterpret_cast<uint8_t*>(e->w.wgu[l]) + blk, 2 * blk,
                                 gu_tmp + static_cast<size_t>(e->ffn) * H, blk, blk, e->ffn / 128,
                                 cudaMemcpyDeviceToDevice, s));
          } else {
            csk::init_matrix(e->w.wgu[l], 2LL * e->ffn, H, H, 0, gu_map, seed, tensor_id(l, kWGu), wscale, 0.f, s);
          }
          csk::init_matrix(e->w.wd[l], H, e->ffn, F_g, static_cast<int64_t>(e->rank) * e->ffn, ident, seed,
                           tensor_id(l, kWD), wscale, 0.f, s);
        }
        CK(cudaGetLastError());
        if (gu_tmp) {
          CK(cudaStreamSynchronize(s));
          CK(cudaFree(gu_tmp));
        }
        // activations
        const int64_t T = e->max_tok;
        CK(cudaMalloc(&e->x, T * H * 2));
        CK(cudaMalloc(&e->xn, T * H * 2));
        CK(cudaMalloc(&e->qkv, T * qkv_rows * 2));
        CK(cudaMalloc(&e->attn, T * e->hq * e->D * 2));
        CK(cudaMalloc(&e->tmp, (T * H + 64) * 2));
        CK(cudaMemset(e->tmp, 0, (T * H + 64) * 2));
        if (e->tp > 1) {  // peer all-reduce exchange region (own allocation: IPC-exportable)
          e->xchg_part_elems = static_cast<size_t>(T * H + 64);
          const size_t xb = 2 * e->xchg_part_elems * 2 + 64;
          CK(cudaMalloc(&e->xchg, xb));
          CK(cudaMemset(e->xchg, 0, xb));
        }
        CK(cudaMalloc(&e->gu, T * 2 * e->ffn * 2));
        CK(cudaMalloc(&e->act, T * e->ffn * 2));
        CK(cudaMalloc(&e->xl, e->max_ent * H * 2));
        CK(cudaMalloc(&e->logits, static_cast<size_t>(e->max_ent) * e->vocab * 4));
        CK(cudaMalloc(&e->d_out, sizeof(csk::IterDesc) + 8 * e->max_ent));
        CK(cudaMalloc(&e->dec_cnt, sizeof(int32_t) * e->max_ent * e->hkv));
        CK(cudaMemset(e->dec_cnt, 0, sizeof(int32_t) * e->max_ent * e->hkv));
        {
          // K1 stream-K: one resident wave over every SM (CS_K1_SPLITK=1: the
          // per-(entry, head) split-K kernel instead, for A/B)
          // K2 on CTA pairs measured slower than the single-CTA kernel
          // (profiles/r2/k2_pair_ab.md): opt-in only (CS_K2_PAIR=1)
          const char* k2s = std::getenv("CS_K2_PAIR");
          e->k2_pair = e->D == 128 && k2s && k2s[0] == '1';
          const char* sk = std::getenv("CS_K1_SPLITK");
          const char* st = std::getenv("CS_K1_STAGES");
          e->sk_stages = st && st[0] == '3' ? 3 : 2;
          // CS_K1_SK_WAVES=w: w x (resident CTAs) equal ranges, so the block
          // scheduler rebalances the later waves across SMs that stream faster
          const char* wv = std::getenv("CS_K1_SK_WAVES");
          const int waves = wv ? std::max(1, std::atoi(wv)) : 1;
          if (!(sk && sk[0] == '1')) {
            e->sk_resident = csk::decode_sk_ctas_per_sm(e->D, e->G, e->sk_stages) * e->sms;
            e->sk_ctas = e->sk_resident * waves;
            // stream-K below this many (sequence, KV head) pairs, per-pair
            // split-K above: the crossover sits ~15% above one resident wave
            // (56 x 4.3K: stream-K -1.7%; 64 x 4.2K: equal; 80+ rows: split-K
            // better, r3s); CS_K1_SK_PAIRS overrides, for A/B
            const char* sp = std::getenv("CS_K1_SK_PAIRS");
            e->sk_pairs_max = sp ? std::atoi(sp) : e->sk_resident * 115 / 100;
          }
          if (e->sk_ctas > 0) {
            const size_t n = static_cast<size_t>(e->sk_ctas) * 2 * e->G * (e->D + 2);
            CK(cudaMalloc(&e->ws_sk, n * 4));
          }
        }
        CK(cudaHostAlloc(&e->h_out, sizeof(csk::IterDesc) + 8 * e->max_ent, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_out_dev), e->h_out, 0));
        CKB(cublasCreate(&e->blas));
        CKB(cublasSetStream(e->blas, e->s_compute));
        CK(cudaMalloc(&e->blas_ws, 64u << 20));
        CKB(cublasSetWorkspace(e->blas, e->blas_ws, 64u << 20));
        CKB(cublasSetMathMode(e->blas, CUBLAS_DEFAULT_MATH));
        CKB(cublasLtCreate(&e->lt));
        {
          // K7 for the M <= 256 projections: 2 (default) where start-up
          // tuning timed it faster than the best cuBLAS plan, 1 always, 0 never
          const char* nf = std::getenv("CS_NO_FUSE");
          e->fuse_epilogues = !(nf && nf[0] == '1');
          CK(cudaMalloc(&e->rope_tab, static_cast<size_t>(e->max_tok) * (e->D / 2) * sizeof(float2)));
          const char* ksk = std::getenv("CS_K7_SK");
          e->k7_sk = ksk && ksk[0] == '1';
          const char* v = std::getenv("CS_WGEMM");
          e->wgemm_mode = (v && v[0] == '1') ? 1 : (v && v[0] == '0') ? 0 : 2;
        }
        // Workspaces and the metadata buffer at their upper bounds, so no
        // iteration frees device memory (cudaFree synchronises the device:
        // it would stall the copy streams, and deadlock TP ranks that share
        // a device while a peer spins in the all-reduce).
        //   K1 splits: rows*hkv*splits < 2 * (4 * sms) whenever splits > 1
        //   K2 splits: tiles*hkv*splits < 2 * sms whenever splits > 1
        e->ws_floats = static_cast<size_t>(2 * 4 * e->sms) * e->G * (2 + e->D);
        CK(cudaMalloc(&e->ws, e->ws_floats * 4));
        //   K7 stream-K: [SM][2 slots][Mp <= 256][128 features] fp32 + per-tile counters
        if (e->k7_sk) {
          CK(cudaMalloc(&e->k7_ws, static_cast<size_t>(e->sms) * 2 * 256 * 128 * 4));
          CK(cudaMalloc(&e->k7_cnt, sizeof(int32_t) * 8192));
          CK(cudaMemset(e->k7_cnt, 0, sizeof(int32_t) * 8192));
        }
        e->ws2_floats = static_cast<size_t>(2 * e->sms) * (e->D + 2) * 256;
        CK(cudaMalloc(&e->ws2, e->ws2_floats * 4));
        const size_t E = static_cast<size_t>(e->max_ent);
        const size_t tiles_max = static_cast<size_t>(T) * e->G / 256 + E + 1;
        e->meta_cap = align_up(sizeof(csk::IterDesc) + 12 * static_cast<size_t>(T) + 32 * E + 8 +
                                   (sizeof(csk::PrefillTile) + 4) * (tiles_max + 1) +
                                   4 * (static_cast<size_t>(pc.n_blocks) + E + 1) + 8 * 16,
                               1 << 20);
        CK(cudaMalloc(&e->d_meta, e->meta_cap));
        CK(cudaHostAlloc(&e->h_meta, e->meta_cap, cudaHostAllocMapped | cudaHostAllocPortable));
        CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&e->h_meta_dev), e->h_meta, 0));
        // cuBLASLt algorithm choice for every decode-graph bucket now, at
        // start-up, instead of inside the first iteration of each bucket
        const char* nt = std::getenv("CS_NO_GEMM_TUNE");
        if (e->graphs_enabled && !(nt && nt[0] == '1'))
          for (int b = 8; b <= 256 && b <= e->max_ent && b <= e->max_tok; b *= 2) e->tune_gemms(b);
      }
      CK(cudaStreamSynchronize(e->s_compute));
      // globaltimer <-> CLOCK_MONOTONIC offset (preemption latency probe)
      {
        volatile uint64_t* mbx = reinterpret_cast<volatile uint64_t*>(const_cast<uint64_t*>(&e->mailbox->flag_host_ns));
        int64_t best = INT64_MAX;
        for (int rep = 0; rep < 5; ++rep) {
          e->mailbox->flag_host_ns = 0;
          e->mailbox->seen_gpu_ns = 0;
          csk::calib_clock(reinterpret_cast<volatile uint64_t*>(e->mailbox_dev), e->s_compute);
          struct timespec ts {0, 200000};
          nanosleep(&ts, nullptr);
          const uint64_t t0 = host_ns();
          *mbx = t0;
          while (e->mailbox->seen_gpu_ns == 0) {
          }
          if (e->mailbox->seen_gpu_ns != 1) {  // 1 = the kernel gave up (profiler)
            const int64_t off = static_cast<int64_t>(e->mailbox->seen_gpu_ns) - static_cast<int64_t>(t0);
            best = std::min(best, off);
          }
          CK(cudaStreamSynchronize(e->s_compute));
        }
        e->clock_offset_ns = best == INT64_MAX ? 0 : best;
        e->mailbox->flag_host_ns = 0;
        e->mailbox->seen_gpu_ns = 0;
        e->mailbox->seen_epoch = 0;
        e->mailbox->seen_layer = -1;
      }
    }
    e->pool = std::make_unique<csb::BlockPool>(pc, e->mover.get());
    *out = e.release();
  });
}

int cs_destroy(cs_engine* e) {
  if (!e) return CS_OK;
  if (std::getenv("CS_HOST_TIMERS") && e->host_launches > 0)
    std::fprintf(stderr,
                 "{\"host_timers\": {\"forwards\": %lld, \"prepare_ms\": %.1f, \"enqueue_ms\": %.1f, "
                 "\"wait_ms\": %.1f, \"post_ms\": %.1f}}\n",
                 static_cast<long long>(e->host_launches), e->host_prep_ms, e->host_enq_ms, e->host_wait_ms,
                 e->host_post_ms);
  return guard([&] {
    if (!e->host_only) {
      cudaDeviceSynchronize();
      e->drop_graphs();
      e->mover.reset();
      for (auto& r : e->ring) r.live.clear();
      if (e->blas) cublasDestroy(e->blas);
      for (auto& kv : e->lt_plans) {
        cublasLtMatmulDescDestroy(kv.second.op);
        cublasLtMatrixLayoutDestroy(kv.second.a);
        cublasLtMatrixLayoutDestroy(kv.second.b);
        cublasLtMatrixLayoutDestroy(kv.second.c);
      }
      if (e->lt) cublasLtDestroy(e->lt);
      if (e->comm) ncclCommDestroy(e->comm);
      for (void* p : e->opened_ptrs) cudaIpcCloseMemHandle(p);
      if (e->xchg) cudaFree(e->xchg);
      cudaFree(e->kv);
      free_host_pool(e->host_kv, e->host_kv_bytes, e->host_numa_node);
      for (int d = 0; d < 2; ++d)
        if (e->stage[d]) cudaFree(e->stage[d]);
      for (auto& r : e->ring) cudaFreeHost(r.host);
      cudaFreeHost(e->mailbox);
      cudaFree(e->weight_mem);
      for (void* p : {static_cast<void*>(e->x), static_cast<void*>(e->xn), static_cast<void*>(e->qkv),
                      static_cast<void*>(e->attn), static_cast<void*>(e->tmp), static_cast<void*>(e->gu),
                      static_cast<void*>(e->act), static_cast<void*>(e->xl), static_cast<void*>(e->logits),
                      static_cast<void*>(e->ws), static_cast<void*>(e->ws2), static_cast<void*>(e->dec_cnt),
                      static_cast<void*>(e->ws_sk), static_cast<void*>(e->k7_ws), static_cast<void*>(e->k7_cnt),
                      static_cast<void*>(e->rope_tab),
                      static_cast<void*>(e->d_meta),
                      static_cast<void*>(e->d_out),
                      e->blas_ws})
        if (p) cudaFree(p);
      if (e->h_meta) cudaFreeHost(e->h_meta);
      if (e->h_out) cudaFreeHost(e->h_out);
      cudaEventDestroy(e->ev_start);
      cudaEventDestroy(e->ev_end);
      cudaEventDestroy(e->ev_fwd_done);
      cudaStreamDestroy(e->s_compute);
      cudaStreamDestroy(e->s_d2h);
      cudaStreamDestroy(e->s_h2d);
    }
    delete e;
  });
}

int cs_nccl_unique_id(uint8_t out_id[128]) {
  return guard([&] {
    ncclUniqueId id;
    CKN(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "nccl id size");
    std::memcpy(out_id, &id, 128);
  });
}

int cs_nccl_init(cs_engine* e, const uint8_t id[128]) {
  return guard([&] {
    if (e->tp <= 1) return;
    ncclUniqueId nid;
    std::memcpy(&nid, id, 128);
    CK(cudaSetDevice(e->cfg.device));
    CKN(ncclCommInitRank(&e->comm, e->tp, nid, e->rank));
  });
}

int cs_tp_exchange_ptr(cs_engine* e, void** out) {
  return guard([&] {
    if (!e->xchg) throw std::logic_error("no exchange region: tp_size must be > 1 with a model");
    *out = e->xchg;
  });
}

int cs_tp_exchange_ipc_handle(cs_engine* e, uint8_t out[64]) {
  return guard([&] {
    if (!e->xchg) throw std::logic_error("no exchange region: tp_size must be > 1 with a model");
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "ipc handle size");
    CK(cudaIpcGetMemHandle(&h, e->xchg));
    std::memcpy(out, &h, 64);
  });
}

static void attach_common(cs_engine* e, const std::vector<uint8_t*>& peers, bool same_device) {
  if (static_cast<int>(peers.size()) != e->tp) throw std::invalid_argument("need one exchange region per rank");
  if (e->tp > 8) throw std::invalid_argument("peer all-reduce supports up to 8 ranks");
  if (peers[static_cast<size_t>(e->rank)] != e->xchg) throw std::invalid_argument("own exchange region out of place");
  e->peer_xchg = peers;
  e->p2p = true;
  e->part_slot = 0;
  // same-device (loopback) peers run concurrently with this kernel's
  // spinning blocks: keep all ranks' spinners together at <= 32 CTAs so the
  // ranks still behind get SMs for their layer kernels
  e->p2p_blocks = same_device ? std::max(2, 32 / e->tp) : 2 * e->sms;
  if (const char* m = std::getenv("CS_P2P_ALLREDUCE")) {
    e->p2p_mode = std::strcmp(m, "twoshot") == 0 ? 2 : std::strcmp(m, "oneshot") == 0 ? 1 : 0;
  }
  e->drop_graphs();
}

int cs_tp_attach_peers(cs_engine* e, void* const* peers, int32_t n, int32_t same_device) {
  return guard([&] {
    std::vector<uint8_t*> v;
    for (int i = 0; i < n; ++i) v.push_back(static_cast<uint8_t*>(peers[i]));
    attach_common(e, v, same_device != 0);
  });
}

int cs_tp_attach_ipc(cs_engine* e, const uint8_t* handles, int32_t n) {
  return guard([&] {
    std::vector<uint8_t*> v(static_cast<size_t>(n), nullptr);
    CK(cudaSetDevice(e->cfg.device));
    for (int i = 0; i < n; ++i) {
      if (i == e->rank) {
        v[static_cast<size_t>(i)] = e->xchg;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles + 64 * i, 64);
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e->opened_ptrs.push_back(p);
      v[static_cast<size_t>(i)] = static_cast<uint8_t*>(p);
    }
    attach_common(e, v, false);
  });
}

// ------------------------------------------------------------ KV pool API --
int cs_kv_register_request(cs_engine* e, int64_t id, int32_t online) {
  return guard([&] { e->pool->register_request(id, online != 0); });
}
int cs_kv_allocate(cs_engine* e, int64_t id, int64_t n, int64_t now, cs_alloc_result* out) {
  (void)now;
  return guard([&] { *out = e->pool->allocate(id, n); });
}
int cs_kv_commit(cs_engine* e, int64_t id) { return guard([&] { e->pool->commit(id); }); }
int cs_kv_rollback(cs_engine* e, int64_t id) { return guard([&] { e->pool->rollback(id); }); }
int cs_kv_evict_request_gpu(cs_engine* e, int64_t id, int64_t now, int64_t max_pages, cs_evict_stats* out) {
  (void)now;
  return guard([&] { *out = e->pool->evict_request_gpu(id, max_pages); });
}
int cs_kv_discard_request(cs_engine* e, int64_t id, int64_t now, cs_evict_stats* out) {
  (void)now;
  return guard([&] { *out = e->pool->discard_request(id); });
}
int cs_kv_release_offline_pages_on_demand(cs_engine* e, int64_t needed, int64_t now, int64_t* freed,
                                          int64_t* discards, int64_t cap, int64_t* n_discards) {
  (void)now;
  return guard([&] {
    csb::ReleaseResult r = e->pool->release_offline_pages_on_demand(needed);
    *freed = r.freed_pages;
    *n_discards = static_cast<int64_t>(r.discards.size());
    for (size_t i = 0; i < r.discards.size() && static_cast<int64_t>(i) < cap; ++i) {
      discards[2 * i] = r.discards[i].first;
      discards[2 * i + 1] = r.discards[i].second;
    }
  });
}
int cs_kv_releasable_offline_pages_now(cs_engine* e, int64_t* out) {
  return guard([&] { *out = e->pool->releasable_offline_pages_now(); });
}
int cs_kv_stage_checkpoint(cs_engine* e, int64_t id, int64_t from, int64_t to) {
  return guard([&] { e->pool->stage_checkpoint(id, from, to); });
}
int cs_kv_flush_checkpoints(cs_engine* e, int64_t now, cs_transfer_job* job, int32_t* has_job) {
  return guard([&] {
    auto j = e->pool->flush_checkpoints(now);
    *has_job = j.has_value() ? 1 : 0;
    if (j) *job = *j;
  });
}
int cs_kv_resume_cost(cs_engine* e, int64_t id, cs_resume_cost* out) {
  return guard([&] { *out = e->pool->resume_cost(id); });
}
int cs_kv_fully_resident(cs_engine* e, int64_t id, int32_t* out) {
  return guard([&] { *out = e->pool->fully_resident(id) ? 1 : 0; });
}
int cs_kv_prefetch_inflight(cs_engine* e, int64_t id, int32_t* out) {
  return guard([&] { *out = e->pool->prefetch_inflight(id) ? 1 : 0; });
}
int cs_kv_start_prefetch(cs_engine* e, int64_t id, int64_t now, cs_transfer_job* job, int32_t* has_job) {
  return guard([&] {
    auto j = e->pool->start_prefetch(id, now);
    *has_job = j.has_value() ? 1 : 0;
    if (j) *job = *j;
  });
}
int cs_kv_recompute_chunk(cs_engine* e, int64_t id, int64_t desired, int64_t cap, int64_t* out) {
  return guard([&] { *out = e->pool->recompute_chunk(id, desired, cap); });
}
int cs_kv_on_transfer_done(cs_engine* e, int64_t job_id, int64_t now, cs_transfer_done* out) {
  (void)now;
  return guard([&] {
    csb::DoneResult r = e->pool->on_transfer_done(job_id);
    out->freed_pages = r.freed_pages;
    out->n_became_resident = static_cast<int32_t>(r.became_resident.size());
    for (size_t i = 0; i < r.became_resident.size() && i < 4; ++i) out->became_resident[i] = r.became_resident[i];
  });
}
// Real completion of a reference transfer job (SURVEY.md 8b "Completion"):
// done = its device copy finished; *ms = the copy's device time (-1 while
// running, 0 when it moved nothing on the device).
static void job_state(cs_engine* e, int64_t job_id, bool wait, int32_t* done, double* ms) {
  const auto [dir, ord] = e->pool->job_device(job_id);
  *done = 1;
  if (ms) *ms = 0;
  if (ord == 0 || !e->mover) return;
  if (wait) {
    if (cudaEvent_t ev = e->mover->pending_event(dir, ord)) CK(cudaEventSynchronize(ev));
  }
  e->mover->poll(dir);
  if (e->mover->done[dir] < ord) {
    *done = 0;
    if (ms) *ms = -1;
    return;
  }
  auto f = e->mover->ms_of[dir].find(ord);
  if (ms) *ms = f == e->mover->ms_of[dir].end() ? -1 : f->second;
}
int cs_job_poll(cs_engine* e, int64_t job_id, int32_t* done, double* ms) {
  return guard([&] { job_state(e, job_id, false, done, ms); });
}
int cs_job_wait(cs_engine* e, int64_t job_id, double* ms) {
  return guard([&] {
    int32_t d = 0;
    job_state(e, job_id, true, &d, ms);
  });
}
int cs_kv_on_request_paused(cs_engine* e, int64_t id, uint64_t seq) {
  return guard([&] { e->pool->on_request_paused(id, seq); });
}
int cs_kv_on_request_active(cs_engine* e, int64_t id) { return guard([&] { e->pool->on_request_active(id); }); }
int cs_kv_release_request(cs_engine* e, int64_t id) { return guard([&] { e->pool->release_request(id); }); }
int cs_kv_note_written(cs_engine* e, int64_t id, int64_t w0, int64_t w1) {
  return guard([&] { e->pool->note_written(id, w0, w1); });
}
int cs_kv_stats_get(cs_engine* e, cs_kv_stats* o) {
  return guard([&] {
    if (e->mover) {
      e->mover->poll(CS_D2H);
      e->mover->poll(CS_H2D);
    }
    const csb::BlockPool& p = *e->pool;
    o->gpu_used_bytes = p.gpu_used();
    o->gpu_free_bytes = p.gpu_free();
    o->host_used_bytes = p.host_used();
    o->gpu_free_pages = p.gpu_free_pages();
    o->page_bytes = p.page_bytes();
    o->total_d2h_bytes = p.total_d2h();
    o->total_h2d_bytes = p.total_h2d();
    o->recompute_tagged_tokens = p.recompute_tagged();
    o->transfers_inflight = p.transfers_inflight() ? 1 : 0;
    o->n_blocks = p.n_blocks();
    o->free_blocks = p.free_blocks();
    o->quarantined_blocks = p.quarantined_blocks();
    o->n_host_slots = p.n_slots();
    o->free_host_slots = p.free_slots();
    o->moved_d2h_bytes = p.moved_d2h();
    o->moved_h2d_bytes = p.moved_h2d();
    o->nonresident_reads = p.nonresident_reads();
    o->host_lru_evicted_pages = p.host_lru_evicted();
    o->unbacked_reads = p.unbacked_reads();
    o->host_numa_node = e->host_numa_node;
    o->moved_d2h_ms = e->moved_ms[CS_D2H];
    o->kernel_launches = e->launches.load();
    o->moved_h2d_ms = e->moved_ms[CS_H2D];
  });
}
int cs_kv_request_info(cs_engine* e, int64_t id, int64_t* gpu_pages, int64_t* covered, int64_t* pending) {
  return guard([&] {
    *gpu_pages = e->pool->request_gpu_pages(id);
    *covered = e->pool->covered_tokens(id);
    *pending = e->pool->pending_append_tokens(id);
  });
}
int cs_kv_audit(cs_engine* e) { return guard([&] { e->pool->audit(); }); }
int cs_kv_page_table_json(cs_engine* e, int64_t id, char* buf, size_t cap, size_t* len) {
  return guard([&] {
    const std::string s = e->pool->page_table_json(id);
    *len = s.size();
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, s.size());
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}
int cs_kv_block_table(cs_engine* e, int64_t id, int32_t* blocks, int32_t* slots, int64_t cap, int64_t* n) {
  return guard([&] {
    const csb::Req* r = e->pool->find(id);
    if (!r) throw std::logic_error("unknown request id in kv manager");
    *n = static_cast<int64_t>(r->pages.size());
    for (int64_t i = 0; i < *n && i < cap; ++i) {
      if (blocks) blocks[i] = r->pages[static_cast<size_t>(i)].block;
      if (slots) slots[i] = r->pages[static_cast<size_t>(i)].slot;
    }
  });
}

// ---------------------------------------------------------------- forward --
int cs_forward_launch(cs_engine* e, const cs_batch_entry* entries, int32_t n, uint64_t epoch) {
  const int rc = guard([&] {
    const double h0 = host_ms_now();
    if (!prepare_iteration(e, entries, n, epoch)) return;
    const double h1 = host_ms_now();
    e->host_prep_ms += h1 - h0;
    auto& it = e->it;
    // the forward's device time starts here, so a stall on a restore below
    // counts as time of this iteration
    CK(cudaEventRecord(e->ev_start, e->s_compute));
    // restores the reference already counts complete may still be copying:
    // the forward (not the host) waits for the ones writing blocks it reads
    if (it.wait_h2d > 0 && e->mover && e->mover->done_prefix(CS_H2D) < it.wait_h2d) {
      if (cudaEvent_t w = e->mover->pending_event(CS_H2D, it.wait_h2d)) CK(cudaStreamWaitEvent(e->s_compute, w, 0));
    }
    csk::sm_copy(e->d_meta, e->h_meta_dev, static_cast<size_t>(it.meta_bytes), e->s_compute);
    e->any_forward = true;
    it.active = true;
    it.device_m = e->use_pf(it.n_tok, (e->hq + 2 * e->hkv) * e->D, e->hidden) && !it.graph;
    e->enqueue_layers();
    e->host_enq_ms += host_ms_now() - h1;
    ++e->host_launches;
  });
  if (rc != CS_OK && e->it.active) {  // balance the pool's forward counters
    e->it.active = false;
    e->pool->on_forward_completed();
  }
  return rc;
}

// Times the paged-attention kernels alone (layer 0) for one plan: reps
// back-to-back launches between CUDA events on the compute stream. The plan's
// pages must be allocated. *bytes = algorithmic K/V + Q/O bytes per launch
// (sum kv_len*Hkv*d*2*2 + sum P*Hq*d*2*2), *flops = causal
// attention flops per launch (4*Hq*d per query-key pair).
int cs_bench_attention(cs_engine* e, const cs_batch_entry* entries, int32_t n, int32_t reps, double* ms_per_launch,
                       int64_t* bytes, int64_t* flops) {
  return guard([&] {
    if (!prepare_iteration(e, entries, n, 0)) throw std::logic_error("attention bench needs a device engine");
    auto& it = e->it;
    csk::sm_copy(e->d_meta, e->h_meta_dev, static_cast<size_t>(it.meta_bytes), e->s_compute);
    csk::AttnParams ap = it.ap;
    ap.layer = 0;
    for (int w = 0; w < 2; ++w) csk::launch_attention(ap, &e->kv_map, e->D, e->G, it.n_dec, it.n_pt, e->s_compute);
    CK(cudaEventRecord(e->ev_start, e->s_compute));
    for (int r = 0; r < reps; ++r) csk::launch_attention(ap, &e->kv_map, e->D, e->G, it.n_dec, it.n_pt, e->s_compute);
    CK(cudaEventRecord(e->ev_end, e->s_compute));
    CK(cudaEventSynchronize(e->ev_end));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e->ev_start, e->ev_end));
    *ms_per_launch = ms / reps;
    int64_t b = 0, f = 0;
    for (int i = 0; i < n; ++i) {
      const cs_batch_entry& be = entries[i];
      const int64_t q = (be.kind == CS_DECODE) ? 1 : be.compute_tokens;
      const int64_t kv = (be.kind == CS_DECODE) ? be.context_tokens : be.context_tokens + be.compute_tokens;
      b += kv * e->hkv * e->D * 2 * 2 + q * e->hq * e->D * 2 * 2;
      // causal pairs: query j (0-based within the chunk) sees C + j + 1 keys
      const int64_t pairs = (be.kind == CS_DECODE) ? be.context_tokens
                                                   : q * be.context_tokens + q * (q + 1) / 2;
      f += pairs * 4LL * e->hq * e->D;
    }
    *bytes = b;
    *flops = f;
    it.active = false;
    e->pool->on_forward_completed();
  });
}

int cs_bench_gemm(cs_engine* e, int32_t M, int32_t N, int32_t K, int32_t reps, double* ms_k7, double* ms_cublas,
                  double* max_abs_diff, double* max_abs_ref) {
  return guard([&] {
    if (e->host_only || e->no_model) throw std::logic_error("gemm bench needs a device engine");
    if (!csk::wgemm_supported(M, N, K)) throw std::invalid_argument("gemm bench: M <= 256, N % 128, K % 64");
    __nv_bfloat16 *x = nullptr, *w = nullptr, *y7 = nullptr, *yb = nullptr;
    const size_t nx = static_cast<size_t>(M) * K, nw = static_cast<size_t>(N) * K, ny = static_cast<size_t>(M) * N;
    // rotate over copies of W totalling >= 256 MB: every launch streams its
    // weights from HBM, as in a decode step (the L2 holds 126 MB)
    const int copies = static_cast<int>(std::max<size_t>(1, ((256u << 20) + nw * 2 - 1) / (nw * 2)));
    CK(cudaMalloc(&x, nx * 2));
    CK(cudaMalloc(&w, nw * 2 * copies));
    CK(cudaMalloc(&y7, ny * 2));
    CK(cudaMalloc(&yb, ny * 2));
    csk::fill_pool(x, nx, 11, e->s_compute);
    for (int c = 0; c < copies; ++c) csk::fill_pool(w + nw * c, nw, 12, e->s_compute);
    const int saved = e->wgemm_mode;
    auto time = [&](bool k7, __nv_bfloat16* y) {
      e->wgemm_mode = k7 ? 1 : 0;
      for (int r = 0; r < 3; ++r) e->gemm(x, w + nw * (r % copies), y, M, N, K, false);
      CK(cudaEventRecord(e->ev_start, e->s_compute));
      for (int r = 0; r < reps; ++r) e->gemm(x, w + nw * (r % copies), y, M, N, K, false);
      CK(cudaEventRecord(e->ev_end, e->s_compute));
      CK(cudaEventSynchronize(e->ev_end));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e->ev_start, e->ev_end));
      return static_cast<double>(ms) / reps;
    };
    try {
      *ms_k7 = time(true, y7);
      *ms_cublas = time(false, yb);
    } catch (...) {
      e->wgemm_mode = saved;
      throw;
    }
    e->wgemm_mode = saved;
    CK(cudaGetLastError());
    std::vector<__nv_bfloat16> h7(ny), hb(ny);
    CK(cudaMemcpy(h7.data(), y7, ny * 2, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hb.data(), yb, ny * 2, cudaMemcpyDeviceToHost));
    double md = 0, mr = 0;
    for (size_t i = 0; i < ny; ++i) {
      const double a = __bfloat162float(h7[i]), b = __bfloat162float(hb[i]);
      md = std::max(md, std::fabs(a - b));
      mr = std::max(mr, std::fabs(b));
    }
    *max_abs_diff = md;
    *max_abs_ref = mr;
    cudaFree(x);
    cudaFree(w);
    cudaFree(y7);
    cudaFree(yb);
  });
}

int cs_preempt_signal(cs_engine* e, uint64_t epoch) {
  return guard([&] {
    if (e->host_only) return;
    e->mailbox->flag_host_ns = host_ns();
    __atomic_thread_fence(__ATOMIC_SEQ_CST);
    e->mailbox->flag_epoch = epoch;
    e->it.signal_ns = e->mailbox->flag_host_ns;
  });
}

int cs_set_kernel_timing(cs_engine* e, int32_t on) {
  return guard([&] {
    e->ktime_on = on != 0;
    for (auto& t : e->ktime) t = cs_engine::KTime{};
  });
}

int cs_kernel_timing(cs_engine* e, int32_t cls, cs_ktime* out) {
  return guard([&] {
    if (cls < 0 || cls >= CS_KT_N) throw std::invalid_argument("unknown kernel class");
    out->launches = e->ktime[cls].launches;
    out->ms = e->ktime[cls].ms;
    out->units = e->ktime[cls].units;
  });
}

int cs_iter_elapsed(cs_engine* e, double* ms) {
  return guard([&] {
    *ms = -1;
    if (!e->it.active) throw std::logic_error("no iteration in flight");
    if (e->host_only || e->no_model || e->dry) return;
    const cudaError_t q = cudaEventQuery(e->ev_end);
    if (q == cudaErrorNotReady) return;
    CK(q);
    float v = 0;
    CK(cudaEventElapsedTime(&v, e->ev_start, e->ev_end));
    *ms = v;
  });
}

int cs_iter_retro_drop(cs_engine* e, int32_t layer) {
  return guard([&] {
    if (!e->it.active) throw std::logic_error("no iteration in flight");
    if (layer < 1) throw std::invalid_argument("drop layer must be >= 1");
    e->it.retro_layer = layer;
  });
}

int cs_iter_progress(cs_engine* e, int32_t* layer) {
  return guard([&] {
    *layer = -1;
    if (e->host_only || e->no_model || e->dry || !e->it.active || !e->mailbox) return;
    const uint64_t p = e->mailbox->progress;
    if (p / 1024ull == e->it.epoch) *layer = static_cast<int32_t>(p % 1024ull);
  });
}

int cs_iter_poll(cs_engine* e, int32_t* done) {
  return guard([&] {
    if (!e->it.active) {
      *done = 1;
      return;
    }
    if (e->host_only || e->no_model || e->dry) {
      *done = 1;
      return;
    }
    const cudaError_t q = cudaEventQuery(e->ev_end);
    if (q == cudaErrorNotReady) {
      *done = 0;
      return;
    }
    CK(q);
    *done = 1;
  });
}

int cs_iter_wait(cs_engine* e, cs_iter_info* info, int32_t* out_tokens, int32_t cap, float* logits) {
  return guard([&] {
    auto& it = e->it;
    if (!it.active) throw std::logic_error("no iteration in flight");
    // any exit (CUDA error included) ends the iteration and balances the
    // pool's launched/completed forward counters
    struct End {
      cs_engine* e;
      bool done = false;
      ~End() {
        if (done) return;
        e->it.active = false;
        e->pool->on_forward_completed();
      }
    } end{e};
    cs_iter_info inf{};
    inf.preempted_at_layer = -1;
    inf.gemm_trunc_layer = -1;
    int n_alive = it.n_ent;
    const double w0 = host_ms_now();
    double w1 = w0;
    if (!(e->host_only || e->no_model || e->dry)) {
      // spin on the event (the iteration's end is the host loop's critical
      // path: a yielding/blocking wait adds its wake-up latency to every
      // iteration of the serving loop)
      static const bool block_wait = [] {
        const char* v = std::getenv("CS_WAIT_BLOCK");
        return v && v[0] == '1';
      }();
      if (block_wait) {
        CK(cudaEventSynchronize(e->ev_end));
      } else {
        for (;;) {
          const cudaError_t q = cudaEventQuery(e->ev_end);
          if (q == cudaSuccess) break;
          if (q != cudaErrorNotReady) CK(q);
        }
      }
      w1 = host_ms_now();
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e->ev_start, e->ev_end));
      inf.gpu_ms = ms;
      const auto* desc = reinterpret_cast<const csk::IterDesc*>(e->h_out);
      if (e->ktime_on && it.graph && desc->dropped_at < 0) {
        cs_engine::KTime& t = e->ktime[CS_KT_GRAPH];
        t.launches += 1;
        t.ms += ms;
        t.units += it.n_tok;
      }
      if (!e->kt_pending.empty()) {
        if (desc->dropped_at < 0) {
          for (size_t k = 0; k < e->kt_pending.size(); ++k) {
            float kms = 0;
            CK(cudaEventElapsedTime(&kms, e->kt_ev[2 * k], e->kt_ev[2 * k + 1]));
            const cs_engine::KtPending& kp = e->kt_pending[k];
            cs_engine::KTime& t = e->ktime[kp.cls];
            t.launches += kp.weight;
            t.ms += static_cast<double>(kms) * kp.weight;
            t.units += kp.units * kp.weight;
          }
        }
        e->kt_pending.clear();
      }
      // argmax keys: low 32 bits = ~id (0 -> -1 for rows past n_ent_cur)
      const uint64_t* keys = reinterpret_cast<const uint64_t*>(e->h_out + sizeof(csk::IterDesc));
      if (desc->dropped_at >= 0) {
        inf.preempted_at_layer = desc->dropped_at;
        n_alive = it.n_ent_on;
        if (it.signal_ns != 0) {
          const int64_t drop_host = static_cast<int64_t>(desc->drop_ns) - e->clock_offset_ns;
          inf.preempt_signal_to_drop_us = static_cast<double>(drop_host - static_cast<int64_t>(it.signal_ns)) / 1e3;
        }
        if (desc->start_ns != 0 && desc->drop_ns > desc->start_ns && desc->dropped_at > 0)
          inf.pre_drop_layer_us = static_cast<double>(desc->drop_ns - desc->start_ns) / 1e3 / desc->dropped_at;
      }
      if (desc->dropped_at < 0 && it.retro_layer >= 0) {
        inf.preempted_at_layer = it.retro_layer;
        n_alive = it.n_ent_on;
      }
      inf.n_outputs = n_alive;
      inf.h2d_bytes = it.meta_bytes;
      inf.d2h_bytes = static_cast<int64_t>(sizeof(csk::IterDesc) + sizeof(uint64_t) * (it.graph ? it.bucket : it.n_ent));
      // K8 layer GEMMs follow the device drop: the first layer after the
      // safepoint already runs every kernel on the truncated batch
      inf.gemm_trunc_layer = it.device_m ? inf.preempted_at_layer : -1;
      if (out_tokens)
        for (int i = 0; i < n_alive && i < cap; ++i)
          out_tokens[i] = static_cast<int32_t>(0xFFFFFFFFu - static_cast<uint32_t>(keys[i] & 0xFFFFFFFFull));
      if (logits && n_alive > 0)
        CK(cudaMemcpy(logits, e->logits, static_cast<size_t>(n_alive) * e->vocab * 4, cudaMemcpyDeviceToHost));
    } else {
      if (it.retro_layer >= 0) {
        inf.preempted_at_layer = it.retro_layer;
        n_alive = it.n_ent_on;
      }
      inf.n_outputs = n_alive;
    }
    inf.n_entries_after = n_alive;
    inf.done = 1;
    // KV written by the surviving entries (the known->written map of 0.11)
    for (int i = 0; i < n_alive; ++i) {
      const auto& wr = it.writes[static_cast<size_t>(i)];
      if (wr[1] >= 0 && e->pool->find(wr[0])) e->pool->note_written(wr[0], wr[1], wr[2]);
    }
    end.done = true;
    e->pool->on_forward_completed();
    it.active = false;
    if (info) *info = inf;
    e->host_wait_ms += w1 - w0;
    e->host_post_ms += host_ms_now() - w1;
  });
}

// ---------------------------------------------------------------- debug --
int cs_debug_read_block(cs_engine* e, int32_t block, void* dst, size_t bytes) {
  return guard([&] {
    const size_t bb = static_cast<size_t>(e->block_elems) * 2;
    if (bytes < bb) throw std::invalid_argument("buffer too small");
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(dst, e->kv + static_cast<size_t>(block) * e->block_elems, bb, cudaMemcpyDeviceToHost));
  });
}
int cs_debug_write_block(cs_engine* e, int32_t block, const void* src, size_t bytes) {
  return guard([&] {
    const size_t bb = static_cast<size_t>(e->block_elems) * 2;
    if (bytes < bb) throw std::invalid_argument("buffer too small");
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(e->kv + static_cast<size_t>(block) * e->block_elems, src, bb, cudaMemcpyHostToDevice));
  });
}
int cs_debug_read_host_slot(cs_engine* e, int32_t slot, void* dst, size_t bytes) {
  return guard([&] {
    const size_t bb = static_cast<size_t>(e->block_elems) * 2;
    if (bytes < bb) throw std::invalid_argument("buffer too small");
    // the slot is token-major [16][runs][D]; hand it out in the device
    // block's run-major [runs][16][D] order so callers compare them directly
    const size_t runs = static_cast<size_t>(e->L) * 2 * e->hkv, D = static_cast<size_t>(e->D);
    const __nv_bfloat16* src = e->host_kv + static_cast<size_t>(slot) * e->block_elems;
    auto* out = static_cast<__nv_bfloat16*>(dst);
    for (size_t t = 0; t < 16; ++t)
      for (size_t r = 0; r < runs; ++r) std::memcpy(out + (r * 16 + t) * D, src + (t * runs + r) * D, D * 2);
  });
}
int cs_debug_fill_pool(cs_engine* e, uint64_t seed) {
  return guard([&] {
    csk::fill_pool(e->kv, static_cast<size_t>(e->pool->n_blocks()) * e->block_elems, seed, e->s_compute);
    CK(cudaStreamSynchronize(e->s_compute));
  });
}
int cs_debug_read_weight(cs_engine* e, int32_t layer, int32_t which, void* dst, size_t bytes, size_t* needed) {
  return guard([&] {
    const int64_t H = e->hidden;
    const __nv_bfloat16* src = nullptr;
    int64_t n = 0;
    switch (which) {
      case 0: src = e->w.attn_norm[layer]; n = H; break;
      case 1: src = e->w.wqkv[layer]; n = static_cast<int64_t>(e->hq + 2 * e->hkv) * e->D * H; break;
      case 2: src = e->w.wo[layer]; n = H * e->hq * e->D; break;
      case 3: src = e->w.mlp_norm[layer]; n = H; break;
      case 4: src = e->w.wgu[layer]; n = 2LL * e->ffn * H; break;
      case 5: src = e->w.wd[layer]; n = H * e->ffn; break;
      case 6: src = e->w.emb; n = static_cast<int64_t>(e->vocab) * H; break;
      case 7: src = e->w.lm_head; n = static_cast<int64_t>(e->vocab) * H; break;
      case 8: src = e->w.final_norm; n = H; break;
      default: throw std::invalid_argument("unknown weight");
    }
    *needed = static_cast<size_t>(n) * 2;
    if (dst && bytes >= *needed) {
      if (which == 4 && e->gu_interleave) {  // hand out the gate | up order
        const size_t blk = static_cast<size_t>(128) * H * 2;
        CK(cudaMemcpy2D(dst, blk, src, 2 * blk, blk, e->ffn / 128, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy2D(static_cast<uint8_t*>(dst) + static_cast<size_t>(e->ffn) * H * 2, blk,
                        reinterpret_cast<const uint8_t*>(src) + blk, 2 * blk, blk, e->ffn / 128,
                        cudaMemcpyDeviceToHost));
      } else {
        CK(cudaMemcpy(dst, src, *needed, cudaMemcpyDeviceToHost));
      }
    }
  });
}
int cs_debug_read_activation(cs_engine* e, int32_t which, void* dst, size_t bytes) {
  return guard([&] {
    CK(cudaDeviceSynchronize());
    const __nv_bfloat16* src = which == 0 ? e->attn : (which == 1 ? e->x : e->qkv);
    CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  });
}
int cs_set_dry(cs_engine* e, int32_t dry) {
  return guard([&] {
    if (e->it.active) throw std::logic_error("cannot toggle dry mode with an iteration in flight");
    e->dry = dry != 0;
  });
}

int32_t cs_token_id(uint64_t seed, int64_t req, int64_t pos, int32_t vocab) {
  return csk::token_id(seed, req, pos, vocab);
}
float cs_hash_uniform(uint64_t seed, uint64_t tensor, uint64_t idx) { return csk::hash_uniform(seed, tensor, idx); }

int cs_sync(cs_engine* e) {
  return guard([&] {
    if (!e->host_only) CK(cudaDeviceSynchronize());
  });
}

}  // extern "C"
