/*
 * conserve_b200.h -- C-ABI of the B200-native ConServe co-serving data plane.
 *
 * This is the drop-in boundary for the hot path of the reference CPU simulator
 * (/root/reference/proj, arXiv 2410.01228). The reference has no plugin/FFI
 * layer; its seams are C++ calls inside SimEngine. Each export below replaces
 * one of those calls (file:line into /root/reference), with plain pointers and
 * sizes only -- no C++ or torch types cross this boundary.
 *
 *   reference seam                                   replaced by
 *   ------------------------------------------------ ----------------------------
 *   KvCacheManager(ClusterConfig,bool)  kv_cache.cpp:38-46      cs_create / cs_destroy
 *   KvCacheManager::* (allocate, commit, rollback, evict,       cs_kv_*
 *     release, stage, flush, prefetch, transfer-done, audit,
 *     page_table_json)  kv_cache.hpp:97-173
 *   oracle_latency(plan)  sim_engine.cpp:256 / perf_model.cpp:56-96   cs_forward_launch
 *   exec_->signal_preempt()  sim_engine.cpp:130                 cs_preempt_signal
 *   exec_->safepoint_check(layer)  sim_engine.cpp:149 /         cs_iter_wait (preempted_at)
 *     preemption.cpp:95-114
 *   TransferChannel::enqueue  kv_cache.cpp:23-36                real D2H/H2D streams; cs_job_*
 *
 * Conventions:
 *   - Every function returns int status: CS_OK (0) or a negative CS_ERR_*.
 *     No exception crosses the boundary; cs_last_error() gives a thread-local
 *     message. The error kinds mirror the reference's exception types
 *     (std::logic_error, std::invalid_argument, std::runtime_error,
 *     ConfigError) so an adapter can rethrow the same type.
 *   - The caller owns every host buffer it passes; the engine owns device
 *     memory, the pinned host KV pool, streams and events.
 *   - Single-threaded caller. cs_preempt_signal may be called
 *     from any thread.
 *   - Times are integer microseconds (coserve::UsecT, time.hpp:13-41).
 */
#ifndef CONSERVE_B200_H_
#define CONSERVE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status -- */
enum {
  CS_OK = 0,
  CS_ERR_LOGIC = -1,        /* std::logic_error (unknown id, audit failure, ...) */
  CS_ERR_INVALID = -2,      /* std::invalid_argument */
  CS_ERR_RUNTIME = -3,      /* std::runtime_error */
  CS_ERR_CONFIG = -4,       /* coserve::ConfigError */
  CS_ERR_CUDA = -5,         /* CUDA / cuBLAS / NCCL failure */
  CS_ERR_POOL = -6,         /* physical pool exhausted although byte accounting fit */
  CS_ERR_NOT_READY = -7     /* asynchronous object not complete yet (poll) */
};
const char* cs_last_error(void);
const char* cs_version(void);

/* ---------------------------------------------------------------- config -- */
/* Engine flags. */
enum {
  CS_FLAG_NO_MODEL = 1 << 0,     /* KV pool + checkpoint path only (no weights) */
  CS_FLAG_RESERVED1 = 1 << 1,
  CS_FLAG_RESERVED2 = 1 << 2,
  CS_FLAG_SYNC_DEBUG = 1 << 3,   /* synchronize after every launch (debug) */
  CS_FLAG_HOST_ONLY = 1 << 4,    /* bookkeeping only: no CUDA calls at all
                                    (CPU tests, oracle-clock shadow runs) */
  CS_FLAG_NO_FWD_QUARANTINE = 1 << 5 /* freed blocks need no forward to drain
                                        (bookkeeping-only call sequences) */
};

typedef struct cs_config {
  /* --- model shape (Llama-style decoder; SURVEY.md 8 model table) --- */
  int32_t num_layers;        /* == ClusterConfig::num_layers (config.hpp:34) */
  int32_t hidden;
  int32_t n_heads;           /* query heads (global, before sharding) */
  int32_t n_kv_heads;        /* KV heads (global) */
  int32_t head_dim;
  int32_t ffn;
  int32_t vocab;
  float rope_theta;
  float rms_eps;
  uint64_t weight_seed;      /* seeded random-init weights */
  uint64_t token_seed;       /* teacher-forced ids: id(req,pos) = hash(seed,req,pos) % vocab */
  /* --- cluster (mirrors coserve::ClusterConfig, config.hpp:33-59) --- */
  int64_t kv_bytes_per_token;    /* must equal 2*L*H_kv*d*2 (whole model) */
  int64_t gpu_kv_capacity;       /* bytes, byte-granular accounting as reference */
  int64_t host_kv_capacity;
  double d2h_bandwidth;          /* bytes/s; only for the modelled job timeline */
  double h2d_bandwidth;
  double gather_cost_us;
  int32_t page_tokens;           /* fixed at 16 (config.cpp:60) */
  int32_t safepoint_interval_layers;
  int64_t max_batched_tokens;
  int32_t incremental;           /* SchedulerPolicy::incremental() */
  int32_t instrumented;          /* SchedulerPolicy::instrumented() */
  /* --- B200 data-plane sizing --- */
  /* Physical-pool slack over ceil(cap/page_bytes). Each live request's
   * partial tail page counts only its tokens against the reference's byte
   * capacity but occupies a whole block, so the pool needs one spare block
   * per live request. <0 = auto: 2*(max_batched_tokens/16
   * + max_entries) + 64, i.e. it assumes at most ~max_entries live requests
   * hold partial pages; a deployment with more live (e.g. paused offline)
   * requests sets this to its live-request bound, else allocate may fail with
   * CS_ERR_POOL where the reference's byte accounting still succeeds. */
  int64_t extra_blocks;
  int64_t extra_host_slots;      /* host-pool slack (one slot per partially checkpointed page); <0 = auto: max_entries + 64 */
  int32_t max_entries;           /* max entries per plan (0 = 1024) */
  int32_t layer_lookahead;       /* unused since r2 (the forward is no longer host-paced); kept for ABI */
  /* --- sharding (KV-head groups) --- */
  int32_t tp_rank;
  int32_t tp_size;
  int32_t device;
  int32_t flags;                 /* CS_FLAG_* */
} cs_config;

/* Fills *cfg with the reference defaults (config.hpp:33-59) and the tiny
 * config-1 model shape; callers override fields. */
void cs_config_default(cs_config* cfg);

typedef struct cs_engine cs_engine;

int cs_create(const cs_config* cfg, cs_engine** out);
int cs_destroy(cs_engine* e);
/* NCCL communicator for tp_size > 1: rank 0 calls cs_nccl_unique_id, the
 * caller broadcasts the 128 bytes, every rank calls cs_nccl_init. */
int cs_nccl_unique_id(uint8_t out_id[128]);
int cs_nccl_init(cs_engine* e, const uint8_t id[128]);
/* Peer-memory all-reduce instead of NCCL: one kernel per
 * o_proj / down-proj reads every rank's partial buffer directly over NVLink
 * (device-side step flags; graph-safe). Each rank exports its exchange
 * region (cs_tp_exchange_ipc_handle, 64 bytes; the caller all-gathers them)
 * and attaches all ranks' regions in rank order (cs_tp_attach_ipc). Ranks in
 * one process (cs_tp_exchange_ptr / cs_tp_attach_peers) may share a device:
 * same_device != 0 keeps the spinning kernel small (loopback tests). */
int cs_tp_exchange_ptr(cs_engine* e, void** out);
int cs_tp_exchange_ipc_handle(cs_engine* e, uint8_t out[64]);
int cs_tp_attach_peers(cs_engine* e, void* const* peers, int32_t n, int32_t same_device);
int cs_tp_attach_ipc(cs_engine* e, const uint8_t* handles, int32_t n);

/* ------------------------------------------- KV block pool (C1 + C2 rows) -- */
/* Mirrors coserve::AllocResult / EvictStats / ResumeCost / TransferJob /
 * TransferDoneEffects (kv_cache.hpp:44-95). */
typedef struct { int32_t ok; int64_t shortfall_pages; } cs_alloc_result;
typedef struct { int64_t freed_pages, pending_pages, discarded_tokens; } cs_evict_stats;
typedef struct { int64_t host_only_pages, host_only_bytes, discarded_tokens; } cs_resume_cost;
enum { CS_D2H = 0, CS_H2D = 1 };
typedef struct {
  int64_t id;
  int32_t direction;       /* CS_D2H / CS_H2D */
  int64_t bytes;           /* reference byte count (known-token accounting) */
  int64_t enqueue_time, start_time, done_time;   /* modelled FIFO timeline (us) */
  double transfer_us, gather_us;
  int64_t moved_bytes;     /* bytes this rank actually moved over the host link */
} cs_transfer_job;
typedef struct {
  int64_t freed_pages;
  int32_t n_became_resident;
  int64_t became_resident[4];
} cs_transfer_done;

int cs_kv_register_request(cs_engine* e, int64_t id, int32_t online);
int cs_kv_allocate(cs_engine* e, int64_t id, int64_t n_tokens, int64_t now, cs_alloc_result* out);
int cs_kv_commit(cs_engine* e, int64_t id);
int cs_kv_rollback(cs_engine* e, int64_t id);
int cs_kv_evict_request_gpu(cs_engine* e, int64_t id, int64_t now, int64_t max_pages, cs_evict_stats* out);
int cs_kv_discard_request(cs_engine* e, int64_t id, int64_t now, cs_evict_stats* out);
/* ReleaseStats: freed pages plus (owner, discarded tokens) pairs written to
 * discards[2*i], discards[2*i+1] (capacity cap pairs; *n_discards = count). */
int cs_kv_release_offline_pages_on_demand(cs_engine* e, int64_t needed_pages, int64_t now,
                                          int64_t* freed_pages, int64_t* discards,
                                          int64_t cap, int64_t* n_discards);
int cs_kv_releasable_offline_pages_now(cs_engine* e, int64_t* out);
int cs_kv_stage_checkpoint(cs_engine* e, int64_t id, int64_t from_token, int64_t to_token);
/* Coalesces staged deltas into one D2H job (kv_cache.cpp:364-400) and launches
 * the gather on the D2H stream behind the last forward. *has_job = 0 if none. */
int cs_kv_flush_checkpoints(cs_engine* e, int64_t now, cs_transfer_job* job, int32_t* has_job);
int cs_kv_resume_cost(cs_engine* e, int64_t id, cs_resume_cost* out);
int cs_kv_fully_resident(cs_engine* e, int64_t id, int32_t* out);
int cs_kv_prefetch_inflight(cs_engine* e, int64_t id, int32_t* out);
/* Restore all HostOnly pages of one request into newly allocated blocks
 * (kv_cache.cpp:428-455), H2D on its own stream. */
int cs_kv_start_prefetch(cs_engine* e, int64_t id, int64_t now, cs_transfer_job* job, int32_t* has_job);
int cs_kv_recompute_chunk(cs_engine* e, int64_t id, int64_t desired, int64_t cap, int64_t* out);
/* Completion (kv_cache.cpp:471-520; the reference engine calls it at the job's
 * modelled done_time, sim_engine.cpp:242-248). Applies the bookkeeping without
 * waiting for the device: blocks and host slots stay quarantined until the
 * device jobs that touch them complete, a restore is stream-ordered after the
 * gathers still writing its slots, and the next forward after the restores
 * of the blocks it reads. Never blocks the caller. */
int cs_kv_on_transfer_done(cs_engine* e, int64_t job_id, int64_t now, cs_transfer_done* out);
/* Real completion of a transfer job (SURVEY.md 8b "Completion"): *done = 1
 * once its device copy finished; *ms = the copy's device time (-1 while it
 * runs, 0 if it moved nothing on the device). cs_job_wait blocks until done.
 * Replaces the reference's modelled TransferChannel done_time in live mode
 * (kv_cache.cpp:23-36). */
int cs_job_poll(cs_engine* e, int64_t job_id, int32_t* done, double* ms);
int cs_job_wait(cs_engine* e, int64_t job_id, double* ms);
int cs_kv_on_request_paused(cs_engine* e, int64_t id, uint64_t pause_seq);
int cs_kv_on_request_active(cs_engine* e, int64_t id);
int cs_kv_release_request(cs_engine* e, int64_t id);
/* Declares that the last forward wrote KV positions [w0, w1) of request id;
 * cs_iter_wait calls this itself for surviving entries. Used to map the
 * reference's known-token checkpoint ranges onto written positions
 * (SURVEY.md 0 item 11). */
int cs_kv_note_written(cs_engine* e, int64_t id, int64_t w0, int64_t w1);

typedef struct {
  int64_t gpu_used_bytes, gpu_free_bytes, host_used_bytes, gpu_free_pages, page_bytes;
  int64_t total_d2h_bytes, total_h2d_bytes, recompute_tagged_tokens;
  int32_t transfers_inflight;
  /* physical state (B200 only) */
  int64_t n_blocks, free_blocks, quarantined_blocks, n_host_slots, free_host_slots;
  int64_t moved_d2h_bytes, moved_h2d_bytes;
  int64_t nonresident_reads;     /* block-table reads of pages the reference marks non-resident (D3) */
  double moved_d2h_ms, moved_h2d_ms;  /* summed device time of the gather / scatter kernels */
  int64_t kernel_launches;       /* hand-written kernels launched so far (cuBLAS/NCCL excluded) */
  int64_t host_lru_evicted_pages; /* host copies dropped by the host LRU (kv_cache.cpp:326-362) */
  int64_t unbacked_reads;        /* block-table reads past a request's pages (reference defect D5) */
  int32_t host_numa_node;        /* NUMA node the pinned host pool is bound to (-1: not bound) */
} cs_kv_stats;
int cs_kv_stats_get(cs_engine* e, cs_kv_stats* out);
int cs_kv_request_info(cs_engine* e, int64_t id, int64_t* gpu_pages, int64_t* covered_tokens,
                       int64_t* pending_append_tokens);
/* Deep invariant check (kv_cache.cpp:566-620) plus the physical invariants
 * (every resident page owns a distinct block, free-list partition). */
int cs_kv_audit(cs_engine* e);
/* Same JSON as KvCacheManager::page_table_json (kv_cache.cpp:622-634). */
int cs_kv_page_table_json(cs_engine* e, int64_t id, char* buf, size_t cap, size_t* len);
/* Physical block ids (-1 = not resident) and host slot ids (-1 = none), one
 * per logical page. */
int cs_kv_block_table(cs_engine* e, int64_t id, int32_t* blocks, int32_t* slots, int64_t cap, int64_t* n);

/* -------------------------------- forward over a mixed batch (A1/A2/A5) -- */
/* Mirrors coserve::BatchEntry (perf_model.hpp:15-21); EntryKind order kept. */
enum { CS_PREFILL = 0, CS_DECODE = 1, CS_RECOMPUTE = 2 };
typedef struct {
  int64_t request_id;
  int64_t compute_tokens;   /* P */
  int64_t context_tokens;   /* C */
  int32_t kind;
  int32_t online;
} cs_batch_entry;

typedef struct {
  int32_t n_outputs;          /* sampled rows (decode + final prefill chunks) */
  int32_t preempted_at_layer; /* -1 if not preempted */
  int32_t n_entries_after;    /* entries that ran to the end */
  int32_t done;
  double gpu_ms;              /* device time of the iteration (events) */
  double preempt_signal_to_drop_us; /* host flag store -> device drop (calibrated clocks) */
  int64_t h2d_bytes;          /* plan metadata uploaded for this iteration */
  int64_t d2h_bytes;          /* sampled ids + descriptor read back */
  int32_t gemm_trunc_layer;   /* first layer whose GEMMs ran on the online rows (-1) */
  double pre_drop_layer_us;   /* dropped iterations: mean device layer time before the drop */
} cs_iter_info;

/* Launches the L-layer forward for one plan (online entries must form a
 * prefix, scheduler.cpp:183-317). Asynchronous. epoch tags the iteration
 * for the preemption flag. Outputs (argmax ids, one per
 * sampled row, entry order) are copied to out_tokens at cs_iter_wait. */
int cs_forward_launch(cs_engine* e, const cs_batch_entry* entries, int32_t n, uint64_t epoch);
/* Host flag store: drop offline entries at the next safepoint of the
 * iteration tagged epoch (preemption.cpp:95-114). */
int cs_preempt_signal(cs_engine* e, uint64_t epoch);
/* Waits for the running iteration. out_tokens (cap entries) receives sampled
 * ids; logits (optional, n_outputs x vocab fp32) the raw logits. Marks KV
 * written for surviving entries and releases quarantined blocks. */
int cs_iter_wait(cs_engine* e, cs_iter_info* info, int32_t* out_tokens, int32_t cap, float* logits);
int cs_iter_poll(cs_engine* e, int32_t* done);
/* Layer the in-flight instrumented forward has entered (its layer-head
 * kernel ran; -1 before layer 0 or when none is in flight). Lets a host
 * monitor time its flag store against the device's layer clock
 * (IterationExecution::safepoint_time, preemption.cpp:74-82). */
int cs_iter_progress(cs_engine* e, int32_t* layer);
/* Device time of the in-flight forward once it completed (*ms = -1 while it
 * runs; bookkeeping-only engines report -1). Does not end the iteration. */
int cs_iter_elapsed(cs_engine* e, double* ms);
/* Live mode (oracle/lockstep/live.cpp): the host's event loop decided the
 * in-flight iteration drops its offline entries at `layer`
 * (IterationExecution::apply_drop, preemption.cpp:105-114) after the device
 * already ran the whole plan. cs_iter_wait then treats it as dropped: only
 * the online prefix produces outputs and records written KV. */
int cs_iter_retro_drop(cs_engine* e, int32_t layer);

/* Per-kernel-class device timing for the roofline (bench): while enabled,
 * every non-graph launch of a class is bracketed by CUDA events on its
 * stream; totals cover iterations that completed without a drop.
 * units = algorithmic work of the timed launches: flops for
 * K8 (2*M*N*K), K2 (4*Hq*d per causal query-key pair) and the library
 * (cuBLAS) GEMMs of non-graph forwards (CS_KT_LIB), bytes for K1 (K/V read
 * + Q/O); CS_KT_GRAPH counts whole decode-graph forwards (units = token
 * rows). Enabling resets the totals. */
enum { CS_KT_K8 = 0, CS_KT_K2 = 1, CS_KT_K1 = 2, CS_KT_LIB = 3, CS_KT_GRAPH = 4, CS_KT_N = 5 };
typedef struct {
  int64_t launches;
  double ms;
  double units;
} cs_ktime;
int cs_set_kernel_timing(cs_engine* e, int32_t on);
int cs_kernel_timing(cs_engine* e, int32_t cls, cs_ktime* out);

/* --------------------------------------------------------------- replay -- */
/* Replays a recorded reference call log (oracle/lockstep/recorder.cpp) through
 * this C-ABI: the same sequence of KvCacheManager calls, dispatches,
 * preemption signals and iteration ends the reference SimEngine issued
 * (sim_engine.cpp call sites). ops: n_ops records of 8 int64 (see
 * paper_2410_01228_b200/replay.py for the encoding); plans: 5 int64 per
 * entry. Iteration outputs (one per DISPATCH in [op_begin, op_end)) go to
 * the caller's arrays. Returns the number of result mismatches against the
 * recorded reference results in *mismatches. */
typedef struct {
  int64_t iterations, mismatches, first_mismatch_op;
  double wall_ms;
  /* host wall ms spent in each replayed op kind (index = op code: 14 dispatch
   * = plan build + enqueue, 16 iteration end = blocked on the device + outputs) */
  double op_ms[20];
} cs_replay_stats;
int cs_replay_run(cs_engine* e, const int64_t* ops, int64_t op_begin, int64_t op_end, const int64_t* plans,
                  double* gpu_ms, double* wall_end_ms, int32_t* dropped_layer, double* drop_latency_us,
                  double* pre_drop_layer_us, int32_t* gemm_trunc_layer, int64_t* h2d_bytes, int64_t* d2h_bytes,
                  cs_replay_stats* st);
/* Times the paged-attention kernels (K1/K2) alone for one plan (pages must be
 * allocated): average ms per launch over reps, algorithmic bytes and flops
 * per launch. */
int cs_bench_attention(cs_engine* e, const cs_batch_entry* entries, int32_t n, int32_t reps, double* ms_per_launch,
                       int64_t* bytes, int64_t* flops);
/* Times one M x N x K projection (Y = X W^T, bf16, seeded synthetic X and W)
 * on the engine's own tcgen05 weight-streaming kernel (K7) and on cuBLASLt,
 * rotating over copies of W that exceed the L2 (each launch reads W from HBM):
 * ms per launch of each, and the max |K7 - cuBLAS| / max |cuBLAS| of the
 * outputs. M <= 256, N % 128 == 0, K % 64 == 0. */
int cs_bench_gemm(cs_engine* e, int32_t M, int32_t N, int32_t K, int32_t reps, double* ms_k7, double* ms_cublas,
                  double* max_abs_diff, double* max_abs_ref);
/* Dry mode: forwards and transfers are bookkeeping only (fast-forward). */
int cs_set_dry(cs_engine* e, int32_t dry);

/* ------------------------------------------------------- test / bench hooks -- */
/* Copies one physical block (all layers of this rank's shard) to host. */
int cs_debug_read_block(cs_engine* e, int32_t block, void* dst, size_t bytes);
int cs_debug_write_block(cs_engine* e, int32_t block, const void* src, size_t bytes);
/* Host pool slot contents (this rank's shard of one page). */
int cs_debug_read_host_slot(cs_engine* e, int32_t slot, void* dst, size_t bytes);
/* Fill every block with a deterministic pattern (seeded). */
int cs_debug_fill_pool(cs_engine* e, uint64_t seed);
/* which: 0 = attention output [T, Hq*d], 1 = residual stream x [T, hidden],
 * 2 = qkv [T, (Hq+2Hkv)*d] (bf16, rank-local, last layer run). */
int cs_debug_read_activation(cs_engine* e, int32_t which, void* dst, size_t bytes);
/* Model weights (bf16 bits) for parity. which: 0 attn_norm, 1 wqkv, 2 wo,
 * 3 mlp_norm, 4 w_gate_up, 5 w_down (per layer); 6 embedding, 7 lm_head,
 * 8 final_norm. *needed receives the byte size. */
int cs_debug_read_weight(cs_engine* e, int32_t layer, int32_t which, void* dst, size_t bytes, size_t* needed);
int cs_sync(cs_engine* e);
/* Host copies of the device hashes (teacher-forced ids, weight init) so a CPU
 * oracle can be checked against them without a GPU. */
int32_t cs_token_id(uint64_t seed, int64_t req, int64_t pos, int32_t vocab);
float cs_hash_uniform(uint64_t seed, uint64_t tensor, uint64_t idx);

#ifdef __cplusplus
}
#endif
#endif /* CONSERVE_B200_H_ */
