// Block pool: the reference's token-granular KV bookkeeping (coserve::
// KvCacheManager, /root/reference/proj/include/coserve/kv_cache.hpp:97-229,
// src/kv_cache.cpp) restated with PHYSICAL placement: every GPU-resident page
// owns one HBM block of the KV pool and every page with host data owns one
// slot of the pinned host pool. Logical decisions (byte-granular capacity,
// eviction order, checkpoint staging, FIFO channel timeline) follow the
// reference exactly so page tables and byte counters stay bit-identical; the
// physical layer adds deterministic block/slot ids, quarantine of freed
// blocks until no in-flight reader remains and the
// known-token -> written-token mapping of checkpoint ranges.
//
// CUDA-free: data movement is delegated to a Mover (engine.cu) so the pool is
// testable on CPU against the compiled reference (tests/cpp/shadow_fuzz.cpp).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/conserve_b200.h"

namespace csb {

// Error types mirror the reference's exceptions; the C-ABI maps them to codes.
struct LogicError : std::logic_error { using std::logic_error::logic_error; };
struct InvalidArg : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct PoolError : std::runtime_error { using std::runtime_error::runtime_error; };

enum class Loc { kGpuOnly, kHostOnly, kBoth, kDiscarded };
const char* loc_name(Loc l);

struct Page {
  int64_t tokens = 0;        // filled known tokens (<= page_tokens)
  int64_t host_tokens = 0;   // known tokens with a completed host copy
  int64_t inflight_to = 0;   // target host_tokens of the in-flight D2H
  bool on_gpu = false;
  bool discarded = false;
  bool recompute_on_evict = false;
  bool h2d_inflight = false;
  bool evict_on_ckpt = false;
  int32_t block = -1;        // physical HBM block while resident / restoring
  int32_t slot = -1;         // host pool slot while it holds host data
  int32_t last_block = -1;   // block held before the last drop (D3 stale reads)
  uint32_t gen = 0;          // bumped when a discarded page is re-materialized

  Loc loc() const {
    if (discarded) return Loc::kDiscarded;
    if (on_gpu) return host_tokens == tokens ? Loc::kBoth : Loc::kGpuOnly;
    return Loc::kHostOnly;
  }
};

// One contiguous token run [t0, t1) of one page: device block <-> host slot.
struct Segment {
  int32_t block;
  int32_t slot;
  int32_t t0;
  int32_t t1;
};

// Data movement backend (engine.cu). Device jobs are FIFO per direction and
// numbered 1, 2, ... in issue order (an "ordinal"); the pool never blocks on
// them. It holds a block or host slot back from reuse only until the last
// device job that touches it has completed (done_prefix), and orders a
// restore after the gathers still writing its slots (`after`).
struct Mover {
  virtual ~Mover() = default;
  // Launch one device job; `after` = ordinal of a job of the OTHER direction
  // that must complete first (0: none). Returns the job's ordinal, or 0 when
  // nothing was launched (dry replay).
  virtual int64_t gather_to_host(const std::vector<Segment>& segs, int64_t after_h2d) = 0;
  virtual int64_t scatter_from_host(const std::vector<Segment>& segs, int64_t after_d2h) = 0;
  // Every job of `dir` with ordinal <= the result has completed on the device.
  virtual int64_t done_prefix(int32_t dir) = 0;
};

struct PoolConfig {
  int64_t page_tokens = 16;
  int64_t kv_bytes_per_token = 0;   // reference accounting unit
  int64_t gpu_capacity = 0;
  int64_t host_capacity = 0;
  double d2h_bw = 1, h2d_bw = 1, gather_us = 0;
  bool incremental = true;
  int64_t n_blocks = 0;             // physical blocks
  int64_t n_slots = 0;              // physical host slots
  int64_t moved_bytes_per_token = 0;  // this rank's bytes per token (shard)
  bool fwd_quarantine = true;         // freed blocks wait for the next forward
};

struct Growth {  // uncommitted allocation segment (kv_cache.hpp:206-212)
  size_t page;
  int64_t prev_tokens;
  bool was_discarded;
  bool was_on_gpu;
};

struct Req {
  bool online = false;
  bool paused = false;
  uint64_t pause_seq = 0;
  std::vector<Page> pages;
  int64_t gpu_tokens = 0;
  std::vector<Growth> growth;
  int64_t w0 = -1, w1 = -1;  // last written KV positions [w0, w1)
};

struct Delta {
  int64_t req;
  size_t page;
  int64_t from, to;  // page-local known-token offsets
  // Known -> written mapping captured at stage time: known
  // position k holds the KV written at k - shift; nothing at or past w1 has
  // been written yet. w1 < 0: identity (no forward noted, bookkeeping only).
  int64_t shift = 0;
  int64_t w1 = -1;
  uint32_t gen = 0;  // page generation at flush: a re-materialized page's old copy is stale
};

struct Job {
  cs_transfer_job info{};
  std::vector<Delta> deltas;                          // D2H payload
  std::vector<std::pair<int64_t, size_t>> restores;   // H2D payload
  int64_t dev = 0;                                    // device ordinal (0: nothing launched)
};

struct ReleaseResult {
  int64_t freed_pages = 0;
  std::vector<std::pair<int64_t, int64_t>> discards;
};

struct DoneResult {
  int64_t freed_pages = 0;
  std::vector<int64_t> became_resident;
};

class BlockPool {
 public:
  BlockPool(const PoolConfig& cfg, Mover* mover);

  // --- reference surface (kv_cache.hpp:100-173) ---
  void register_request(int64_t id, bool online);
  cs_alloc_result allocate(int64_t id, int64_t n_tokens);
  void commit(int64_t id);
  void rollback(int64_t id);
  cs_evict_stats evict_request_gpu(int64_t id, int64_t max_pages);
  cs_evict_stats discard_request(int64_t id);
  ReleaseResult release_offline_pages_on_demand(int64_t needed_pages);
  int64_t releasable_offline_pages_now() const;
  void stage_checkpoint(int64_t id, int64_t from_token, int64_t to_token);
  std::optional<cs_transfer_job> flush_checkpoints(int64_t now);
  cs_resume_cost resume_cost(int64_t id) const;
  bool fully_resident(int64_t id) const;
  bool prefetch_inflight(int64_t id) const;
  std::optional<cs_transfer_job> start_prefetch(int64_t id, int64_t now);
  int64_t recompute_chunk(int64_t id, int64_t desired, int64_t cap) const;
  DoneResult on_transfer_done(int64_t job_id);
  void on_request_paused(int64_t id, uint64_t seq);
  void on_request_active(int64_t id);
  void release_request(int64_t id);
  void audit() const;
  std::string page_table_json(int64_t id) const;

  int64_t gpu_used() const { return gpu_used_; }
  int64_t gpu_free() const { return cfg_.gpu_capacity - gpu_used_; }
  int64_t host_used() const { return host_used_; }
  int64_t page_bytes() const { return cfg_.page_tokens * cfg_.kv_bytes_per_token; }
  int64_t gpu_free_pages() const { return gpu_free() / page_bytes(); }
  int64_t total_d2h() const { return total_d2h_; }
  int64_t total_h2d() const { return total_h2d_; }
  int64_t recompute_tagged() const { return recompute_tagged_; }
  int64_t host_lru_evicted() const { return host_lru_evicted_; }
  int64_t unbacked_reads() const { return unbacked_reads_; }
  // one device block past the pool, never allocated: target of rows the
  // reference dispatched without pages (block_for_read)
  int32_t scratch_block() const { return static_cast<int32_t>(cfg_.n_blocks); }
  bool transfers_inflight() const { return !jobs_.empty(); }
  // Device ordinal of a reference job (dir, ordinal); ordinal 0 when it moved
  // nothing on the device. Known for every job id issued so far.
  std::pair<int32_t, int64_t> job_device(int64_t job_id) const;
  // Device ordinal of the last restore that wrote block b (the forward that
  // reads b must be ordered after it).
  int64_t block_h2d(int32_t b) const { return blk_h2d_[static_cast<size_t>(b)]; }
  int64_t fixup_gathers() const { return fixups_; }
  int64_t request_gpu_pages(int64_t id) const;
  int64_t covered_tokens(int64_t id) const;
  int64_t pending_append_tokens(int64_t id) const;

  // --- physical layer (B200) ---
  void note_written(int64_t id, int64_t w0, int64_t w1);
  // Forward bookkeeping: a forward was launched / completed (quarantine).
  void on_forward_launched() { ++fwd_launched_; }
  void on_forward_completed();
  const Req* find(int64_t id) const;
  Req* find_mut(int64_t id);
  // Block that attention should read for page idx of request id; counts
  // stale (non-resident) reads. -1 if the page never had a block.
  int32_t block_for_read(int64_t id, size_t page_idx);
  // block_for_read of pages [0, n) appended to `out` with ONE request lookup
  // (the plan build's hot loop: ~10K pages per decode step); also raises
  // `wait_h2d` to the last restore writing any of those blocks
  void blocks_for_read(int64_t id, size_t n, std::vector<int32_t>& out, int64_t& wait_h2d);
  int64_t n_blocks() const { return cfg_.n_blocks; }
  int64_t free_blocks() const { return static_cast<int64_t>(free_blocks_.size()); }
  int64_t quarantined_blocks() const { return static_cast<int64_t>(block_q_.size()); }
  int64_t n_slots() const { return cfg_.n_slots; }
  int64_t free_slots() const { return static_cast<int64_t>(free_slots_.size()); }
  int64_t moved_d2h() const { return moved_d2h_; }
  int64_t moved_h2d() const { return moved_h2d_; }
  int64_t nonresident_reads() const { return nonresident_reads_; }
  const PoolConfig& config() const { return cfg_; }

 private:
  struct Lane {  // TransferChannel (kv_cache.hpp:57-64, kv_cache.cpp:23-36)
    int32_t dir = CS_D2H;
    double bw = 1, gather_us = 0;
    int64_t busy_until = 0;
    cs_transfer_job enqueue(int64_t id, int64_t bytes, int64_t now);
  };
  struct Quarantined {
    int32_t id;
    uint64_t fwd_tag;  // forwards launched at retire time
    int64_t d2h;       // last device gather touching it (0: none)
    int64_t h2d;       // last device restore touching it
  };

  Req& req(int64_t id);
  const Req& req(int64_t id) const;
  void drop_gpu_page(Req& r, Page& p);
  int64_t evict_host_bytes(int64_t needed);
  int32_t take_block();
  int32_t take_slot();
  void retire_block(Page& p);
  void retire_slot(Page& p);
  void reclaim();
  bool dev_done(int32_t dir, int64_t ord);
  int64_t launch_gather(const std::vector<Segment>& segs);
  int64_t launch_scatter(const std::vector<Segment>& segs);

  PoolConfig cfg_;
  Mover* mover_;
  std::map<int64_t, Req> reqs_;
  Lane d2h_, h2d_;
  std::vector<Delta> staged_;
  std::map<int64_t, Job> jobs_;
  int64_t next_job_ = 1;
  int64_t gpu_used_ = 0, host_used_ = 0;
  int64_t total_d2h_ = 0, total_h2d_ = 0, recompute_tagged_ = 0;
  int64_t host_lru_evicted_ = 0, unbacked_reads_ = 0;
  uint64_t host_stamp_ = 0;
  std::map<uint64_t, std::pair<int64_t, size_t>> host_lru_;  // stamp -> (req, page)

  // physical state
  std::vector<int32_t> free_blocks_, free_slots_;  // LIFO stacks
  std::vector<Quarantined> block_q_, slot_q_;
  uint64_t fwd_launched_ = 0, fwd_completed_ = 0;
  // last device job per block / host slot: gathers read blocks and write
  // slots, restores read slots and write blocks (ordinals per direction)
  std::vector<int64_t> blk_d2h_, blk_h2d_, slot_d2h_, slot_h2d_;
  int64_t dev_done_[2] = {0, 0};                        // cached done_prefix
  std::map<int64_t, std::pair<int32_t, int64_t>> job_dev_;  // job id -> (dir, ordinal)
  int64_t moved_d2h_ = 0, moved_h2d_ = 0, nonresident_reads_ = 0, fixups_ = 0;
};

}  // namespace csb
