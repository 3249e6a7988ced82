// Block pool: see block_pool.h. Every logical rule cites the reference
// function it restates (/root/reference/proj/src/kv_cache.cpp).
#include "block_pool.h"

#include <algorithm>
#include <cmath>
#include <limits>
#include <sstream>

namespace csb {

const char* loc_name(Loc l) {
  switch (l) {
    case Loc::kGpuOnly: return "gpu";
    case Loc::kHostOnly: return "host";
    case Loc::kBoth: return "both";
    case Loc::kDiscarded: return "discarded";
  }
  return "?";
}

// TransferChannel::enqueue (kv_cache.cpp:23-36): FIFO lane, integer-us done.
cs_transfer_job BlockPool::Lane::enqueue(int64_t id, int64_t bytes, int64_t now) {
  cs_transfer_job j{};
  j.id = id;
  j.direction = dir;
  j.bytes = bytes;
  j.enqueue_time = now;
  j.start_time = std::max(now, busy_until);
  j.transfer_us = static_cast<double>(bytes) / bw * 1e6;
  j.gather_us = gather_us;
  j.done_time = j.start_time + static_cast<int64_t>(std::llround(j.transfer_us + j.gather_us));
  busy_until = j.done_time;
  return j;
}

BlockPool::BlockPool(const PoolConfig& cfg, Mover* mover) : cfg_(cfg), mover_(mover) {
  d2h_.dir = CS_D2H;
  d2h_.bw = cfg.d2h_bw;
  d2h_.gather_us = cfg.gather_us;
  h2d_.dir = CS_H2D;
  h2d_.bw = cfg.h2d_bw;
  h2d_.gather_us = cfg.gather_us;
  free_blocks_.reserve(static_cast<size_t>(cfg.n_blocks));
  for (int64_t b = cfg.n_blocks; b-- > 0;) free_blocks_.push_back(static_cast<int32_t>(b));
  free_slots_.reserve(static_cast<size_t>(cfg.n_slots));
  for (int64_t s = cfg.n_slots; s-- > 0;) free_slots_.push_back(static_cast<int32_t>(s));
  // one entry past the pool: the scratch block (scratch_block()) is returned
  // by block_for_read and never copied, so its ordinals stay 0
  blk_d2h_.assign(static_cast<size_t>(cfg.n_blocks) + 1, 0);
  blk_h2d_.assign(static_cast<size_t>(cfg.n_blocks) + 1, 0);
  slot_d2h_.assign(static_cast<size_t>(cfg.n_slots), 0);
  slot_h2d_.assign(static_cast<size_t>(cfg.n_slots), 0);
}

Req& BlockPool::req(int64_t id) {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) throw LogicError("unknown request id in kv manager");
  return it->second;
}
const Req& BlockPool::req(int64_t id) const {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) throw LogicError("unknown request id in kv manager");
  return it->second;
}
const Req* BlockPool::find(int64_t id) const {
  auto it = reqs_.find(id);
  return it == reqs_.end() ? nullptr : &it->second;
}
Req* BlockPool::find_mut(int64_t id) {
  auto it = reqs_.find(id);
  return it == reqs_.end() ? nullptr : &it->second;
}

// ------------------------------------------------------------ physical ----
int32_t BlockPool::take_block() {
  if (free_blocks_.empty()) reclaim();
  if (free_blocks_.empty()) {
    throw PoolError("physical KV block pool exhausted (byte accounting fit; raise extra_blocks)");
  }
  int32_t b = free_blocks_.back();
  free_blocks_.pop_back();
  return b;
}

int32_t BlockPool::take_slot() {
  if (free_slots_.empty()) reclaim();
  if (free_slots_.empty()) {
    throw PoolError("host slot pool exhausted (byte accounting fit; raise extra_host_slots)");
  }
  int32_t s = free_slots_.back();
  free_slots_.pop_back();
  return s;
}

void BlockPool::retire_block(Page& p) {
  if (p.block < 0) return;
  const size_t b = static_cast<size_t>(p.block);
  block_q_.push_back({p.block, fwd_launched_, blk_d2h_[b], blk_h2d_[b]});
  p.last_block = p.block;
  p.block = -1;
}

void BlockPool::retire_slot(Page& p) {
  if (p.slot < 0) return;
  const size_t s = static_cast<size_t>(p.slot);
  slot_q_.push_back({p.slot, 0, slot_d2h_[s], slot_h2d_[s]});
  p.slot = -1;
}

// True once device job `ord` of `dir` has completed (no device: always).
bool BlockPool::dev_done(int32_t dir, int64_t ord) {
  if (ord <= dev_done_[dir]) return true;
  if (mover_ == nullptr) return true;
  dev_done_[dir] = mover_->done_prefix(dir);
  return ord <= dev_done_[dir];
}

// One device gather / restore; records it as the last job touching each
// block and slot of its segments. A gather first waits for restores still
// writing its blocks; a restore for gathers still writing its slots (a page
// whose last delta is still in flight can be evicted and restored at once:
// ADVICE r1, restore ordering).
int64_t BlockPool::launch_gather(const std::vector<Segment>& segs) {
  if (mover_ == nullptr || segs.empty()) return 0;
  int64_t after = 0;
  for (const Segment& g : segs) after = std::max(after, blk_h2d_[static_cast<size_t>(g.block)]);
  if (dev_done(CS_H2D, after)) after = 0;
  const int64_t ord = mover_->gather_to_host(segs, after);
  if (ord > 0) {
    for (const Segment& g : segs) {
      blk_d2h_[static_cast<size_t>(g.block)] = ord;
      slot_d2h_[static_cast<size_t>(g.slot)] = ord;
    }
  }
  return ord;
}

int64_t BlockPool::launch_scatter(const std::vector<Segment>& segs) {
  if (mover_ == nullptr || segs.empty()) return 0;
  int64_t after = 0;
  for (const Segment& g : segs) after = std::max(after, slot_d2h_[static_cast<size_t>(g.slot)]);
  if (dev_done(CS_D2H, after)) after = 0;
  const int64_t ord = mover_->scatter_from_host(segs, after);
  if (ord > 0) {
    for (const Segment& g : segs) {
      blk_h2d_[static_cast<size_t>(g.block)] = ord;
      slot_h2d_[static_cast<size_t>(g.slot)] = ord;
    }
  }
  return ord;
}

// A freed block is reusable once (a) the forward dispatched after its release
// has completed -- so a plan that still reads it (reference defect D3) reads
// stale-but-intact KV -- and (b) the last device gather reading it and the
// last restore writing it have completed. Slots likewise wait only for the
// device jobs that touched them (no hold behind unrelated copies).
void BlockPool::reclaim() {
  auto keep_b = std::stable_partition(block_q_.begin(), block_q_.end(), [&](const Quarantined& q) {
    return !((!cfg_.fwd_quarantine || fwd_completed_ >= q.fwd_tag + 1) && dev_done(CS_D2H, q.d2h) &&
             dev_done(CS_H2D, q.h2d));
  });
  for (auto it = keep_b; it != block_q_.end(); ++it) free_blocks_.push_back(it->id);
  block_q_.erase(keep_b, block_q_.end());
  auto keep_s = std::stable_partition(slot_q_.begin(), slot_q_.end(), [&](const Quarantined& q) {
    return !(dev_done(CS_D2H, q.d2h) && dev_done(CS_H2D, q.h2d));
  });
  for (auto it = keep_s; it != slot_q_.end(); ++it) free_slots_.push_back(it->id);
  slot_q_.erase(keep_s, slot_q_.end());
}

std::pair<int32_t, int64_t> BlockPool::job_device(int64_t job_id) const {
  auto f = job_dev_.find(job_id);
  if (f == job_dev_.end()) {
    if (job_id >= 1 && job_id < next_job_) return {CS_D2H, 0};
    throw LogicError("unknown transfer job");
  }
  return f->second;
}

void BlockPool::on_forward_completed() {
  ++fwd_completed_;
  reclaim();
}

void BlockPool::note_written(int64_t id, int64_t w0, int64_t w1) {
  Req& r = req(id);
  r.w0 = w0;
  r.w1 = w1;
}

int32_t BlockPool::block_for_read(int64_t id, size_t page_idx) {
  Req& r = req(id);
  if (page_idx >= r.pages.size()) {
    // The reference dispatched an entry over positions it holds no pages for
    // (host-limited regime: a prefill continuation of a request whose context
    // release_offline_pages_on_demand discarded in the same build, DESIGN.md
    // D5). Those rows read and write the scratch block, never a live one.
    ++unbacked_reads_;
    return scratch_block();
  }
  Page& p = r.pages[page_idx];
  if (p.on_gpu && !p.discarded && p.block >= 0) return p.block;
  // The reference dispatched a plan whose context is not GPU-resident (D3).
  ++nonresident_reads_;
  if (p.block >= 0) return p.block;  // restore in flight: bytes may be partial
  if (p.last_block >= 0) {
    for (const Quarantined& q : block_q_) {
      if (q.id == p.last_block) return p.last_block;  // still intact
    }
  }
  throw LogicError("attention reads a page whose block was reallocated");
}

void BlockPool::blocks_for_read(int64_t id, size_t n, std::vector<int32_t>& out, int64_t& wait_h2d) {
  Req& r = req(id);
  for (size_t pg = 0; pg < n; ++pg) {
    int32_t b;
    if (pg < r.pages.size()) {
      const Page& p = r.pages[pg];
      b = (p.on_gpu && !p.discarded && p.block >= 0) ? p.block : block_for_read(id, pg);
    } else {
      b = block_for_read(id, pg);
    }
    out.push_back(b);
    wait_h2d = std::max(wait_h2d, blk_h2d_[static_cast<size_t>(b)]);
  }
}

// -------------------------------------------------------------- logical ----
void BlockPool::register_request(int64_t id, bool online) {
  Req r;
  r.online = online;
  reqs_.emplace(id, std::move(r));  // emplace: an existing id is left untouched
}

// KvCacheManager::allocate (kv_cache.cpp:70-142).
cs_alloc_result BlockPool::allocate(int64_t id, int64_t n_tokens) {
  if (n_tokens < 1) throw InvalidArg("allocate requires n >= 1");
  Req& r = req(id);
  const int64_t bpt = cfg_.kv_bytes_per_token;
  auto shortfall = [&](int64_t need) {
    const int64_t short_bytes = need - gpu_free();
    return cs_alloc_result{0, (short_bytes + page_bytes() - 1) / page_bytes()};
  };

  size_t first_disc = r.pages.size();
  for (size_t i = 0; i < r.pages.size(); ++i) {
    if (r.pages[i].discarded) {
      first_disc = i;
      break;
    }
  }
  if (first_disc < r.pages.size()) {
    // Recompute: re-materialize discarded pages head-first, whole pages.
    int64_t left = n_tokens, need = 0;
    std::vector<size_t> targets;
    for (size_t i = first_disc; i < r.pages.size() && left > 0; ++i) {
      if (!r.pages[i].discarded) continue;
      targets.push_back(i);
      left -= r.pages[i].tokens;
      need += r.pages[i].tokens * bpt;
    }
    if (need > gpu_free()) return shortfall(need);
    for (size_t i : targets) {
      Page& p = r.pages[i];
      r.growth.push_back({i, p.tokens, true, false});
      p.discarded = false;
      p.on_gpu = true;
      p.host_tokens = 0;
      p.recompute_on_evict = false;
      ++p.gen;  // any D2H of the old contents still in flight is stale now
      p.block = take_block();
      gpu_used_ += p.tokens * bpt;
      r.gpu_tokens += p.tokens;
    }
    return {1, 0};
  }

  const int64_t need = n_tokens * bpt;
  if (need > gpu_free()) return shortfall(need);
  int64_t left = n_tokens;
  if (!r.pages.empty()) {
    Page& tail = r.pages.back();
    if (tail.on_gpu && tail.tokens < cfg_.page_tokens) {
      const int64_t add = std::min(left, cfg_.page_tokens - tail.tokens);
      r.growth.push_back({r.pages.size() - 1, tail.tokens, false, true});
      tail.tokens += add;
      gpu_used_ += add * bpt;
      r.gpu_tokens += add;
      left -= add;
    }
  }
  while (left > 0) {
    const int64_t add = std::min(left, cfg_.page_tokens);
    Page p;
    p.tokens = add;
    p.on_gpu = true;
    p.block = take_block();
    r.growth.push_back({r.pages.size(), 0, false, false});
    r.pages.push_back(p);
    gpu_used_ += add * bpt;
    r.gpu_tokens += add;
    left -= add;
  }
  return {1, 0};
}

void BlockPool::commit(int64_t id) { req(id).growth.clear(); }

// KvCacheManager::rollback_allocations (kv_cache.cpp:146-174).
void BlockPool::rollback(int64_t id) {
  Req& r = req(id);
  const int64_t bpt = cfg_.kv_bytes_per_token;
  for (auto it = r.growth.rbegin(); it != r.growth.rend(); ++it) {
    const bool fresh = it->prev_tokens == 0 && !it->was_discarded && !it->was_on_gpu;
    if (fresh && it->page == r.pages.size() - 1) {
      Page& p = r.pages.back();
      gpu_used_ -= p.tokens * bpt;
      r.gpu_tokens -= p.tokens;
      retire_block(p);
      retire_slot(p);
      r.pages.pop_back();
      continue;
    }
    Page& p = r.pages[it->page];
    if (it->was_discarded) {
      gpu_used_ -= p.tokens * bpt;
      r.gpu_tokens -= p.tokens;
      p.discarded = true;
      p.on_gpu = false;
      p.host_tokens = 0;
      retire_block(p);
      retire_slot(p);
    } else {
      const int64_t delta = p.tokens - it->prev_tokens;
      gpu_used_ -= delta * bpt;
      r.gpu_tokens -= delta;
      p.tokens = it->prev_tokens;
    }
  }
  r.growth.clear();
}

void BlockPool::drop_gpu_page(Req& r, Page& p) {
  gpu_used_ -= p.tokens * cfg_.kv_bytes_per_token;
  r.gpu_tokens -= p.tokens;
  p.on_gpu = false;
  retire_block(p);
}

// KvCacheManager::evict_request_gpu (kv_cache.cpp:183-232).
cs_evict_stats BlockPool::evict_request_gpu(int64_t id, int64_t max_pages) {
  Req& r = req(id);
  if (r.online) throw LogicError("online pages are not evictable");
  cs_evict_stats st{0, 0, 0};
  const bool whole = max_pages < 0;
  int64_t quota = whole ? std::numeric_limits<int64_t>::max() : max_pages;

  // Pass 1: pages with a complete host copy drop for free, newest first.
  for (auto it = r.pages.rbegin(); it != r.pages.rend() && quota > 0; ++it) {
    Page& p = *it;
    if (!p.on_gpu || p.discarded) continue;
    if (p.loc() == Loc::kBoth) {
      drop_gpu_page(r, p);
      ++st.freed_pages;
      --quota;
    }
  }
  if (!whole && quota <= 0) return st;

  // Pass 2: mid-checkpoint pages drop when the D2H lands; the rest discard.
  for (auto it = r.pages.rbegin(); it != r.pages.rend() && quota > 0; ++it) {
    Page& p = *it;
    if (!p.on_gpu || p.discarded || p.loc() == Loc::kBoth) continue;
    if (p.inflight_to == p.tokens) {
      if (!p.evict_on_ckpt) {
        p.evict_on_ckpt = true;
        ++st.pending_pages;
      }
      continue;
    }
    st.discarded_tokens += p.tokens;
    if (p.host_tokens > 0) {
      host_used_ -= p.host_tokens * cfg_.kv_bytes_per_token;
      p.host_tokens = 0;
    }
    drop_gpu_page(r, p);
    retire_slot(p);
    p.discarded = true;
    p.recompute_on_evict = false;
    ++st.freed_pages;
    --quota;
  }
  return st;
}

// KvCacheManager::discard_request (kv_cache.cpp:234-256).
cs_evict_stats BlockPool::discard_request(int64_t id) {
  Req& r = req(id);
  if (r.online) throw LogicError("online pages are not evictable");
  cs_evict_stats st{0, 0, 0};
  for (Page& p : r.pages) {
    if (p.discarded) continue;
    if (p.on_gpu) {
      drop_gpu_page(r, p);
      ++st.freed_pages;
    }
    if (p.host_tokens > 0) {
      host_used_ -= p.host_tokens * cfg_.kv_bytes_per_token;
      p.host_tokens = 0;
    }
    retire_slot(p);
    p.discarded = true;
    p.recompute_on_evict = false;
    p.evict_on_ckpt = false;
    st.discarded_tokens += p.tokens;
  }
  return st;
}

// KvCacheManager::release_offline_pages_on_demand (kv_cache.cpp:258-287).
ReleaseResult BlockPool::release_offline_pages_on_demand(int64_t needed) {
  if (needed <= 0) throw InvalidArg("needed_pages must be > 0");
  std::vector<std::pair<uint64_t, int64_t>> victims;
  for (const auto& [id, r] : reqs_) {
    if (!r.online && r.paused && !prefetch_inflight(id)) victims.emplace_back(r.pause_seq, id);
  }
  std::sort(victims.begin(), victims.end(),
            [](const auto& a, const auto& b) { return a.first > b.first; });
  ReleaseResult out;
  for (const auto& v : victims) {
    if (out.freed_pages >= needed) break;
    const cs_evict_stats ev = evict_request_gpu(v.second, needed - out.freed_pages);
    out.freed_pages += ev.freed_pages;
    if (ev.discarded_tokens > 0) out.discards.emplace_back(v.second, ev.discarded_tokens);
  }
  if (out.freed_pages < needed) {
    for (const auto& v : victims) evict_request_gpu(v.second, needed - out.freed_pages);
  }
  return out;
}

// KvCacheManager::releasable_offline_pages_now (kv_cache.cpp:289-306).
int64_t BlockPool::releasable_offline_pages_now() const {
  int64_t n = 0;
  for (const auto& [id, r] : reqs_) {
    if (r.online || !r.paused || prefetch_inflight(id)) continue;
    for (const Page& p : r.pages) {
      if (!p.on_gpu || p.discarded) continue;
      if (p.loc() == Loc::kBoth) {
        ++n;
      } else if (!cfg_.incremental || (p.recompute_on_evict && p.inflight_to != p.tokens)) {
        ++n;
      }
    }
  }
  return n;
}

// KvCacheManager::stage_checkpoint (kv_cache.cpp:308-324).
void BlockPool::stage_checkpoint(int64_t id, int64_t from_token, int64_t to_token) {
  if (!cfg_.incremental) return;
  if (to_token <= from_token) return;
  Req& r = req(id);
  const int64_t pt = cfg_.page_tokens;
  for (int64_t pi = from_token / pt; pi <= (to_token - 1) / pt; ++pi) {
    // The reference indexes r.pages[page_idx] unchecked here (kv_cache.cpp:
    // 315, undefined behaviour past the vector) when it stages the range of
    // an entry it dispatched without pages (D5); there is nothing to copy.
    if (pi >= static_cast<int64_t>(r.pages.size())) break;
    Page& p = r.pages[static_cast<size_t>(pi)];
    if (p.discarded || !p.on_gpu) continue;
    const int64_t target = std::min(p.tokens, to_token - pi * pt);
    const int64_t from = std::max(p.host_tokens, p.inflight_to);
    if (target <= from) continue;
    Delta d{id, static_cast<size_t>(pi), from, target};
    // The range starts at the request's known length before the iteration;
    // the forward wrote [w0, w1). A decode step writes position C-1 while the
    // reference stages known slot C (shift 1); a prefill chunk writes its own
    // positions (shift 0) and the final chunk's extra first-token slot is past
    // w1. Ranges not produced by the last forward map identically.
    if (r.w0 >= 0 && (from_token - r.w0 == 0 || from_token - r.w0 == 1)) {
      d.shift = from_token - r.w0;
      d.w1 = r.w1;
    }
    staged_.push_back(d);
  }
}

// KvCacheManager::evict_host_bytes (kv_cache.cpp:326-362): host LRU.
int64_t BlockPool::evict_host_bytes(int64_t needed) {
  const int64_t bpt = cfg_.kv_bytes_per_token;
  int64_t freed = 0;
  auto it = host_lru_.begin();
  while (it != host_lru_.end() && freed < needed) {
    const auto [rid, pi] = it->second;
    auto rit = reqs_.find(rid);
    if (rit == reqs_.end() || rit->second.online) {
      it = host_lru_.erase(it);
      continue;
    }
    Req& r = rit->second;
    if (pi >= r.pages.size()) {
      it = host_lru_.erase(it);
      continue;
    }
    Page& p = r.pages[pi];
    if (p.host_tokens == 0 || p.inflight_to > p.host_tokens || p.h2d_inflight) {
      it = host_lru_.erase(it);
      continue;
    }
    freed += p.host_tokens * bpt;
    ++host_lru_evicted_;
    host_used_ -= p.host_tokens * bpt;
    p.host_tokens = 0;
    retire_slot(p);
    if (p.on_gpu) {
      p.recompute_on_evict = true;
    } else {
      p.discarded = true;
      recompute_tagged_ += p.tokens;
    }
    it = host_lru_.erase(it);
  }
  return freed;
}

// KvCacheManager::flush_checkpoints (kv_cache.cpp:364-400), plus the gather:
// accepted known-token deltas are mapped onto written positions and moved
// device block -> host slot by one kernel on the D2H stream.
std::optional<cs_transfer_job> BlockPool::flush_checkpoints(int64_t now) {
  if (staged_.empty()) return std::nullopt;
  const int64_t bpt = cfg_.kv_bytes_per_token;
  const int64_t pt = cfg_.page_tokens;
  std::vector<Delta> accepted;
  int64_t bytes = 0;
  for (const Delta& d : staged_) {
    auto rit = reqs_.find(d.req);
    if (rit == reqs_.end()) continue;
    Page& p = rit->second.pages[d.page];
    if (p.discarded || !p.on_gpu) continue;
    const int64_t db = (d.to - d.from) * bpt;
    if (host_used_ + db > cfg_.host_capacity) evict_host_bytes(host_used_ + db - cfg_.host_capacity);
    if (host_used_ + db > cfg_.host_capacity) {
      p.recompute_on_evict = true;  // host pool exhausted: recompute fallback
      recompute_tagged_ += d.to - d.from;
      continue;
    }
    host_used_ += db;
    p.inflight_to = d.to;
    if (p.slot < 0) p.slot = take_slot();
    bytes += db;
    accepted.push_back(d);
    accepted.back().gen = p.gen;
  }
  staged_.clear();
  if (accepted.empty()) return std::nullopt;

  // Physical payload: known positions [page*pt + from, page*pt + to) hold
  // written positions shifted by s in {0,1}; truncate at the frontier w1.
  std::vector<Segment> segs;
  int64_t moved = 0;
  for (const Delta& d : accepted) {
    Req& r = reqs_.at(d.req);
    int64_t a = static_cast<int64_t>(d.page) * pt + d.from;
    int64_t b = static_cast<int64_t>(d.page) * pt + d.to;
    if (d.w1 >= 0) {
      a -= d.shift;
      b = std::min(b - d.shift, d.w1);
    }
    for (int64_t pos = std::max<int64_t>(a, 0); pos < b;) {
      const size_t q = static_cast<size_t>(pos / pt);
      const int64_t end = std::min(b, static_cast<int64_t>(q + 1) * pt);
      if (q < r.pages.size()) {
        Page& pq = r.pages[q];
        if (pq.on_gpu && pq.block >= 0 && pq.slot >= 0) {
          segs.push_back({pq.block, pq.slot, static_cast<int32_t>(pos - static_cast<int64_t>(q) * pt),
                          static_cast<int32_t>(end - static_cast<int64_t>(q) * pt)});
          moved += (end - pos) * cfg_.moved_bytes_per_token;
        }
      }
      pos = end;
    }
  }

  cs_transfer_job info = d2h_.enqueue(next_job_++, bytes, now);
  info.moved_bytes = moved;
  total_d2h_ += bytes;
  moved_d2h_ += moved;
  Job job;
  job.info = info;
  job.deltas = std::move(accepted);
  job.dev = launch_gather(segs);
  job_dev_[info.id] = {CS_D2H, job.dev};
  jobs_.emplace(info.id, std::move(job));
  return info;
}

// KvCacheManager::resume_cost (kv_cache.cpp:402-415).
cs_resume_cost BlockPool::resume_cost(int64_t id) const {
  const Req& r = req(id);
  cs_resume_cost c{0, 0, 0};
  for (const Page& p : r.pages) {
    if (p.discarded) {
      c.discarded_tokens += p.tokens;
    } else if (!p.on_gpu) {
      ++c.host_only_pages;
      c.host_only_bytes += p.tokens * cfg_.kv_bytes_per_token;
    }
  }
  return c;
}

bool BlockPool::fully_resident(int64_t id) const {
  const Req& r = req(id);
  return std::all_of(r.pages.begin(), r.pages.end(),
                     [](const Page& p) { return p.on_gpu && !p.discarded; });
}

bool BlockPool::prefetch_inflight(int64_t id) const {
  const Req& r = req(id);
  return std::any_of(r.pages.begin(), r.pages.end(), [](const Page& p) { return p.h2d_inflight; });
}

// KvCacheManager::start_prefetch (kv_cache.cpp:428-455), plus the restore:
// every HostOnly page gets a fresh block and one kernel scatters the host
// slots into them on the H2D stream.
std::optional<cs_transfer_job> BlockPool::start_prefetch(int64_t id, int64_t now) {
  Req& r = req(id);
  const int64_t bpt = cfg_.kv_bytes_per_token;
  std::vector<size_t> targets;
  int64_t bytes = 0;
  for (size_t i = 0; i < r.pages.size(); ++i) {
    const Page& p = r.pages[i];
    if (p.discarded || p.on_gpu || p.h2d_inflight) continue;
    targets.push_back(i);
    bytes += p.tokens * bpt;
  }
  if (targets.empty()) return std::nullopt;
  if (bytes > gpu_free()) return std::nullopt;  // deferred

  gpu_used_ += bytes;
  std::vector<Segment> segs;
  int64_t moved = 0;
  for (size_t i : targets) {
    Page& p = r.pages[i];
    p.h2d_inflight = true;
    p.block = take_block();
    if (p.slot < 0) throw LogicError("host-only page has no host slot");
    segs.push_back({p.block, p.slot, 0, static_cast<int32_t>(p.tokens)});
    moved += p.tokens * cfg_.moved_bytes_per_token;
  }
  cs_transfer_job info = h2d_.enqueue(next_job_++, bytes, now);
  info.moved_bytes = moved;
  total_h2d_ += bytes;
  moved_h2d_ += moved;
  Job job;
  job.info = info;
  for (size_t i : targets) job.restores.emplace_back(id, i);
  job.dev = launch_scatter(segs);
  job_dev_[info.id] = {CS_H2D, job.dev};
  jobs_.emplace(info.id, std::move(job));
  return info;
}

// KvCacheManager::recompute_chunk (kv_cache.cpp:457-469).
int64_t BlockPool::recompute_chunk(int64_t id, int64_t desired, int64_t cap) const {
  if (desired <= 0 || cap <= 0) return 0;
  const Req& r = req(id);
  int64_t tokens = 0;
  for (const Page& p : r.pages) {
    if (!p.discarded) continue;
    if (tokens >= desired) break;
    if (tokens + p.tokens > cap) break;
    tokens += p.tokens;
  }
  return tokens;
}

// KvCacheManager::on_transfer_done (kv_cache.cpp:471-520). Bookkeeping only:
// it does not wait for the device (SURVEY.md 8b "Completion"; cs_job_poll /
// cs_job_wait report the real copy). Blocks and slots stay quarantined until
// the device jobs touching them complete, a restore waits for the gathers
// writing its slots, and the forward waits for the restores of the blocks it
// reads (BlockPool::block_h2d), so logical completion may run ahead of the
// bytes without any reader seeing them early.
DoneResult BlockPool::on_transfer_done(int64_t job_id) {
  auto jit = jobs_.find(job_id);
  if (jit == jobs_.end()) throw LogicError("unknown transfer job");
  Job& job = jit->second;
  const int64_t bpt = cfg_.kv_bytes_per_token;
  DoneResult out;

  std::vector<Segment> fixup;
  for (const Delta& d : job.deltas) {
    auto rit = reqs_.find(d.req);
    const int64_t db = (d.to - d.from) * bpt;
    if (rit == reqs_.end()) {
      host_used_ -= db;  // owner finished mid-flight
      continue;
    }
    Req& r = rit->second;
    Page& p = r.pages[d.page];
    if (p.discarded) {
      host_used_ -= db;
      continue;
    }
    p.host_tokens = d.to;
    if (p.inflight_to == d.to) p.inflight_to = 0;
    if (p.gen != d.gen) {
      // The page was discarded and re-materialized (recompute) while this
      // copy was in flight: the reference counts [0, d.to) as checkpointed,
      // but the copy landed in a slot the page no longer owns. Re-gather the
      // recomputed positions into the page's current slot (device-only; the
      // reference byte counters are unchanged). ADVICE r1 (high).
      if (p.slot < 0) p.slot = take_slot();
      if (p.block >= 0) fixup.push_back({p.block, p.slot, 0, static_cast<int32_t>(d.to)});
      ++fixups_;
    }
    host_lru_.emplace(++host_stamp_, std::make_pair(d.req, d.page));
    if (p.evict_on_ckpt && p.loc() == Loc::kBoth) {
      drop_gpu_page(r, p);
      p.evict_on_ckpt = false;
      ++out.freed_pages;
    }
  }
  for (const auto& [rid, pi] : job.restores) {
    auto rit = reqs_.find(rid);
    if (rit == reqs_.end()) continue;
    Req& r = rit->second;
    Page& p = r.pages[pi];
    p.h2d_inflight = false;
    p.on_gpu = true;  // bytes were reserved at enqueue
    r.gpu_tokens += p.tokens;
  }
  if (!job.restores.empty()) {
    const int64_t rid = job.restores.front().first;
    if (reqs_.count(rid) && fully_resident(rid)) out.became_resident.push_back(rid);
  }
  jobs_.erase(jit);
  if (!fixup.empty()) launch_gather(fixup);
  reclaim();
  return out;
}

void BlockPool::on_request_paused(int64_t id, uint64_t seq) {
  Req& r = req(id);
  r.paused = true;
  r.pause_seq = seq;
}

void BlockPool::on_request_active(int64_t id) { req(id).paused = false; }

// KvCacheManager::release_request (kv_cache.cpp:530-540).
void BlockPool::release_request(int64_t id) {
  Req& r = req(id);
  const int64_t bpt = cfg_.kv_bytes_per_token;
  for (Page& p : r.pages) {
    if (p.on_gpu) gpu_used_ -= p.tokens * bpt;
    host_used_ -= p.host_tokens * bpt;
    retire_block(p);
    retire_slot(p);
  }
  reqs_.erase(id);
}

int64_t BlockPool::request_gpu_pages(int64_t id) const {
  const Req& r = req(id);
  return std::count_if(r.pages.begin(), r.pages.end(), [](const Page& p) { return p.on_gpu; });
}

int64_t BlockPool::covered_tokens(int64_t id) const {
  int64_t n = 0;
  for (const Page& p : req(id).pages) n += p.tokens;
  return n;
}

int64_t BlockPool::pending_append_tokens(int64_t id) const {
  const Req& r = req(id);
  int64_t n = 0;
  for (const Growth& g : r.growth) {
    if (g.was_discarded) continue;
    n += r.pages[g.page].tokens - g.prev_tokens;
  }
  return n;
}

// KvCacheManager::audit (kv_cache.cpp:566-620) plus physical invariants.
void BlockPool::audit() const {
  const int64_t bpt = cfg_.kv_bytes_per_token;
  int64_t gpu_recount = 0, host_recount = 0;
  std::vector<uint8_t> block_seen(static_cast<size_t>(cfg_.n_blocks), 0);
  std::vector<uint8_t> slot_seen(static_cast<size_t>(cfg_.n_slots), 0);
  auto claim = [](std::vector<uint8_t>& seen, int32_t id, const char* what) {
    if (id < 0 || static_cast<size_t>(id) >= seen.size()) throw LogicError(std::string(what) + " id out of range");
    if (seen[static_cast<size_t>(id)]++) throw LogicError(std::string(what) + " owned twice");
  };
  for (const auto& [id, r] : reqs_) {
    int64_t gpu_tokens = 0;
    for (size_t i = 0; i < r.pages.size(); ++i) {
      const Page& p = r.pages[i];
      if (p.tokens < 1 || p.tokens > cfg_.page_tokens) throw LogicError("page token count out of range");
      if (i + 1 < r.pages.size() && p.tokens != cfg_.page_tokens) throw LogicError("interior page is partial");
      if (p.host_tokens > p.tokens) throw LogicError("host copy exceeds page fill");
      if (p.discarded && (p.on_gpu || p.host_tokens > 0)) throw LogicError("discarded page still holds data");
      if (p.on_gpu) {
        gpu_recount += p.tokens * bpt;
        gpu_tokens += p.tokens;
      } else if (p.h2d_inflight) {
        gpu_recount += p.tokens * bpt;
      } else if (!p.discarded && p.host_tokens != p.tokens) {
        throw LogicError("non-resident page lacks full host copy");
      }
      host_recount += p.host_tokens * bpt;
      // physical: resident or restoring pages own exactly one block
      if ((p.on_gpu || p.h2d_inflight) != (p.block >= 0)) throw LogicError("page residency and block ownership disagree");
      if (p.block >= 0) claim(block_seen, p.block, "block");
      if (p.host_tokens > 0 && p.slot < 0) throw LogicError("host data without a host slot");
      if (p.slot >= 0) claim(slot_seen, p.slot, "host slot");
    }
    if (gpu_tokens != r.gpu_tokens) throw LogicError("cached gpu token count drifted");
  }
  for (const auto& [jid, job] : jobs_) {
    for (const Delta& d : job.deltas) host_recount += (d.to - d.from) * bpt;
  }
  if (gpu_recount != gpu_used_) throw LogicError("gpu byte accounting drifted");
  if (host_recount != host_used_) throw LogicError("host byte accounting drifted");
  if (gpu_used_ > cfg_.gpu_capacity) throw LogicError("gpu capacity exceeded");
  if (host_used_ > cfg_.host_capacity) throw LogicError("host capacity exceeded");
  for (int32_t b : free_blocks_) claim(block_seen, b, "block");
  for (const Quarantined& q : block_q_) claim(block_seen, q.id, "block");
  for (int32_t s : free_slots_) claim(slot_seen, s, "host slot");
  for (const Quarantined& q : slot_q_) claim(slot_seen, q.id, "host slot");
  for (uint8_t v : block_seen) {
    if (!v) throw LogicError("block leaked from the pool");
  }
  for (uint8_t v : slot_seen) {
    if (!v) throw LogicError("host slot leaked from the pool");
  }
}

// Byte-identical to KvCacheManager::page_table_json (kv_cache.cpp:622-634):
// nlohmann::json::dump() of an object with sorted keys, compact separators.
std::string BlockPool::page_table_json(int64_t id) const {
  const Req& r = req(id);
  std::ostringstream out;
  out << "{\"pages\":[";
  int64_t start = 0;
  for (size_t i = 0; i < r.pages.size(); ++i) {
    const Page& p = r.pages[i];
    if (i) out << ",";
    out << "{\"location\":\"" << loc_name(p.loc()) << "\",\"range\":[" << start << ","
        << start + p.tokens << "]}";
    start += p.tokens;
  }
  out << "],\"request\":" << id << "}";
  return out.str();
}

}  // namespace csb
