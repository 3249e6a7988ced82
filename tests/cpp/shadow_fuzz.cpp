// Shadow-mode parity fuzz: drives the reference coserve::KvCacheManager
// (compiled from /root/reference into oracle/_ref/libcoserve.a -- the checker)
// and the B200 block pool (paper_2410_01228_b200/csrc/block_pool.cpp -- the
// product) with identical random operation sequences and compares, after
// every operation: return values, thrown exception type + message, byte
// counters, page_table_json of every live request, per-request page/token
// counts and both audits. Also checks the physical invariants (every resident
// page owns a distinct block; no block or slot leaks) via the pool's audit.
//
// Physical content model: a SimMover carries a tag per (block | host slot,
// token) -- tag(req, pos) is written when an allocation covers a position
// (the forward that computes it), gathers copy block -> slot, restores slot ->
// block, synchronously. After every call every GPU-resident page's block must
// hold tag(req, pos) for all its tokens and every page's host slot for its
// first host_tokens tokens: a checkpoint or restore that moves the wrong
// bytes is caught even when the page tables agree with the reference.
//
// usage: shadow_fuzz <seed> <ops> [incremental=1] [host_pages=256] [gpu_pages=64]
//        seed 0: the directed ADVICE r1 sequence (late partial checkpoint of a
//        page that was discarded and recomputed while its copy was in flight)
#include <cstdio>
#include <cstdlib>
#include <map>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "coserve/kv_cache.hpp"
#include "block_pool.h"

using namespace coserve;

struct SimMover : csb::Mover {
  std::vector<std::vector<int64_t>> blk, slot;  // [id][16] content tags (-1 = garbage)
  int64_t issued[2] = {0, 0};
  SimMover(int64_t n_blocks, int64_t n_slots)
      : blk(static_cast<size_t>(n_blocks), std::vector<int64_t>(16, -1)),
        slot(static_cast<size_t>(n_slots), std::vector<int64_t>(16, -1)) {}
  int64_t gather_to_host(const std::vector<csb::Segment>& segs, int64_t) override {
    for (const auto& g : segs)
      for (int t = g.t0; t < g.t1; ++t) slot[g.slot][t] = blk[g.block][t];
    return ++issued[0];
  }
  int64_t scatter_from_host(const std::vector<csb::Segment>& segs, int64_t) override {
    for (const auto& g : segs)
      for (int t = g.t0; t < g.t1; ++t) blk[g.block][t] = slot[g.slot][t];
    return ++issued[1];
  }
  int64_t done_prefix(int32_t dir) override { return issued[dir]; }
};

static int64_t tag(int64_t req, int64_t pos) { return req * 1000003 + pos; }

static int g_fail = 0;
#define EXPECT(cond, ...)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      std::fprintf(stderr, "MISMATCH line %d: ", __LINE__); \
      std::fprintf(stderr, __VA_ARGS__);                    \
      std::fprintf(stderr, "\n");                           \
      if (++g_fail > 5) std::exit(1);                       \
    }                                                       \
  } while (0)

struct Outcome {
  std::string kind;  // "" = ok, else exception class
  std::string msg;
};

template <typename F>
Outcome run(F&& f) {
  try {
    f();
    return {"", ""};
  } catch (const std::invalid_argument& e) {
    return {"invalid_argument", e.what()};
  } catch (const std::logic_error& e) {
    return {"logic_error", e.what()};
  } catch (const std::runtime_error& e) {
    return {"runtime_error", e.what()};
  }
}

static bool same_job(const std::optional<TransferJob>& a, const std::optional<cs_transfer_job>& b) {
  if (a.has_value() != b.has_value()) return false;
  if (!a) return true;
  return a->id == b->id && a->bytes == b->bytes && a->enqueue_time == b->enqueue_time &&
         a->start_time == b->start_time && a->done_time == b->done_time &&
         a->transfer_us == b->transfer_us && a->gather_us == b->gather_us &&
         static_cast<int>(a->direction) == b->direction;
}

int main(int argc, char** argv) {
  const uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1;
  const int ops = argc > 2 ? std::atoi(argv[2]) : 2000;
  const bool incremental = argc > 3 ? std::atoi(argv[3]) != 0 : true;
  const int64_t host_pages = argc > 4 ? std::atoll(argv[4]) : 256;
  const int64_t gpu_pages = argc > 5 ? std::atoll(argv[5]) : 64;

  ClusterConfig c;
  c.kv_bytes_per_token = 2048;
  c.gpu_kv_capacity = c.kv_bytes_per_token * 16 * gpu_pages;
  c.host_kv_capacity = c.kv_bytes_per_token * 16 * host_pages;
  c.d2h_bandwidth = 38797312000.0;
  c.h2d_bandwidth = 38797312000.0;
  c.gather_cost_us = 500.0;
  KvCacheManager ref(c, incremental);

  csb::PoolConfig pc;
  pc.page_tokens = 16;
  pc.kv_bytes_per_token = c.kv_bytes_per_token;
  pc.gpu_capacity = c.gpu_kv_capacity;
  pc.host_capacity = c.host_kv_capacity;
  pc.d2h_bw = c.d2h_bandwidth;
  pc.h2d_bw = c.h2d_bandwidth;
  pc.gather_us = c.gather_cost_us;
  pc.incremental = incremental;
  // Physical need = ceil(cap/page_bytes) + live requests with partial tails
  // + quarantine; random ops create many tiny requests.
  pc.n_blocks = gpu_pages * 8 + ops / 4 + 64;
  pc.n_slots = host_pages * 4 + ops / 4 + 64;
  pc.moved_bytes_per_token = c.kv_bytes_per_token;
  SimMover sim(pc.n_blocks, pc.n_slots);
  csb::BlockPool pool(pc, &sim);

  std::mt19937_64 rng(seed);
  auto rnd = [&](int64_t lo, int64_t hi) {  // inclusive
    return lo + static_cast<int64_t>(rng() % static_cast<uint64_t>(hi - lo + 1));
  };
  std::map<int64_t, bool> live;        // id -> online
  std::set<int64_t> uncommitted;
  std::map<int64_t, int64_t> job_done;  // job id -> done time
  int64_t next_id = 0, now = 0;
  uint64_t pause_seq = 0;
  std::map<std::string, int> op_count;

  auto pick = [&](bool offline_only) -> int64_t {
    std::vector<int64_t> ids;
    for (auto& [id, on] : live)
      if (!offline_only || !on) ids.push_back(id);
    if (ids.empty()) return -1;
    return ids[static_cast<size_t>(rnd(0, static_cast<int64_t>(ids.size()) - 1))];
  };

  // the forward of an allocation writes the KV of every position it covers
  auto write_growth = [&](int64_t id) {
    const csb::Req* r = pool.find(id);
    for (const csb::Growth& g : r->growth) {
      const csb::Page& p = r->pages[g.page];
      if (p.block < 0) continue;
      for (int64_t t = g.was_discarded ? 0 : g.prev_tokens; t < p.tokens; ++t)
        sim.blk[p.block][t] = tag(id, static_cast<int64_t>(g.page) * 16 + t);
    }
  };
  auto check_content = [&](const char* op) {
    for (auto& [id, on] : live) {
      const csb::Req* r = pool.find(id);
      for (size_t i = 0; i < r->pages.size(); ++i) {
        const csb::Page& p = r->pages[i];
        if (p.on_gpu && !p.discarded)
          for (int64_t t = 0; t < p.tokens; ++t)
            EXPECT(sim.blk[p.block][t] == tag(id, static_cast<int64_t>(i) * 16 + t),
                   "%s: block %d of req %lld page %zu holds wrong KV at %lld", op, p.block, (long long)id, i,
                   (long long)t);
        if (p.host_tokens > 0 && p.slot >= 0)
          for (int64_t t = 0; t < p.host_tokens; ++t)
            EXPECT(sim.slot[p.slot][t] == tag(id, static_cast<int64_t>(i) * 16 + t),
                   "%s: host slot %d of req %lld page %zu holds wrong KV at %lld", op, p.slot, (long long)id, i,
                   (long long)t);
      }
    }
  };
  auto compare_state = [&](const char* op) {
    check_content(op);
    EXPECT(ref.gpu_used_bytes() == pool.gpu_used(), "%s gpu_used %lld vs %lld", op,
           (long long)ref.gpu_used_bytes(), (long long)pool.gpu_used());
    EXPECT(ref.host_used_bytes() == pool.host_used(), "%s host_used %lld vs %lld", op,
           (long long)ref.host_used_bytes(), (long long)pool.host_used());
    EXPECT(ref.total_d2h_bytes() == pool.total_d2h(), "%s d2h", op);
    EXPECT(ref.total_h2d_bytes() == pool.total_h2d(), "%s h2d", op);
    EXPECT(ref.recompute_tagged_tokens() == pool.recompute_tagged(), "%s tagged", op);
    EXPECT(ref.gpu_free_pages() == pool.gpu_free_pages(), "%s free pages", op);
    EXPECT(ref.transfers_inflight() == pool.transfers_inflight(), "%s inflight", op);
    EXPECT(ref.releasable_offline_pages_now() == pool.releasable_offline_pages_now(), "%s releasable", op);
    for (auto& [id, on] : live) {
      const std::string a = ref.page_table_json(id), b = pool.page_table_json(id);
      EXPECT(a == b, "%s page table id %lld\n ref %s\n b200 %s", op, (long long)id, a.c_str(), b.c_str());
      EXPECT(ref.request_gpu_pages(id) == pool.request_gpu_pages(id), "%s gpu pages", op);
      EXPECT(ref.covered_tokens(id) == pool.covered_tokens(id), "%s covered", op);
      EXPECT(ref.pending_append_tokens(id) == pool.pending_append_tokens(id), "%s pending", op);
      EXPECT(ref.fully_resident(id) == pool.fully_resident(id), "%s resident", op);
      EXPECT(ref.prefetch_inflight(id) == pool.prefetch_inflight(id), "%s prefetch", op);
      auto rc = ref.resume_cost(id);
      auto bc = pool.resume_cost(id);
      EXPECT(rc.host_only_pages == bc.host_only_pages && rc.host_only_bytes == bc.host_only_bytes &&
                 rc.discarded_tokens == bc.discarded_tokens,
             "%s resume cost", op);
    }
    Outcome ra = run([&] { ref.audit(); });
    Outcome pa = run([&] { pool.audit(); });
    if (ra.kind.empty()) {
      EXPECT(pa.kind.empty(), "%s audit: reference clean, b200 threw %s", op, pa.msg.c_str());
    } else {
      // The reference itself can reach audit-failing states (SURVEY.md App. A
      // D3); the pool must report the same logical violation.
      EXPECT(pa.msg == ra.msg, "%s audit: ref '%s' b200 '%s'", op, ra.msg.c_str(), pa.msg.c_str());
    }
  };

  if (seed == 0) {
    // tail checkpoint in flight (inflight_to 4), the tail
    // grows, evict pass 2 discards the page and frees its slot, recompute
    // re-materializes it, then the old copy completes.
    auto both = [&](const char* op, auto&& fr, auto&& fp) {
      Outcome oa = run(fr), ob = run(fp);
      EXPECT(oa.kind == ob.kind && oa.msg == ob.msg, "%s outcome '%s' vs '%s'", op, oa.msg.c_str(), ob.msg.c_str());
      compare_state(op);
    };
    ref.register_request(0, false);
    pool.register_request(0, false);
    live[0] = false;
    both("allocate 20", [&] { ref.allocate(0, 20, 0); }, [&] { pool.allocate(0, 20); write_growth(0); });
    both("commit", [&] { ref.commit_allocations(0); }, [&] { pool.commit(0); });
    both("stage", [&] { ref.stage_checkpoint(0, 0, 20); }, [&] { pool.stage_checkpoint(0, 0, 20); });
    int64_t jid = -1;
    both("flush", [&] { jid = ref.flush_checkpoints(0)->id; }, [&] { pool.flush_checkpoints(0); });
    both("allocate 2", [&] { ref.allocate(0, 2, 0); }, [&] { pool.allocate(0, 2); write_growth(0); });
    both("commit", [&] { ref.commit_allocations(0); }, [&] { pool.commit(0); });
    both("pause", [&] { ref.on_request_paused(0, 1); }, [&] { pool.on_request_paused(0, 1); });
    both("evict", [&] { ref.evict_request_gpu(0, 0, -1); }, [&] { pool.evict_request_gpu(0, -1); });
    both("active", [&] { ref.on_request_active(0); }, [&] { pool.on_request_active(0); });
    both("recompute allocate", [&] { ref.allocate(0, 6, 0); }, [&] { pool.allocate(0, 6); write_growth(0); });
    both("commit", [&] { ref.commit_allocations(0); }, [&] { pool.commit(0); });
    both("transfer done", [&] { ref.on_transfer_done(jid, 100000); }, [&] { pool.on_transfer_done(jid); });
    // the page now counts [0,4) as checkpointed: finish it and bring it back from host
    both("stage rest", [&] { ref.stage_checkpoint(0, 16, 22); }, [&] { pool.stage_checkpoint(0, 16, 22); });
    int64_t j2 = -1;
    both("flush 2", [&] { j2 = ref.flush_checkpoints(1)->id; }, [&] { pool.flush_checkpoints(1); });
    both("transfer done 2", [&] { ref.on_transfer_done(j2, 200000); }, [&] { pool.on_transfer_done(j2); });
    both("pause", [&] { ref.on_request_paused(0, 2); }, [&] { pool.on_request_paused(0, 2); });
    both("evict all", [&] { ref.evict_request_gpu(0, 0, -1); }, [&] { pool.evict_request_gpu(0, -1); });
    int64_t j3 = -1;
    both("prefetch", [&] { j3 = ref.start_prefetch(0, 300000)->id; }, [&] { pool.start_prefetch(0, 300000); });
    both("transfer done 3", [&] { ref.on_transfer_done(j3, 400000); }, [&] { pool.on_transfer_done(j3); });
    // blocks freed by one request must not wait behind an
    // unrelated checkpoint that is still copying on the device. 64-page pool
    // with 2 spare blocks; request 1 has a checkpoint in flight (never
    // completes here); request 2 releases 40 pages; 39 fresh pages for
    // request 3 must come from request 2's blocks.
    struct Pending : SimMover {
      using SimMover::SimMover;
      int64_t done_prefix(int32_t) override { return 0; }
    } pend(66, 64);
    csb::PoolConfig pc2 = pc;
    pc2.gpu_capacity = c.kv_bytes_per_token * 16 * 64;
    pc2.n_blocks = 66;
    pc2.n_slots = 64;
    pc2.fwd_quarantine = false;
    csb::BlockPool p2(pc2, &pend);
    p2.register_request(1, false);
    p2.register_request(2, false);
    p2.register_request(3, false);
    p2.allocate(1, 16);
    p2.commit(1);
    p2.stage_checkpoint(1, 0, 16);
    p2.flush_checkpoints(0);
    p2.allocate(2, 40 * 16);
    p2.commit(2);
    p2.release_request(2);
    Outcome o = run([&] { p2.allocate(3, 39 * 16); });
    EXPECT(o.kind.empty(), "allocate behind an unrelated in-flight checkpoint: %s", o.msg.c_str());
    std::printf("shadow_fuzz directed failures=%d fixups=%lld\n", g_fail, (long long)pool.fixup_gathers());
    return g_fail == 0 && pool.fixup_gathers() == 1 ? 0 : 1;
  }

  for (int step = 0; step < ops; ++step) {
    now += rnd(0, 3000);
    const int64_t r = rnd(0, 99);
    std::string op;
    if (r < 8 || live.empty()) {
      op = "register";
      const int64_t id = next_id++;
      const bool on = rnd(0, 3) == 0;
      ref.register_request(id, on);
      pool.register_request(id, on);
      live[id] = on;
    } else if (r < 30) {
      op = "allocate";
      const int64_t id = pick(false);
      const int64_t n = rnd(0, 3) == 0 ? rnd(0, 3) : rnd(1, 200);
      AllocResult a{};
      cs_alloc_result b{};
      Outcome oa = run([&] { a = ref.allocate(id, n, now); });
      Outcome ob = run([&] { b = pool.allocate(id, n); });
      EXPECT(oa.kind == ob.kind && oa.msg == ob.msg, "allocate outcome '%s' vs '%s'", oa.msg.c_str(), ob.msg.c_str());
      if (oa.kind.empty() && ob.kind.empty()) {
        EXPECT(a.ok == (b.ok != 0) && a.shortfall_pages == b.shortfall_pages, "allocate result");
        if (a.ok) uncommitted.insert(id);
        if (b.ok) write_growth(id);
      }
    } else if (r < 42) {
      op = "commit";
      const int64_t id = pick(false);
      ref.commit_allocations(id);
      pool.commit(id);
      uncommitted.erase(id);
    } else if (r < 46) {
      op = "rollback";
      const int64_t id = pick(false);
      ref.rollback_allocations(id);
      pool.rollback(id);
      uncommitted.erase(id);
    } else if (r < 50) {
      op = "evict";
      const int64_t id = pick(rnd(0, 5) != 0);
      const int64_t maxp = rnd(-1, 6);
      EvictStats a{};
      cs_evict_stats b{};
      Outcome oa = run([&] { a = ref.evict_request_gpu(id, now, maxp); });
      Outcome ob = run([&] { b = pool.evict_request_gpu(id, maxp); });
      EXPECT(oa.kind == ob.kind && oa.msg == ob.msg, "evict outcome");
      EXPECT(a.freed_pages == b.freed_pages && a.pending_pages == b.pending_pages &&
                 a.discarded_tokens == b.discarded_tokens,
             "evict stats");
    } else if (r < 52) {
      op = "discard";
      const int64_t id = pick(true);
      if (id < 0) continue;
      EvictStats a{};
      cs_evict_stats b{};
      Outcome oa = run([&] { a = ref.discard_request(id, now); });
      Outcome ob = run([&] { b = pool.discard_request(id); });
      EXPECT(oa.kind == ob.kind, "discard outcome");
      EXPECT(a.freed_pages == b.freed_pages && a.discarded_tokens == b.discarded_tokens, "discard stats");
    } else if (r < 56) {
      op = "release_on_demand";
      const int64_t need = rnd(0, 12);
      ReleaseStats a{};
      csb::ReleaseResult b{};
      Outcome oa = run([&] { a = ref.release_offline_pages_on_demand(need, now); });
      Outcome ob = run([&] { b = pool.release_offline_pages_on_demand(need); });
      EXPECT(oa.kind == ob.kind && oa.msg == ob.msg, "release outcome");
      EXPECT(a.freed_pages == b.freed_pages && a.discards == b.discards, "release stats");
    } else if (r < 70) {
      op = "stage";
      const int64_t id = pick(false);
      if (uncommitted.count(id)) continue;  // stage only committed coverage
      const int64_t cov = ref.covered_tokens(id);
      if (cov == 0) continue;
      const int64_t from = rnd(0, cov - 1), to = rnd(from, cov);
      ref.stage_checkpoint(id, from, to);
      pool.stage_checkpoint(id, from, to);
    } else if (r < 78) {
      op = "flush";
      std::optional<TransferJob> a;
      std::optional<cs_transfer_job> b;
      a = ref.flush_checkpoints(now);
      b = pool.flush_checkpoints(now);
      EXPECT(same_job(a, b), "flush job");
      if (a) job_done[a->id] = a->done_time;
    } else if (r < 84) {
      op = "prefetch";
      const int64_t id = pick(false);
      auto a = ref.start_prefetch(id, now);
      auto b = pool.start_prefetch(id, now);
      EXPECT(same_job(a, b), "prefetch job");
      if (a) job_done[a->id] = a->done_time;
    } else if (r < 90) {
      op = "transfer_done";
      if (job_done.empty()) continue;
      // event order: earliest done time, ties by job id
      auto best = job_done.begin();
      for (auto it = job_done.begin(); it != job_done.end(); ++it)
        if (it->second < best->second) best = it;
      const int64_t jid = best->first;
      now = std::max(now, best->second);
      job_done.erase(best);
      auto a = ref.on_transfer_done(jid, now);
      auto b = pool.on_transfer_done(jid);
      EXPECT(a.freed_pages == b.freed_pages && a.became_resident == b.became_resident, "done effects");
    } else if (r < 93) {
      op = "pause";
      const int64_t id = pick(false);
      ref.on_request_paused(id, ++pause_seq);
      pool.on_request_paused(id, pause_seq);
    } else if (r < 95) {
      op = "active";
      const int64_t id = pick(false);
      ref.on_request_active(id);
      pool.on_request_active(id);
    } else if (r < 97) {
      op = "release";
      const int64_t id = pick(false);
      ref.release_request(id);
      pool.release_request(id);
      live.erase(id);
      uncommitted.erase(id);
    } else {
      op = "recompute_chunk";
      const int64_t id = pick(false);
      const int64_t d = rnd(-1, 100), cap = rnd(-1, 200);
      EXPECT(ref.recompute_chunk(id, d, cap) == pool.recompute_chunk(id, d, cap), "recompute_chunk");
    }
    // An "iteration boundary" every few ops lets the physical quarantine drain.
    if (rnd(0, 4) == 0) {
      pool.on_forward_launched();
      pool.on_forward_completed();
    }
    op_count[op]++;
    compare_state(op.c_str());
  }
  std::printf("shadow_fuzz seed=%llu ops=%d incremental=%d failures=%d blocks_free=%lld/%lld\n",
              (unsigned long long)seed, ops, (int)incremental, g_fail, (long long)pool.free_blocks(),
              (long long)pool.n_blocks());
  for (auto& [k, v] : op_count) std::printf("  %s=%d", k.c_str(), v);
  std::printf("\n");
  return g_fail == 0 ? 0 : 1;
}
