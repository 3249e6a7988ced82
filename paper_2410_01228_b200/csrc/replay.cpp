// Replay of a recorded reference call log through the C-ABI -- the engine
// loop of coserve::SimEngine (sim_engine.cpp:250-294 dispatch, :146-185
// safepoint, :187-240 iteration end, :242-248 transfer completion) reduced to
// its hot-path call sites, in C++ so host overhead per iteration stays at
// the level of the reference's own loop. Ops are pre-encoded by replay.py.
#include <time.h>

#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "../../include/conserve_b200.h"

namespace {
enum Op : int64_t {
  kRegister = 0, kAlloc = 1, kCommit = 2, kRollback = 3, kEvict = 4, kDiscard = 5, kReleaseOd = 6, kStage = 7,
  kFlush = 8, kPrefetch = 9, kDone = 10, kPaused = 11, kActive = 12, kRelease = 13, kDispatch = 14, kSignal = 15,
  kIterEnd = 16, kBuild = 17, kDrop = 18, kPageTables = 19
};

// Same digest as oracle/lockstep/recorder.cpp page_table_digest(): FNV-1a over
// page_table_json | request_gpu_pages | covered_tokens of every live request,
// ascending id -- computed here from the B200 engine's block pool.
bool page_table_digest(cs_engine* e, const std::set<int64_t>& live, uint64_t* out) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const char* s, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      h ^= static_cast<unsigned char>(s[i]);
      h *= 1099511628211ull;
    }
  };
  std::string buf(1 << 16, '\0');
  for (int64_t id : live) {
    size_t len = 0;
    if (cs_kv_page_table_json(e, id, nullptr, 0, &len) != CS_OK) return false;
    if (len + 1 > buf.size()) buf.resize(len + 1);
    if (cs_kv_page_table_json(e, id, &buf[0], buf.size(), &len) != CS_OK) return false;
    mix(buf.data(), len);
    int64_t pages = 0, covered = 0, pending = 0;
    if (cs_kv_request_info(e, id, &pages, &covered, &pending) != CS_OK) return false;
    const std::string tail = "|" + std::to_string(pages) + "|" + std::to_string(covered) + "\n";
    mix(tail.data(), tail.size());
  }
  *out = h;
  return true;
}

double now_ms() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<double>(ts.tv_sec) * 1e3 + static_cast<double>(ts.tv_nsec) / 1e6;
}
}  // namespace

extern "C" int cs_replay_run(cs_engine* e, const int64_t* ops, int64_t op_begin, int64_t op_end,
                             const int64_t* plans, double* gpu_ms, double* wall_end_ms, int32_t* dropped_layer,
                             double* drop_latency_us, double* pre_drop_layer_us, int32_t* gemm_trunc_layer,
                             int64_t* h2d_bytes,
                             int64_t* d2h_bytes, cs_replay_stats* st) {
  std::memset(st, 0, sizeof(*st));
  st->first_mismatch_op = -1;
  auto mismatch = [&](int64_t i) {
    if (st->first_mismatch_op < 0) st->first_mismatch_op = i;
    ++st->mismatches;
  };
  static uint64_t epoch = 1000;  // distinct from any flag left by earlier runs
  std::vector<cs_batch_entry> entries;
  std::set<int64_t> live;  // registered, not released (as the recorder tracks them)
  bool inflight = false, signal_armed = false;
  int32_t signal_layer = 0;  // the reference's drop layer of the in-flight iteration
  int64_t it = 0;
  const double t0 = now_ms();
  for (int64_t i = op_begin; i < op_end; ++i) {
    const int64_t* o = ops + 8 * i;
    int rc = CS_OK;
    const double t_op = now_ms();
    switch (o[0]) {
      case kRegister:
        rc = cs_kv_register_request(e, o[1], static_cast<int32_t>(o[2]));
        live.insert(o[1]);
        break;
      case kAlloc: {
        cs_alloc_result r{};
        rc = cs_kv_allocate(e, o[1], o[2], o[3], &r);
        if (rc == CS_OK && (r.ok != o[4] || r.shortfall_pages != o[5])) mismatch(i);
        break;
      }
      case kCommit:
        rc = cs_kv_commit(e, o[1]);
        break;
      case kRollback:
        rc = cs_kv_rollback(e, o[1]);
        break;
      case kEvict: {
        cs_evict_stats s{};
        rc = cs_kv_evict_request_gpu(e, o[1], o[2], o[3], &s);
        if (rc == CS_OK && (s.freed_pages != o[4] || s.pending_pages != o[5] || s.discarded_tokens != o[6]))
          mismatch(i);
        break;
      }
      case kDiscard: {
        cs_evict_stats s{};
        rc = cs_kv_discard_request(e, o[1], o[2], &s);
        if (rc == CS_OK && (s.freed_pages != o[3] || s.discarded_tokens != o[4])) mismatch(i);
        break;
      }
      case kReleaseOd: {
        int64_t freed = 0, nd = 0, disc[512];
        rc = cs_kv_release_offline_pages_on_demand(e, o[1], o[2], &freed, disc, 256, &nd);
        if (rc == CS_OK && freed != o[3]) mismatch(i);
        break;
      }
      case kStage:
        rc = cs_kv_stage_checkpoint(e, o[1], o[2], o[3]);
        break;
      case kFlush:
      case kPrefetch: {
        cs_transfer_job j{};
        int32_t has = 0;
        rc = o[0] == kFlush ? cs_kv_flush_checkpoints(e, o[1], &j, &has)
                            : cs_kv_start_prefetch(e, o[7], o[1], &j, &has);
        if (rc == CS_OK && (has != o[2] || (has && (j.id != o[3] || j.bytes != o[4] || j.done_time != o[5]))))
          mismatch(i);
        break;
      }
      case kDone: {
        cs_transfer_done d{};
        rc = cs_kv_on_transfer_done(e, o[1], o[2], &d);
        if (rc == CS_OK && d.freed_pages != o[3]) mismatch(i);
        break;
      }
      case kPaused:
        rc = cs_kv_on_request_paused(e, o[1], static_cast<uint64_t>(o[2]));
        break;
      case kActive:
        rc = cs_kv_on_request_active(e, o[1]);
        break;
      case kRelease:
        rc = cs_kv_release_request(e, o[1]);
        live.erase(o[1]);
        break;
      case kDispatch: {
        const int64_t off = o[1], n = o[2];
        entries.resize(static_cast<size_t>(n));
        for (int64_t k = 0; k < n; ++k) {
          const int64_t* p = plans + 5 * (off + k);
          entries[static_cast<size_t>(k)] = cs_batch_entry{p[0], p[1], p[2], static_cast<int32_t>(p[3]),
                                                           static_cast<int32_t>(p[4])};
        }
        ++epoch;
        rc = cs_forward_launch(e, entries.data(), static_cast<int32_t>(n), epoch);
        inflight = rc == CS_OK;
        // o[3] = 1 + the layer at which the reference dropped offline work
        // this iteration (0: no drop)
        signal_armed = o[3] != 0;
        signal_layer = static_cast<int32_t>(o[3] - 1);
        break;
      }
      case kSignal:
        if (inflight && signal_armed) {
          // Alg. 1 fired while the reference's forward was in layer
          // signal_layer - 1 (its drop took effect at the next safepoint,
          // preemption.cpp:95-114): store the flag once the device has
          // entered that layer, so the drop lands where the reference's did
          // and flag -> drop is the real one-safepoint latency.
          const double w0 = now_ms();
          for (;;) {
            int32_t at = -1, done = 0;
            rc = cs_iter_progress(e, &at);
            if (rc != CS_OK || at >= signal_layer - 1) break;
            rc = cs_iter_poll(e, &done);
            if (rc != CS_OK || done || now_ms() - w0 > 5000.0) break;
          }
          if (rc == CS_OK) rc = cs_preempt_signal(e, epoch);
          signal_armed = false;
        }
        break;
      case kIterEnd: {
        if (!inflight) break;
        cs_iter_info info{};
        rc = cs_iter_wait(e, &info, nullptr, 0, nullptr);
        inflight = false;
        if (rc == CS_OK) {
          if (gpu_ms) gpu_ms[it] = info.gpu_ms;
          if (wall_end_ms) wall_end_ms[it] = now_ms() - t0;
          if (dropped_layer) dropped_layer[it] = info.preempted_at_layer;
          if (drop_latency_us) drop_latency_us[it] = info.preempt_signal_to_drop_us;
          if (pre_drop_layer_us) pre_drop_layer_us[it] = info.pre_drop_layer_us;
          if (gemm_trunc_layer) gemm_trunc_layer[it] = info.gemm_trunc_layer;
          if (h2d_bytes) h2d_bytes[it] = info.h2d_bytes;
          if (d2h_bytes) d2h_bytes[it] = info.d2h_bytes;
          ++it;
        }
        break;
      }
      case kPageTables: {
        // o[1] live requests, o[2] reference digest, o[3] != 0: check enabled
        if (o[3] == 0) break;
        uint64_t h = 0;
        if (!page_table_digest(e, live, &h)) {
          rc = CS_ERR_LOGIC;
          break;
        }
        if (static_cast<int64_t>(live.size()) != o[1] || static_cast<int64_t>(h) != o[2]) mismatch(i);
        break;
      }
      case kBuild:
      case kDrop:
        break;
      default:
        rc = CS_ERR_INVALID;
    }
    if (o[0] >= 0 && o[0] < 20) st->op_ms[o[0]] += now_ms() - t_op;
    if (rc != CS_OK) {
      st->iterations = it;
      st->wall_ms = now_ms() - t0;
      if (st->first_mismatch_op < 0) st->first_mismatch_op = i;
      return rc;
    }
  }
  if (inflight) {  // the reference stops at termination with an iteration in flight
    cs_iter_info info{};
    const int rc = cs_iter_wait(e, &info, nullptr, 0, nullptr);
    if (rc != CS_OK) return rc;
    if (gpu_ms) gpu_ms[it] = info.gpu_ms;
    if (wall_end_ms) wall_end_ms[it] = now_ms() - t0;
    if (dropped_layer) dropped_layer[it] = info.preempted_at_layer;
    ++it;
  }
  st->iterations = it;
  st->wall_ms = now_ms() - t0;
  return CS_OK;
}
