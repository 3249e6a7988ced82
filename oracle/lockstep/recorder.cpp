// Lockstep recorder -- TEST / BENCH INFRASTRUCTURE ONLY (the checker side).
//
// Runs the UNMODIFIED reference coserve::SimEngine (compiled from
// /root/reference into oracle/_ref by oracle/Makefile) and records, in order,
// every call the reference's engine and scheduler make across the hot-path
// seams: each KvCacheManager mutation with its arguments and
// results, every dispatched BatchPlan (captured at its oracle_latency call,
// sim_engine.cpp:256), every safepoint drop (IterationExecution::apply_drop,
// preemption.cpp:105-114), every preemption signal decision
// (on_recv_online_request / memory_pressure_preempt_needed), every iteration
// end (Scheduler::on_iteration_end) and the engine's own JSONL events.
//
// The calls are intercepted with GNU ld --wrap on the reference's object
// files (cross-object references only, so internal helper calls such as
// release_offline_pages_on_demand -> evict_request_gpu are not double
// counted). Nothing in /root/reference is copied or modified.
//
// The resulting call log is what a drop-in B200 engine receives: tests replay
// it through the C-ABI and compare page tables / byte counts / job timelines
// after every call; bench.py replays it with real GPU execution.
//
// usage: recorder <run_config.json> <out_dir>
//   writes out_dir/calls.jsonl, out_dir/metrics.json, out_dir/requests.jsonl
#include <cstdio>
#include <fstream>
#include <set>
#include <iostream>
#include <sstream>
#include <streambuf>
#include <string>

#include "coserve/config.hpp"
#include "coserve/kv_cache.hpp"
#include "coserve/metrics.hpp"
#include "coserve/perf_model.hpp"
#include "coserve/preemption.hpp"
#include "coserve/scheduler.hpp"
#include "coserve/sim_engine.hpp"

using namespace coserve;

static std::FILE* g_out = nullptr;
static int g_depth = 0;  // nested wrapped calls (none expected; guarded)
static void emit(const std::string& s);
static const KvCacheManager* g_kv = nullptr;  // the engine's manager (first wrapped call)
static std::set<int64_t> g_live;              // registered, not yet released

// FNV-1a over the logical page table of every live request, ascending id:
// page_table_json (kv_cache.cpp:622-634) | request_gpu_pages | covered_tokens.
// The replay recomputes the same digest from the B200 engine's block pool
// (csrc/replay.cpp) -- a per-iteration bit-exact page-table comparison.
static uint64_t page_table_digest() {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const std::string& s) {
    for (unsigned char c : s) {
      h ^= c;
      h *= 1099511628211ull;
    }
  };
  for (int64_t id : g_live) {
    mix(g_kv->page_table_json(id));
    mix("|" + std::to_string(g_kv->request_gpu_pages(id)) + "|" + std::to_string(g_kv->covered_tokens(id)) + "\n");
  }
  return h;
}

static void emit_page_tables(const char* where) {
  if (!g_kv) return;
  char buf[160];
  std::snprintf(buf, sizeof(buf), "{\"op\":\"pt\",\"at\":\"%s\",\"n\":%zu,\"hash\":\"%016llx\"}", where,
                g_live.size(), static_cast<unsigned long long>(page_table_digest()));
  emit(buf);
}

static void emit(const std::string& s) {
  if (g_out) {
    std::fputs(s.c_str(), g_out);
    std::fputc('\n', g_out);
  }
}

static std::string job_json(const std::optional<TransferJob>& j) {
  if (!j) return "null";
  std::ostringstream o;
  o.precision(17);
  o << "{\"id\":" << j->id << ",\"dir\":" << static_cast<int>(j->direction) << ",\"bytes\":" << j->bytes
    << ",\"enqueue\":" << j->enqueue_time << ",\"start\":" << j->start_time << ",\"done\":" << j->done_time
    << ",\"transfer_us\":" << j->transfer_us << ",\"gather_us\":" << j->gather_us << "}";
  return o.str();
}

static std::string plan_json(const BatchPlan& p) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < p.entries.size(); ++i) {
    const BatchEntry& e = p.entries[i];
    if (i) o << ",";
    o << "[" << e.request_id << "," << e.compute_tokens << "," << e.context_tokens << ","
      << static_cast<int>(e.kind) << "," << (e.online ? 1 : 0) << "]";
  }
  o << "]";
  return o.str();
}

// Event sink: forwards every SimEngine JSONL event line into the call log.
class SinkBuf : public std::streambuf {
  std::string line_;

 protected:
  int overflow(int c) override {
    if (c == '\n') {
      emit("{\"ev\":" + line_ + "}");
      line_.clear();
    } else if (c != EOF) {
      line_.push_back(static_cast<char>(c));
    }
    return c;
  }
};

#define REAL(sym) __real_##sym
#define WRAP(sym) __wrap_##sym

extern "C" {
// ---- KvCacheManager mutations (kv_cache.hpp:100-138) ----
void REAL(_ZN7coserve14KvCacheManager16register_requestElb)(KvCacheManager*, int64_t, bool);
void WRAP(_ZN7coserve14KvCacheManager16register_requestElb)(KvCacheManager* s, int64_t id, bool on) {
  REAL(_ZN7coserve14KvCacheManager16register_requestElb)(s, id, on);
  g_kv = s;
  g_live.insert(id);
  emit("{\"op\":\"register\",\"id\":" + std::to_string(id) + ",\"online\":" + (on ? "1" : "0") + "}");
}
AllocResult REAL(_ZN7coserve14KvCacheManager8allocateElll)(KvCacheManager*, int64_t, int64_t, int64_t);
AllocResult WRAP(_ZN7coserve14KvCacheManager8allocateElll)(KvCacheManager* s, int64_t id, int64_t n, int64_t now) {
  AllocResult r = REAL(_ZN7coserve14KvCacheManager8allocateElll)(s, id, n, now);
  emit("{\"op\":\"allocate\",\"id\":" + std::to_string(id) + ",\"n\":" + std::to_string(n) + ",\"now\":" +
       std::to_string(now) + ",\"ok\":" + (r.ok ? "1" : "0") + ",\"short\":" + std::to_string(r.shortfall_pages) +
       "}");
  return r;
}
void REAL(_ZN7coserve14KvCacheManager18commit_allocationsEl)(KvCacheManager*, int64_t);
void WRAP(_ZN7coserve14KvCacheManager18commit_allocationsEl)(KvCacheManager* s, int64_t id) {
  REAL(_ZN7coserve14KvCacheManager18commit_allocationsEl)(s, id);
  emit("{\"op\":\"commit\",\"id\":" + std::to_string(id) + "}");
}
void REAL(_ZN7coserve14KvCacheManager20rollback_allocationsEl)(KvCacheManager*, int64_t);
void WRAP(_ZN7coserve14KvCacheManager20rollback_allocationsEl)(KvCacheManager* s, int64_t id) {
  REAL(_ZN7coserve14KvCacheManager20rollback_allocationsEl)(s, id);
  emit("{\"op\":\"rollback\",\"id\":" + std::to_string(id) + "}");
}
EvictStats REAL(_ZN7coserve14KvCacheManager17evict_request_gpuElll)(KvCacheManager*, int64_t, int64_t, int64_t);
EvictStats WRAP(_ZN7coserve14KvCacheManager17evict_request_gpuElll)(KvCacheManager* s, int64_t id, int64_t now,
                                                                   int64_t maxp) {
  EvictStats r = REAL(_ZN7coserve14KvCacheManager17evict_request_gpuElll)(s, id, now, maxp);
  emit("{\"op\":\"evict\",\"id\":" + std::to_string(id) + ",\"now\":" + std::to_string(now) + ",\"max\":" +
       std::to_string(maxp) + ",\"freed\":" + std::to_string(r.freed_pages) + ",\"pending\":" +
       std::to_string(r.pending_pages) + ",\"discarded\":" + std::to_string(r.discarded_tokens) + "}");
  return r;
}
EvictStats REAL(_ZN7coserve14KvCacheManager15discard_requestEll)(KvCacheManager*, int64_t, int64_t);
EvictStats WRAP(_ZN7coserve14KvCacheManager15discard_requestEll)(KvCacheManager* s, int64_t id, int64_t now) {
  EvictStats r = REAL(_ZN7coserve14KvCacheManager15discard_requestEll)(s, id, now);
  emit("{\"op\":\"discard\",\"id\":" + std::to_string(id) + ",\"now\":" + std::to_string(now) + ",\"freed\":" +
       std::to_string(r.freed_pages) + ",\"discarded\":" + std::to_string(r.discarded_tokens) + "}");
  return r;
}
ReleaseStats REAL(_ZN7coserve14KvCacheManager31release_offline_pages_on_demandEll)(KvCacheManager*, int64_t,
                                                                                   int64_t);
ReleaseStats WRAP(_ZN7coserve14KvCacheManager31release_offline_pages_on_demandEll)(KvCacheManager* s,
                                                                                   int64_t need, int64_t now) {
  ReleaseStats r = REAL(_ZN7coserve14KvCacheManager31release_offline_pages_on_demandEll)(s, need, now);
  std::ostringstream o;
  o << "{\"op\":\"release_on_demand\",\"need\":" << need << ",\"now\":" << now << ",\"freed\":" << r.freed_pages
    << ",\"discards\":[";
  for (size_t i = 0; i < r.discards.size(); ++i)
    o << (i ? "," : "") << "[" << r.discards[i].first << "," << r.discards[i].second << "]";
  o << "]}";
  emit(o.str());
  return r;
}
void REAL(_ZN7coserve14KvCacheManager16stage_checkpointElll)(KvCacheManager*, int64_t, int64_t, int64_t);
void WRAP(_ZN7coserve14KvCacheManager16stage_checkpointElll)(KvCacheManager* s, int64_t id, int64_t a, int64_t b) {
  REAL(_ZN7coserve14KvCacheManager16stage_checkpointElll)(s, id, a, b);
  emit("{\"op\":\"stage\",\"id\":" + std::to_string(id) + ",\"from\":" + std::to_string(a) + ",\"to\":" +
       std::to_string(b) + "}");
}
std::optional<TransferJob> REAL(_ZN7coserve14KvCacheManager17flush_checkpointsEl)(KvCacheManager*, int64_t);
std::optional<TransferJob> WRAP(_ZN7coserve14KvCacheManager17flush_checkpointsEl)(KvCacheManager* s, int64_t now) {
  auto r = REAL(_ZN7coserve14KvCacheManager17flush_checkpointsEl)(s, now);
  emit("{\"op\":\"flush\",\"now\":" + std::to_string(now) + ",\"job\":" + job_json(r) + "}");
  return r;
}
std::optional<TransferJob> REAL(_ZN7coserve14KvCacheManager14start_prefetchEll)(KvCacheManager*, int64_t, int64_t);
std::optional<TransferJob> WRAP(_ZN7coserve14KvCacheManager14start_prefetchEll)(KvCacheManager* s, int64_t id,
                                                                                int64_t now) {
  auto r = REAL(_ZN7coserve14KvCacheManager14start_prefetchEll)(s, id, now);
  emit("{\"op\":\"prefetch\",\"id\":" + std::to_string(id) + ",\"now\":" + std::to_string(now) + ",\"job\":" +
       job_json(r) + "}");
  return r;
}
TransferDoneEffects REAL(_ZN7coserve14KvCacheManager16on_transfer_doneEll)(KvCacheManager*, int64_t, int64_t);
TransferDoneEffects WRAP(_ZN7coserve14KvCacheManager16on_transfer_doneEll)(KvCacheManager* s, int64_t job,
                                                                           int64_t now) {
  TransferDoneEffects r = REAL(_ZN7coserve14KvCacheManager16on_transfer_doneEll)(s, job, now);
  std::ostringstream o;
  o << "{\"op\":\"done\",\"job\":" << job << ",\"now\":" << now << ",\"freed\":" << r.freed_pages
    << ",\"resident\":[";
  for (size_t i = 0; i < r.became_resident.size(); ++i) o << (i ? "," : "") << r.became_resident[i];
  o << "]}";
  emit(o.str());
  return r;
}
void REAL(_ZN7coserve14KvCacheManager17on_request_pausedElm)(KvCacheManager*, int64_t, uint64_t);
void WRAP(_ZN7coserve14KvCacheManager17on_request_pausedElm)(KvCacheManager* s, int64_t id, uint64_t seq) {
  REAL(_ZN7coserve14KvCacheManager17on_request_pausedElm)(s, id, seq);
  emit("{\"op\":\"paused\",\"id\":" + std::to_string(id) + ",\"seq\":" + std::to_string(seq) + "}");
}
void REAL(_ZN7coserve14KvCacheManager17on_request_activeEl)(KvCacheManager*, int64_t);
void WRAP(_ZN7coserve14KvCacheManager17on_request_activeEl)(KvCacheManager* s, int64_t id) {
  REAL(_ZN7coserve14KvCacheManager17on_request_activeEl)(s, id);
  emit("{\"op\":\"active\",\"id\":" + std::to_string(id) + "}");
}
void REAL(_ZN7coserve14KvCacheManager15release_requestEl)(KvCacheManager*, int64_t);
void WRAP(_ZN7coserve14KvCacheManager15release_requestEl)(KvCacheManager* s, int64_t id) {
  REAL(_ZN7coserve14KvCacheManager15release_requestEl)(s, id);
  g_live.erase(id);
  emit("{\"op\":\"release\",\"id\":" + std::to_string(id) + "}");
}

// ---- forward / safepoint seams ----
BuildResult REAL(_ZN7coserve9Scheduler11build_batchEl)(Scheduler*, int64_t);
BuildResult WRAP(_ZN7coserve9Scheduler11build_batchEl)(Scheduler* s, int64_t now) {
  emit_page_tables("build");
  emit("{\"op\":\"build\",\"now\":" + std::to_string(now) + "}");
  return REAL(_ZN7coserve9Scheduler11build_batchEl)(s, now);
}
double REAL(
    _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
    const OracleParams&, const BatchPlan&, Rng&);
double WRAP(
    _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
    const OracleParams& p, const BatchPlan& plan, Rng& rng) {
  const double ms = REAL(
      _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
      p, plan, rng);
  std::ostringstream o;
  o.precision(17);
  o << "{\"op\":\"dispatch\",\"plan\":" << plan_json(plan) << ",\"latency_ms\":" << ms << "}";
  emit(o.str());
  return ms;
}
MonitorDecision REAL(_ZN7coserve22on_recv_online_requestEbddd)(bool, double, double, double);
MonitorDecision WRAP(_ZN7coserve22on_recv_online_requestEbddd)(bool b, double on, double rem, double budget) {
  MonitorDecision d = REAL(_ZN7coserve22on_recv_online_requestEbddd)(b, on, rem, budget);
  if (d == MonitorDecision::kSignalPreempt) emit("{\"op\":\"signal\",\"why\":\"ttft\"}");
  return d;
}
bool REAL(_ZNK7coserve9Scheduler30memory_pressure_preempt_neededEl)(const Scheduler*, int64_t);
bool WRAP(_ZNK7coserve9Scheduler30memory_pressure_preempt_neededEl)(const Scheduler* s, int64_t now) {
  const bool r = REAL(_ZNK7coserve9Scheduler30memory_pressure_preempt_neededEl)(s, now);
  if (r) emit("{\"op\":\"signal\",\"why\":\"memory\",\"now\":" + std::to_string(now) + "}");
  return r;
}
void REAL(_ZN7coserve18IterationExecution10apply_dropElld)(IterationExecution*, int64_t, int64_t, double);
void WRAP(_ZN7coserve18IterationExecution10apply_dropElld)(IterationExecution* s, int64_t layer, int64_t check_end,
                                                          double residual_ms) {
  REAL(_ZN7coserve18IterationExecution10apply_dropElld)(s, layer, check_end, residual_ms);
  std::ostringstream o;
  o.precision(17);
  o << "{\"op\":\"drop\",\"layer\":" << layer << ",\"check_end\":" << check_end << ",\"residual_ms\":" << residual_ms
    << "}";
  emit(o.str());
}
std::vector<int64_t> REAL(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(Scheduler*, const BatchPlan&,
                                                                                    int64_t);
std::vector<int64_t> WRAP(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(Scheduler* s,
                                                                                    const BatchPlan& plan,
                                                                                    int64_t now) {
  emit("{\"op\":\"iter_end\",\"now\":" + std::to_string(now) + ",\"plan\":" + plan_json(plan) + "}");
  auto r = REAL(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(s, plan, now);
  std::ostringstream o;
  o << "{\"op\":\"completed\",\"ids\":[";
  for (size_t i = 0; i < r.size(); ++i) o << (i ? "," : "") << r[i];
  o << "]}";
  emit(o.str());
  return r;
}
}  // extern "C"

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: recorder <run_config.json> <out_dir>\n");
    return 2;
  }
  const std::string out_dir = argv[2];
  RunConfig cfg = load_run_config(argv[1]);
  g_out = std::fopen((out_dir + "/calls.jsonl").c_str(), "w");
  emit("{\"config\":" + [&] {
    std::string s = run_config_to_json_text(cfg);
    std::string t;
    for (char c : s)
      if (c != '\n') t.push_back(c);
    return t;
  }() + "}");
  SinkBuf buf;
  std::ostream sink(&buf);
  SimEngine engine(cfg);
  engine.set_event_sink(&sink);
  MetricsReport rep;
  try {
    rep = engine.run();
  } catch (const std::exception& e) {
    emit(std::string("{\"error\":\"") + e.what() + "\"}");
    std::fclose(g_out);
    std::fprintf(stderr, "reference run failed: %s\n", e.what());
    return 3;
  }
  sink.flush();
  emit_page_tables("end");
  // The reference's own invariant audit (kv_cache.cpp:566-620) on the final
  // state: the replay must reach the same verdict.
  std::string audit = "ok";
  try {
    if (g_kv) g_kv->audit();
  } catch (const std::exception& e) {
    audit = e.what();
  }
  emit("{\"op\":\"audit\",\"result\":\"" + audit + "\"}");
  std::fclose(g_out);
  std::ofstream(out_dir + "/metrics.json") << rep.to_json_text();
  std::ofstream req(out_dir + "/requests.jsonl");
  for (const auto& [id, r] : engine.requests()) {
    req << "{\"id\":" << id << ",\"class\":\"" << to_string(r.cls) << "\",\"arrival\":" << r.arrival_time
        << ",\"in\":" << r.input_tokens << ",\"out\":" << r.output_tokens << ",\"prefill_done\":" << r.prefill_done
        << ",\"decode_done\":" << r.decode_done << ",\"tokens\":[";
    for (size_t i = 0; i < r.token_completion_times.size(); ++i)
      req << (i ? "," : "") << r.token_completion_times[i];
    req << "]}\n";
  }
  std::printf("iterations=%lld horizon_s=%.6f offline_tok_s=%.3f preemptions=%lld d2h=%lld h2d=%lld\n",
              static_cast<long long>(engine.iterations_dispatched()), rep.horizon_s, rep.offline_throughput_tok_s,
              static_cast<long long>(rep.preemptions), static_cast<long long>(rep.d2h_bytes),
              static_cast<long long>(rep.h2d_bytes));
  return 0;
}
