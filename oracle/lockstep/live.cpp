// Live mode -- the reference's own engine loop driving the B200 data plane.
// TOOLS-SIDE EXECUTABLE (oracle/_ref/adapter/live): it links the UNMODIFIED
// reference Scheduler / SimEngine / metrics (compiled against the drop-in
// KvCacheManager of include/conserve_b200_kv.hpp) with libconserve_b200.so;
// the product library itself never links reference code.
//
// This is INTEGRATION.md section 2's dispatch patch, applied with GNU ld
// --wrap instead of an edit (nothing under /root/reference is modified):
//
//   * forward seam, proj/src/sim_engine.cpp:256
//       latency_ms = oracle_latency(config_.oracle, built.plan, noise_rng_)
//     -> the real 32/48/80-layer forward of built.plan on the B200
//        (cs_forward_launch), and the reference's event loop advances its
//        clock by the MEASURED device time of that forward. The reference's
//        own draw is still taken (same RNG stream) and reported beside it.
//   * KV seams: SimEngine's KvCacheManager is the adapter, backed by the
//     engine's HBM block pool / pinned host pool / D2H-H2D kernels
//     (conserve_b200::data_plane_model()).
//   * safepoint seam, IterationExecution::apply_drop (preemption.cpp:105-114):
//     the reference decides the drop on the measured timeline; the forward
//     already ran the whole plan, so the drop is applied to its outputs and
//     written-KV bookkeeping (cs_iter_retro_drop) and the rest of the
//     iteration is re-timed by the reference from the measured/predicted
//     ratio (sim_engine.cpp:156-161).
//   * iteration end, Scheduler::on_iteration_end: cs_iter_wait (outputs,
//     written KV, quarantine release) before the reference's own handling.
//
// Everything the reference writes is written by the reference's own code, so
// a B200 run produces the reference's wire formats: metrics.json
// (MetricsReport::to_json_text, metrics.cpp:114-191), events.jsonl
// (SimEngine::log_event, sim_engine.cpp:44-48 -- dispatch lines carry the
// measured latency_ms), timeseries.csv (metrics.cpp timeseries_csv) and
// requests.csv.
//
// usage: live <run_config.json> <out_dir> <preset: tiny|llama8b|qwen14b|llama70b> [--dry] [--device N]
//   --dry: bookkeeping-only engine and the reference's own latency (no GPU);
//          the outputs must then be byte-identical to the reference's
//          (tests/test_live.py).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "coserve/config.hpp"
#include "coserve/kv_cache.hpp"
#include "coserve/metrics.hpp"
#include "coserve/perf_model.hpp"
#include "coserve/preemption.hpp"
#include "coserve/scheduler.hpp"
#include "coserve/sim_engine.hpp"

using namespace coserve;

#define REAL(sym) __real_##sym
#define WRAP(sym) __wrap_##sym

namespace {
bool g_dry = false;
uint64_t g_epoch = 1;
int64_t g_iters = 0, g_drops = 0;
int32_t g_drop_layer = -1;
double g_measured_ms = 0, g_predicted_ms = 0;
std::vector<double> g_ratio;  // measured / reference-predicted, per dispatch

cs_engine* eng() {
  cs_engine* e = conserve_b200::last_engine();
  if (!e) throw std::logic_error("live: no data-plane engine");
  return e;
}
void check(int rc) {
  if (rc != CS_OK) throw std::runtime_error(std::string("live: ") + cs_last_error());
}

struct Shape {
  const char* name;
  int32_t L, hidden, hq, hkv, d, ffn, vocab;
  float theta;
};
const Shape kShapes[] = {
    {"tiny", 2, 256, 4, 4, 64, 512, 1024, 10000.f},
    {"llama8b", 32, 4096, 32, 8, 128, 14336, 128256, 500000.f},
    {"qwen14b", 48, 5120, 40, 8, 128, 13824, 152064, 1000000.f},
    {"llama70b", 80, 8192, 64, 8, 128, 28672, 128256, 500000.f},
};
}  // namespace

extern "C" {
double REAL(
    _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
    const OracleParams&, const BatchPlan&, Rng&);
double WRAP(
    _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
    const OracleParams& p, const BatchPlan& plan, Rng& rng) {
  const double predicted = REAL(
      _ZN7coserve14oracle_latencyERKNS_12OracleParamsERKNS_9BatchPlanERSt23mersenne_twister_engineImLm64ELm312ELm156ELm31ELm13043109905998158313ELm29ELm6148914691236517205ELm17ELm8202884508482404352ELm37ELm18444473444759240704ELm43ELm6364136223846793005EE)(
      p, plan, rng);
  std::vector<cs_batch_entry> ents;
  ents.reserve(plan.entries.size());
  for (const BatchEntry& b : plan.entries)
    ents.push_back(cs_batch_entry{b.request_id, b.compute_tokens, b.context_tokens, static_cast<int32_t>(b.kind),
                                  b.online ? 1 : 0});
  cs_engine* e = eng();
  check(cs_forward_launch(e, ents.data(), static_cast<int32_t>(ents.size()), ++g_epoch));
  ++g_iters;
  g_drop_layer = -1;
  g_predicted_ms += predicted;
  if (g_dry) return predicted;
  double ms = -1;
  for (;;) {  // the device time of this forward, once it completed
    check(cs_iter_elapsed(e, &ms));
    if (ms >= 0) break;
    std::this_thread::yield();
  }
  g_measured_ms += ms;
  if (predicted > 0) g_ratio.push_back(ms / predicted);
  return ms;
}

void REAL(_ZN7coserve18IterationExecution10apply_dropElld)(IterationExecution*, int64_t, int64_t, double);
void WRAP(_ZN7coserve18IterationExecution10apply_dropElld)(IterationExecution* s, int64_t layer, int64_t check_end,
                                                          double residual_ms) {
  REAL(_ZN7coserve18IterationExecution10apply_dropElld)(s, layer, check_end, residual_ms);
  g_drop_layer = static_cast<int32_t>(layer);
  ++g_drops;
  check(cs_iter_retro_drop(eng(), g_drop_layer));
}

std::vector<int64_t> REAL(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(Scheduler*, const BatchPlan&,
                                                                                    int64_t);
std::vector<int64_t> WRAP(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(Scheduler* s,
                                                                                    const BatchPlan& plan,
                                                                                    int64_t now) {
  cs_iter_info info{};
  check(cs_iter_wait(eng(), &info, nullptr, 0, nullptr));
  if (info.n_entries_after != static_cast<int32_t>(plan.entries.size()))
    throw std::logic_error("live: engine and reference disagree on the surviving entries");
  return REAL(_ZN7coserve9Scheduler16on_iteration_endERKNS_9BatchPlanEl)(s, plan, now);
}
}  // extern "C"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: live <run_config.json> <out_dir> <preset> [--dry] [--device N]\n");
    return 2;
  }
  const std::string out_dir = argv[2];
  const std::string preset = argv[3];
  int device = 0;
  for (int i = 4; i < argc; ++i) {
    if (!std::strcmp(argv[i], "--dry")) g_dry = true;
    if (!std::strcmp(argv[i], "--device") && i + 1 < argc) device = std::atoi(argv[++i]);
  }
  const RunConfig cfg = load_run_config(argv[1]);
  const Shape* sh = nullptr;
  for (const Shape& s : kShapes)
    if (preset == s.name) sh = &s;
  if (!sh) {
    std::fprintf(stderr, "unknown preset %s\n", preset.c_str());
    return 2;
  }
  cs_config model;
  cs_config_default(&model);
  model.num_layers = sh->L;
  model.hidden = sh->hidden;
  model.n_heads = sh->hq;
  model.n_kv_heads = sh->hkv;
  model.head_dim = sh->d;
  model.ffn = sh->ffn;
  model.vocab = sh->vocab;
  model.rope_theta = sh->theta;
  model.device = device;
  model.max_entries = 256;
  model.instrumented = cfg.policy.instrumented() ? 1 : 0;
  model.flags = g_dry ? (CS_FLAG_HOST_ONLY | CS_FLAG_NO_FWD_QUARANTINE) : 0;
  conserve_b200::data_plane_model() = &model;

  std::ostringstream events;
  SimEngine engine(cfg);
  engine.set_event_sink(&events);
  MetricsReport rep;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    rep = engine.run();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "live run failed: %s\n", e.what());
    return 3;
  }
  const double wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::ofstream(out_dir + "/metrics.json") << rep.to_json_text();
  std::ofstream(out_dir + "/events.jsonl") << events.str();
  std::ofstream(out_dir + "/timeseries.csv")
      << timeseries_csv(engine.requests(), engine.offline_commits(), rep.horizon_s);
  std::ofstream(out_dir + "/requests.csv") << requests_csv(engine.requests(), "tbt_samples.csv");
  std::ofstream(out_dir + "/tbt_samples.csv") << tbt_samples_csv(engine.requests());
  std::vector<double> r = g_ratio;
  std::sort(r.begin(), r.end());
  const double med = r.empty() ? 0 : r[r.size() / 2];
  std::printf(
      "{\"iterations\": %lld, \"drops\": %lld, \"horizon_s\": %.6f, \"offline_tok_s\": %.3f, \"p99_tbt_s\": %.6f, "
      "\"p99_ttft_s\": %.6f, \"tbt_attainment\": %.6f, \"ttft_attainment\": %.6f, \"measured_ms\": %.3f, "
      "\"predicted_ms\": %.3f, \"measured_over_predicted_median\": %.4f, \"wall_s\": %.3f, \"dry\": %s}\n",
      static_cast<long long>(g_iters), static_cast<long long>(g_drops), rep.horizon_s, rep.offline_throughput_tok_s,
      rep.p99_tbt_s, rep.p99_ttft_s, rep.tbt_attainment, rep.ttft_attainment, g_measured_ms, g_predicted_ms, med,
      wall_s, g_dry ? "true" : "false");
  return 0;
}
