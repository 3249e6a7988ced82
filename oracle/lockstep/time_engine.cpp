// Times the reference's own CPU control plane -- TEST / BENCH INFRASTRUCTURE
// ONLY (bench.py's cpu_baseline leg, BASELINE.md section 3 CPU path (a)).
// Linked against the UNMODIFIED reference objects in oracle/_ref.
//
//   (1) coserve::SimEngine::run() on a RunConfig (proj/src/sim_engine.cpp:
//       337-392): wall time per dispatched iteration, single-threaded by
//       design (sim_engine.hpp:47). The engine's latency oracle stands in
//       for the forward, so this is the scheduling/bookkeeping cost only.
//   (2) coserve::KvCacheManager bookkeeping (proj/src/kv_cache.cpp): per page
//       of register -> allocate -> commit -> stage -> flush -> on_transfer_done
//       -> evict -> release over 4096-token requests.
//
// usage: time_engine <run_config.json> <iterations of that run> [min_seconds]
// prints one JSON object.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>

#include "coserve/config.hpp"
#include "coserve/kv_cache.hpp"
#include "coserve/metrics.hpp"
#include "coserve/sim_engine.hpp"

using Clock = std::chrono::steady_clock;

static double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: time_engine <run_config.json> <iterations> [min_seconds]\n";
    return 2;
  }
  const coserve::RunConfig cfg = coserve::load_run_config(argv[1]);
  const double iters = std::atof(argv[2]);
  const double min_s = argc > 3 ? std::atof(argv[3]) : 2.0;

  // (1) whole SimEngine runs, repeated until min_s of CPU work
  int runs = 0;
  double engine_s = 0;
  double offline_tok_s = 0;
  while (engine_s < min_s || runs == 0) {
    coserve::SimEngine engine(cfg);
    const auto t0 = Clock::now();
    const coserve::MetricsReport rep = engine.run();
    engine_s += seconds_since(t0);
    offline_tok_s = rep.offline_throughput_tok_s;
    ++runs;
    if (runs >= 50) break;
  }

  // (2) KvCacheManager bookkeeping per page
  coserve::ClusterConfig cl = cfg.cluster;
  cl.gpu_kv_capacity = static_cast<int64_t>(1) << 40;
  cl.host_kv_capacity = static_cast<int64_t>(1) << 42;
  int64_t pages = 0;
  double kv_s = 0;
  int64_t next_id = 0;
  while (kv_s < min_s / 2 || pages == 0) {
    coserve::KvCacheManager kv(cl, true);
    const auto t0 = Clock::now();
    coserve::UsecT now = 0;
    for (int r = 0; r < 64; ++r) {
      const int64_t id = next_id++;
      kv.register_request(id, false);
      kv.allocate(id, 4096, now);
      kv.commit_allocations(id);
      kv.stage_checkpoint(id, 0, 4096);
      auto job = kv.flush_checkpoints(now);
      if (job) kv.on_transfer_done(job->id, job->done_time);
      kv.on_request_paused(id, static_cast<uint64_t>(id));
      kv.evict_request_gpu(id, now, -1);
      kv.release_request(id);
      pages += 4096 / cl.page_tokens;
      now += 1000;
    }
    kv_s += seconds_since(t0);
  }

  std::printf(
      "{\"runs\": %d, \"engine_s\": %.6f, \"iterations_per_run\": %.0f, \"us_per_iteration\": %.4f, "
      "\"sim_offline_tok_s\": %.3f, \"kv_pages\": %lld, \"us_per_page\": %.5f, \"threads\": 1}\n",
      runs, engine_s, iters, engine_s / runs / iters * 1e6, offline_tok_s, static_cast<long long>(pages),
      kv_s / static_cast<double>(pages) * 1e6);
  return 0;
}
