/*
 * conserve_b200_kv.hpp -- C++ drop-in for coserve::KvCacheManager over the
 * C-ABI (include/conserve_b200.h).
 *
 * This is the reference-side binding a maintainer of /root/reference would
 * add: a class with exactly the public surface of
 * coserve::KvCacheManager (proj/include/coserve/kv_cache.hpp:97-173) --
 * same method names, argument meaning, return types and exception types and
 * messages -- whose state lives in the B200 engine (HBM block pool, pinned
 * host pool, D2H/H2D streams). The C-ABI status codes are rethrown as the
 * reference's exception types (SURVEY.md 8b "Errors").
 *
 * It needs the reference's value types (AllocResult, EvictStats, ReleaseStats,
 * ResumeCost, TransferJob, TransferDoneEffects, ClusterConfig, ConfigError,
 * UsecT) declared before inclusion, i.e. include "coserve/kv_cache.hpp" (or
 * the oracle/adapter_include shim, which renames the reference class and
 * aliases coserve::KvCacheManager to this one so the UNMODIFIED reference
 * Scheduler / SimEngine / tests compile against the B200 pool).
 *
 * Two modes:
 *   KvCacheManager(cluster, incremental)         bookkeeping only
 *       (CS_FLAG_HOST_ONLY: no device memory; what the reference simulator
 *       needs, since its forward is still oracle_latency);
 *   KvCacheManager(cluster, incremental, model)  the real data plane: the
 *       caller's cs_config supplies the model shape / device / sharding and
 *       the same engine handle serves cs_forward_launch (engine()).
 */
#ifndef CONSERVE_B200_KV_HPP_
#define CONSERVE_B200_KV_HPP_

#include <array>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "conserve_b200.h"

namespace conserve_b200 {

namespace detail {
inline void check(int rc) {
  if (rc == CS_OK) return;
  const std::string msg = cs_last_error();
  switch (rc) {
    case CS_ERR_LOGIC: throw std::logic_error(msg);
    case CS_ERR_INVALID: throw std::invalid_argument(msg);
    case CS_ERR_CONFIG: throw coserve::ConfigError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline coserve::TransferJob to_job(const cs_transfer_job& j) {
  coserve::TransferJob t;
  t.id = j.id;
  t.direction = j.direction == CS_D2H ? coserve::TransferDirection::kD2H : coserve::TransferDirection::kH2D;
  t.bytes = j.bytes;
  t.enqueue_time = j.enqueue_time;
  t.start_time = j.start_time;
  t.done_time = j.done_time;
  t.transfer_us = j.transfer_us;
  t.gather_us = j.gather_us;
  return t;
}

inline cs_config from_cluster(const coserve::ClusterConfig& c, bool incremental, const cs_config* model) {
  cs_config cfg;
  cs_config_default(&cfg);
  if (model) cfg = *model;
  else cfg.flags = CS_FLAG_HOST_ONLY | CS_FLAG_NO_FWD_QUARANTINE;
  cfg.num_layers = static_cast<int32_t>(c.num_layers);
  cfg.safepoint_interval_layers = static_cast<int32_t>(c.safepoint_interval_layers);
  cfg.kv_bytes_per_token = c.kv_bytes_per_token;
  cfg.gpu_kv_capacity = c.gpu_kv_capacity;
  cfg.host_kv_capacity = c.host_kv_capacity;
  cfg.d2h_bandwidth = c.d2h_bandwidth;
  cfg.h2d_bandwidth = c.h2d_bandwidth;
  cfg.gather_cost_us = c.gather_cost_us;
  cfg.page_tokens = static_cast<int32_t>(c.page_tokens);
  cfg.max_batched_tokens = c.max_batched_tokens;
  cfg.incremental = incremental ? 1 : 0;
  return cfg;
}

struct EngineDeleter {
  void operator()(cs_engine* e) const { cs_destroy(e); }
};
}  // namespace detail

/* Process-wide data-plane model for managers the reference constructs itself
 * (SimEngine builds `KvCacheManager(cluster, incremental)`, sim_engine.cpp):
 * set it before constructing the engine and those managers own a real device
 * engine of that shape (device, sharding, flags) instead of bookkeeping only.
 * last_engine() is the handle of the most recently opened one, for the
 * forward seam (cs_forward_launch) -- the live-mode host. */
inline const cs_config*& data_plane_model() {
  static const cs_config* m = nullptr;
  return m;
}
inline cs_engine*& last_engine() {
  static cs_engine* e = nullptr;
  return e;
}

class KvCacheManager {
 public:
  KvCacheManager() = default;
  KvCacheManager(const coserve::ClusterConfig& cluster, bool incremental) {
    open(cluster, incremental, data_plane_model());
  }
  KvCacheManager(const coserve::ClusterConfig& cluster, bool incremental, const cs_config& model) {
    open(cluster, incremental, &model);
  }

  /* the engine handle, for cs_forward_launch / cs_preempt_signal / ... */
  cs_engine* engine() const { return e_.get(); }

  void register_request(int64_t id, bool online) { detail::check(cs_kv_register_request(h(), id, online ? 1 : 0)); }

  coserve::AllocResult allocate(int64_t id, int64_t n_tokens, coserve::UsecT now) {
    cs_alloc_result r{};
    detail::check(cs_kv_allocate(h(), id, n_tokens, now, &r));
    coserve::AllocResult out;
    out.ok = r.ok != 0;
    out.shortfall_pages = r.shortfall_pages;
    return out;
  }
  void commit_allocations(int64_t id) { detail::check(cs_kv_commit(h(), id)); }
  void rollback_allocations(int64_t id) { detail::check(cs_kv_rollback(h(), id)); }

  coserve::EvictStats evict_request_gpu(int64_t id, coserve::UsecT now, int64_t max_pages = -1) {
    cs_evict_stats s{};
    detail::check(cs_kv_evict_request_gpu(h(), id, now, max_pages, &s));
    return stats(s);
  }
  coserve::EvictStats discard_request(int64_t id, coserve::UsecT now) {
    cs_evict_stats s{};
    detail::check(cs_kv_discard_request(h(), id, now, &s));
    return stats(s);
  }
  coserve::ReleaseStats release_offline_pages_on_demand(int64_t needed_pages, coserve::UsecT now) {
    // one discard pair per victim request at most; sized so the single
    // (mutating) call never truncates
    std::vector<int64_t> buf(2 * kMaxDiscards);
    int64_t freed = 0, n = 0;
    detail::check(
        cs_kv_release_offline_pages_on_demand(h(), needed_pages, now, &freed, buf.data(), kMaxDiscards, &n));
    if (n > kMaxDiscards) throw std::runtime_error("release_offline_pages_on_demand: discard list truncated");
    coserve::ReleaseStats r;
    r.freed_pages = freed;
    for (int64_t i = 0; i < n; ++i) r.discards.emplace_back(buf[2 * i], buf[2 * i + 1]);
    return r;
  }
  int64_t releasable_offline_pages_now() const {
    int64_t v = 0;
    detail::check(cs_kv_releasable_offline_pages_now(h(), &v));
    return v;
  }

  void stage_checkpoint(int64_t id, int64_t from_token, int64_t to_token) {
    detail::check(cs_kv_stage_checkpoint(h(), id, from_token, to_token));
  }
  std::optional<coserve::TransferJob> flush_checkpoints(coserve::UsecT now) {
    cs_transfer_job j{};
    int32_t has = 0;
    detail::check(cs_kv_flush_checkpoints(h(), now, &j, &has));
    if (!has) return std::nullopt;
    return detail::to_job(j);
  }

  coserve::ResumeCost resume_cost(int64_t id) const {
    cs_resume_cost c{};
    detail::check(cs_kv_resume_cost(h(), id, &c));
    coserve::ResumeCost r;
    r.host_only_pages = c.host_only_pages;
    r.host_only_bytes = c.host_only_bytes;
    r.discarded_tokens = c.discarded_tokens;
    return r;
  }
  bool fully_resident(int64_t id) const {
    int32_t v = 0;
    detail::check(cs_kv_fully_resident(h(), id, &v));
    return v != 0;
  }
  bool prefetch_inflight(int64_t id) const {
    int32_t v = 0;
    detail::check(cs_kv_prefetch_inflight(h(), id, &v));
    return v != 0;
  }
  std::optional<coserve::TransferJob> start_prefetch(int64_t id, coserve::UsecT now) {
    cs_transfer_job j{};
    int32_t has = 0;
    detail::check(cs_kv_start_prefetch(h(), id, now, &j, &has));
    if (!has) return std::nullopt;
    return detail::to_job(j);
  }
  int64_t recompute_chunk(int64_t id, int64_t desired, int64_t cap) const {
    int64_t v = 0;
    detail::check(cs_kv_recompute_chunk(h(), id, desired, cap, &v));
    return v;
  }

  coserve::TransferDoneEffects on_transfer_done(int64_t job_id, coserve::UsecT now) {
    cs_transfer_done d{};
    detail::check(cs_kv_on_transfer_done(h(), job_id, now, &d));
    if (d.n_became_resident > 4) throw std::runtime_error("on_transfer_done: resident list truncated");
    coserve::TransferDoneEffects r;
    r.freed_pages = d.freed_pages;
    for (int i = 0; i < d.n_became_resident; ++i) r.became_resident.push_back(d.became_resident[i]);
    return r;
  }

  void on_request_paused(int64_t id, uint64_t pause_seq) { detail::check(cs_kv_on_request_paused(h(), id, pause_seq)); }
  void on_request_active(int64_t id) { detail::check(cs_kv_on_request_active(h(), id)); }
  void release_request(int64_t id) { detail::check(cs_kv_release_request(h(), id)); }

  int64_t gpu_used_bytes() const { return st().gpu_used_bytes; }
  int64_t gpu_free_bytes() const { return st().gpu_free_bytes; }
  int64_t host_used_bytes() const { return st().host_used_bytes; }
  int64_t gpu_free_pages() const { return st().gpu_free_pages; }
  int64_t page_bytes() const { return st().page_bytes; }
  bool transfers_inflight() const { return st().transfers_inflight != 0; }
  int64_t request_gpu_pages(int64_t id) const { return info(id)[0]; }
  int64_t covered_tokens(int64_t id) const { return info(id)[1]; }
  int64_t pending_append_tokens(int64_t id) const { return info(id)[2]; }
  int64_t total_d2h_bytes() const { return st().total_d2h_bytes; }
  int64_t total_h2d_bytes() const { return st().total_h2d_bytes; }
  int64_t recompute_tagged_tokens() const { return st().recompute_tagged_tokens; }

  void audit() const { detail::check(cs_kv_audit(h())); }

  std::string page_table_json(int64_t id) const {
    size_t len = 0;
    detail::check(cs_kv_page_table_json(h(), id, nullptr, 0, &len));
    std::string s(len + 1, '\0');
    detail::check(cs_kv_page_table_json(h(), id, &s[0], s.size(), &len));
    s.resize(len);
    return s;
  }

 private:
  static constexpr int64_t kMaxDiscards = 1 << 16;
  std::shared_ptr<cs_engine> e_;

  void open(const coserve::ClusterConfig& cluster, bool incremental, const cs_config* model) {
    const cs_config cfg = detail::from_cluster(cluster, incremental, model);
    cs_engine* e = nullptr;
    detail::check(cs_create(&cfg, &e));
    e_ = std::shared_ptr<cs_engine>(e, detail::EngineDeleter{});
    last_engine() = e;
  }
  cs_engine* h() const {
    if (!e_) throw std::logic_error("KvCacheManager: default-constructed (no engine)");
    return e_.get();
  }
  static coserve::EvictStats stats(const cs_evict_stats& s) {
    coserve::EvictStats r;
    r.freed_pages = s.freed_pages;
    r.pending_pages = s.pending_pages;
    r.discarded_tokens = s.discarded_tokens;
    return r;
  }
  cs_kv_stats st() const {
    cs_kv_stats s{};
    detail::check(cs_kv_stats_get(h(), &s));
    return s;
  }
  std::array<int64_t, 3> info(int64_t id) const {
    std::array<int64_t, 3> v{};
    detail::check(cs_kv_request_info(h(), id, &v[0], &v[1], &v[2]));
    return v;
  }
};

}  // namespace conserve_b200

#endif  // CONSERVE_B200_KV_HPP_
