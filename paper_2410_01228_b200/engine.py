"""Host-side mirror of the reference interface for the hot path.

`KvPool` mirrors coserve::KvCacheManager (/root/reference/proj/include/coserve/
kv_cache.hpp:97-173): same method names, argument meaning and error kinds
(std::logic_error -> CsLogicError, std::invalid_argument -> CsInvalidArgument,
...), so parity tests read like the reference's test_kv_cache.cpp. `Engine`
adds the forward over a BatchPlan (perf_model.hpp:12-37), the preemption flag
and iteration completion. Everything goes through the C-ABI in
libconserve_b200.so; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _ffi as F

_lib = F.load()


class CsError(RuntimeError):
    pass


class CsLogicError(CsError):
    """std::logic_error in the reference."""


class CsInvalidArgument(CsError, ValueError):
    """std::invalid_argument in the reference."""


class CsRuntimeError(CsError):
    """std::runtime_error in the reference."""


class CsConfigError(CsError):
    """coserve::ConfigError in the reference."""


class CsCudaError(CsError):
    pass


class CsPoolError(CsError):
    """Physical pool exhausted although the reference's byte accounting fit."""


_ERRORS = {
    F.CS_ERR_LOGIC: CsLogicError,
    F.CS_ERR_INVALID: CsInvalidArgument,
    F.CS_ERR_RUNTIME: CsRuntimeError,
    F.CS_ERR_CONFIG: CsConfigError,
    F.CS_ERR_CUDA: CsCudaError,
    F.CS_ERR_POOL: CsPoolError,
}


def _check(rc: int) -> None:
    if rc != F.CS_OK:
        msg = _lib.cs_last_error().decode()
        raise _ERRORS.get(rc, CsError)(msg)


def lib() -> C.CDLL:
    return _lib


@dataclass
class AllocResult:
    ok: bool
    shortfall_pages: int


@dataclass
class EvictStats:
    freed_pages: int
    pending_pages: int
    discarded_tokens: int


@dataclass
class ResumeCost:
    host_only_pages: int
    host_only_bytes: int
    discarded_tokens: int


@dataclass
class TransferJob:
    id: int
    direction: int
    bytes: int
    enqueue_time: int
    start_time: int
    done_time: int
    transfer_us: float
    gather_us: float
    moved_bytes: int


@dataclass
class TransferDoneEffects:
    became_resident: List[int]
    freed_pages: int


@dataclass
class ReleaseStats:
    freed_pages: int
    discards: List[tuple]


@dataclass
class BatchEntry:
    """coserve::BatchEntry (perf_model.hpp:15-21)."""
    request_id: int
    compute_tokens: int
    context_tokens: int
    kind: int = F.CS_PREFILL
    online: bool = False


@dataclass
class IterInfo:
    n_outputs: int
    preempted_at_layer: Optional[int]
    gpu_ms: float
    preempt_signal_to_drop_us: float
    tokens: List[int]


def model_config(preset: str = "tiny", **overrides) -> F.cs_config:
    """cs_config for a named model shape (SURVEY.md 8 model table)."""
    cfg = F.cs_config()
    _lib.cs_config_default(C.byref(cfg))
    shapes = {
        "tiny": dict(num_layers=2, hidden=256, n_heads=4, n_kv_heads=4, head_dim=64, ffn=512, vocab=1024,
                     rope_theta=10000.0),
        "llama8b": dict(num_layers=32, hidden=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336,
                        vocab=128256, rope_theta=500000.0),
        "qwen14b": dict(num_layers=48, hidden=5120, n_heads=40, n_kv_heads=8, head_dim=128, ffn=13824,
                        vocab=152064, rope_theta=1000000.0),
        "llama70b": dict(num_layers=80, hidden=8192, n_heads=64, n_kv_heads=8, head_dim=128, ffn=28672,
                         vocab=128256, rope_theta=500000.0),
    }
    for k, v in shapes[preset].items():
        setattr(cfg, k, v)
    if preset != "tiny":
        cfg.gpu_kv_capacity = 64424509440  # 60 GiB (config.hpp:37)
        cfg.host_kv_capacity = 32 << 30
        cfg.max_batched_tokens = 8192
        cfg.safepoint_interval_layers = 4
    for k, v in overrides.items():
        setattr(cfg, k, v)
    if "kv_bytes_per_token" not in overrides:
        cfg.kv_bytes_per_token = 2 * cfg.num_layers * cfg.n_kv_heads * cfg.head_dim * 2
    return cfg


class KvPool:
    """coserve::KvCacheManager on the B200 block pool."""

    def __init__(self, cfg: F.cs_config):
        self.cfg = cfg
        h = C.c_void_p()
        _check(_lib.cs_create(C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self) -> None:
        if self._h:
            _check(_lib.cs_destroy(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- KvCacheManager surface (kv_cache.hpp:100-173) ---
    def register_request(self, rid: int, online: bool) -> None:
        _check(_lib.cs_kv_register_request(self._h, rid, int(online)))

    def allocate(self, rid: int, n_tokens: int, now: int = 0) -> AllocResult:
        r = F.cs_alloc_result()
        _check(_lib.cs_kv_allocate(self._h, rid, n_tokens, now, C.byref(r)))
        return AllocResult(bool(r.ok), r.shortfall_pages)

    def commit_allocations(self, rid: int) -> None:
        _check(_lib.cs_kv_commit(self._h, rid))

    def rollback_allocations(self, rid: int) -> None:
        _check(_lib.cs_kv_rollback(self._h, rid))

    def evict_request_gpu(self, rid: int, now: int = 0, max_pages: int = -1) -> EvictStats:
        s = F.cs_evict_stats()
        _check(_lib.cs_kv_evict_request_gpu(self._h, rid, now, max_pages, C.byref(s)))
        return EvictStats(s.freed_pages, s.pending_pages, s.discarded_tokens)

    def discard_request(self, rid: int, now: int = 0) -> EvictStats:
        s = F.cs_evict_stats()
        _check(_lib.cs_kv_discard_request(self._h, rid, now, C.byref(s)))
        return EvictStats(s.freed_pages, s.pending_pages, s.discarded_tokens)

    def release_offline_pages_on_demand(self, needed_pages: int, now: int = 0) -> ReleaseStats:
        freed = C.c_int64()
        n = C.c_int64()
        buf = (C.c_int64 * 2048)()
        _check(_lib.cs_kv_release_offline_pages_on_demand(self._h, needed_pages, now, C.byref(freed), buf, 1024,
                                                          C.byref(n)))
        return ReleaseStats(freed.value, [(buf[2 * i], buf[2 * i + 1]) for i in range(min(n.value, 1024))])

    def releasable_offline_pages_now(self) -> int:
        v = C.c_int64()
        _check(_lib.cs_kv_releasable_offline_pages_now(self._h, C.byref(v)))
        return v.value

    def stage_checkpoint(self, rid: int, from_token: int, to_token: int) -> None:
        _check(_lib.cs_kv_stage_checkpoint(self._h, rid, from_token, to_token))

    @staticmethod
    def _job(j: F.cs_transfer_job) -> TransferJob:
        return TransferJob(j.id, j.direction, j.bytes, j.enqueue_time, j.start_time, j.done_time, j.transfer_us,
                           j.gather_us, j.moved_bytes)

    def flush_checkpoints(self, now: int = 0) -> Optional[TransferJob]:
        j = F.cs_transfer_job()
        has = C.c_int32()
        _check(_lib.cs_kv_flush_checkpoints(self._h, now, C.byref(j), C.byref(has)))
        return self._job(j) if has.value else None

    def resume_cost(self, rid: int) -> ResumeCost:
        c = F.cs_resume_cost()
        _check(_lib.cs_kv_resume_cost(self._h, rid, C.byref(c)))
        return ResumeCost(c.host_only_pages, c.host_only_bytes, c.discarded_tokens)

    def fully_resident(self, rid: int) -> bool:
        v = C.c_int32()
        _check(_lib.cs_kv_fully_resident(self._h, rid, C.byref(v)))
        return bool(v.value)

    def prefetch_inflight(self, rid: int) -> bool:
        v = C.c_int32()
        _check(_lib.cs_kv_prefetch_inflight(self._h, rid, C.byref(v)))
        return bool(v.value)

    def start_prefetch(self, rid: int, now: int = 0) -> Optional[TransferJob]:
        j = F.cs_transfer_job()
        has = C.c_int32()
        _check(_lib.cs_kv_start_prefetch(self._h, rid, now, C.byref(j), C.byref(has)))
        return self._job(j) if has.value else None

    def recompute_chunk(self, rid: int, desired: int, cap: int) -> int:
        v = C.c_int64()
        _check(_lib.cs_kv_recompute_chunk(self._h, rid, desired, cap, C.byref(v)))
        return v.value

    def on_transfer_done(self, job_id: int, now: int = 0) -> TransferDoneEffects:
        d = F.cs_transfer_done()
        _check(_lib.cs_kv_on_transfer_done(self._h, job_id, now, C.byref(d)))
        return TransferDoneEffects([d.became_resident[i] for i in range(min(d.n_became_resident, 4))],
                                   d.freed_pages)

    def job_poll(self, job_id: int):
        """(done, device ms) of a transfer job's real copy (cs_job_poll)."""
        d, ms = C.c_int32(), C.c_double()
        _check(_lib.cs_job_poll(self._h, job_id, C.byref(d), C.byref(ms)))
        return bool(d.value), ms.value

    def job_wait(self, job_id: int) -> float:
        """Blocks until the job's device copy finished; returns its device ms."""
        ms = C.c_double()
        _check(_lib.cs_job_wait(self._h, job_id, C.byref(ms)))
        return ms.value

    def on_request_paused(self, rid: int, pause_seq: int) -> None:
        _check(_lib.cs_kv_on_request_paused(self._h, rid, pause_seq))

    def on_request_active(self, rid: int) -> None:
        _check(_lib.cs_kv_on_request_active(self._h, rid))

    def release_request(self, rid: int) -> None:
        _check(_lib.cs_kv_release_request(self._h, rid))

    def note_written(self, rid: int, w0: int, w1: int) -> None:
        _check(_lib.cs_kv_note_written(self._h, rid, w0, w1))

    def stats(self) -> F.cs_kv_stats:
        s = F.cs_kv_stats()
        _check(_lib.cs_kv_stats_get(self._h, C.byref(s)))
        return s

    def gpu_used_bytes(self) -> int:
        return self.stats().gpu_used_bytes

    def gpu_free_bytes(self) -> int:
        return self.stats().gpu_free_bytes

    def host_used_bytes(self) -> int:
        return self.stats().host_used_bytes

    def gpu_free_pages(self) -> int:
        return self.stats().gpu_free_pages

    def total_d2h_bytes(self) -> int:
        return self.stats().total_d2h_bytes

    def total_h2d_bytes(self) -> int:
        return self.stats().total_h2d_bytes

    def recompute_tagged_tokens(self) -> int:
        return self.stats().recompute_tagged_tokens

    def transfers_inflight(self) -> bool:
        return bool(self.stats().transfers_inflight)

    def _info(self, rid: int):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib.cs_kv_request_info(self._h, rid, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def request_gpu_pages(self, rid: int) -> int:
        return self._info(rid)[0]

    def covered_tokens(self, rid: int) -> int:
        return self._info(rid)[1]

    def pending_append_tokens(self, rid: int) -> int:
        return self._info(rid)[2]

    def audit(self) -> None:
        _check(_lib.cs_kv_audit(self._h))

    def page_table_json(self, rid: int) -> str:
        n = C.c_size_t()
        _check(_lib.cs_kv_page_table_json(self._h, rid, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(_lib.cs_kv_page_table_json(self._h, rid, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def block_table(self, rid: int):
        n = C.c_int64()
        _check(_lib.cs_kv_block_table(self._h, rid, None, None, 0, C.byref(n)))
        blocks = (C.c_int32 * max(n.value, 1))()
        slots = (C.c_int32 * max(n.value, 1))()
        _check(_lib.cs_kv_block_table(self._h, rid, blocks, slots, n.value, C.byref(n)))
        return list(blocks[: n.value]), list(slots[: n.value])


class Engine(KvPool):
    """KvPool plus the L-layer forward, the preemption flag and debug reads."""

    def forward_launch(self, entries: Sequence[BatchEntry], epoch: int) -> None:
        arr = (F.cs_batch_entry * len(entries))()
        for i, e in enumerate(entries):
            arr[i] = F.cs_batch_entry(e.request_id, e.compute_tokens, e.context_tokens, e.kind, int(e.online))
        _check(_lib.cs_forward_launch(self._h, arr, len(entries), epoch))

    def preempt_signal(self, epoch: int) -> None:
        _check(_lib.cs_preempt_signal(self._h, epoch))

    def iter_poll(self) -> bool:
        d = C.c_int32()
        _check(_lib.cs_iter_poll(self._h, C.byref(d)))
        return bool(d.value)

    def iter_progress(self) -> int:
        """Layer the in-flight instrumented forward has entered (-1: none)."""
        v = C.c_int32()
        _check(_lib.cs_iter_progress(self._h, C.byref(v)))
        return int(v.value)

    def set_kernel_timing(self, on: bool) -> None:
        _check(_lib.cs_set_kernel_timing(self._h, 1 if on else 0))

    def kernel_timing(self, cls: int) -> F.cs_ktime:
        """(launches, ms, algorithmic units) of one kernel class (CS_KT_*)."""
        t = F.cs_ktime()
        _check(_lib.cs_kernel_timing(self._h, cls, C.byref(t)))
        return t

    def iter_wait(self, want_logits: bool = False):
        info = F.cs_iter_info()
        cap = 4096
        toks = (C.c_int32 * cap)()
        logits = None
        lp = None
        if want_logits:
            rows = self.cfg.max_entries if self.cfg.max_entries > 0 else 1024
            logits = np.zeros((rows, self.cfg.vocab), dtype=np.float32)
            lp = logits.ctypes.data_as(C.POINTER(C.c_float))
        _check(_lib.cs_iter_wait(self._h, C.byref(info), toks, cap, lp))
        out = IterInfo(info.n_outputs, info.preempted_at_layer if info.preempted_at_layer >= 0 else None,
                       info.gpu_ms, info.preempt_signal_to_drop_us, list(toks[: info.n_outputs]))
        if want_logits:
            return out, logits[: info.n_outputs].copy()
        return out

    def forward(self, entries: Sequence[BatchEntry], epoch: int = 1, want_logits: bool = False):
        self.forward_launch(entries, epoch)
        return self.iter_wait(want_logits)

    def sync(self) -> None:
        _check(_lib.cs_sync(self._h))

    def block_bytes(self) -> int:
        c = self.cfg
        return c.num_layers * 2 * (c.n_kv_heads // c.tp_size) * 16 * c.head_dim * 2

    def read_block(self, block: int) -> np.ndarray:
        n = self.block_bytes()
        buf = np.empty(n // 2, dtype=np.uint16)
        _check(_lib.cs_debug_read_block(self._h, block, buf.ctypes.data, n))
        return buf

    def write_block(self, block: int, data: np.ndarray) -> None:
        data = np.ascontiguousarray(data, dtype=np.uint16)
        _check(_lib.cs_debug_write_block(self._h, block, data.ctypes.data, data.nbytes))

    def read_host_slot(self, slot: int) -> np.ndarray:
        n = self.block_bytes()
        buf = np.empty(n // 2, dtype=np.uint16)
        _check(_lib.cs_debug_read_host_slot(self._h, slot, buf.ctypes.data, n))
        return buf

    def fill_pool(self, seed: int) -> None:
        _check(_lib.cs_debug_fill_pool(self._h, seed))

    def read_activation(self, which: int, rows: int, cols: int) -> np.ndarray:
        buf = np.empty(rows * cols, dtype=np.uint16)
        _check(_lib.cs_debug_read_activation(self._h, which, buf.ctypes.data, buf.nbytes))
        return buf.reshape(rows, cols)

    def read_weight(self, layer: int, which: int) -> np.ndarray:
        need = C.c_size_t()
        _check(_lib.cs_debug_read_weight(self._h, layer, which, None, 0, C.byref(need)))
        buf = np.empty(need.value // 2, dtype=np.uint16)
        _check(_lib.cs_debug_read_weight(self._h, layer, which, buf.ctypes.data, need.value, C.byref(need)))
        return buf
