"""ctypes mirror of include/conserve_b200.h (the C-ABI boundary).

The product path is the shared library libconserve_b200.so built from
paper_2410_01228_b200/csrc for sm_100a; there is no Python or CPU fallback:
importing this module fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CS_LIB_PATH") or os.path.join(_HERE, "libconserve_b200.so")  # override: experiments only

CS_OK = 0
CS_ERR_LOGIC = -1
CS_ERR_INVALID = -2
CS_ERR_RUNTIME = -3
CS_ERR_CONFIG = -4
CS_ERR_CUDA = -5
CS_ERR_POOL = -6
CS_ERR_NOT_READY = -7

CS_FLAG_NO_MODEL = 1 << 0
CS_FLAG_SYNC_DEBUG = 1 << 3
CS_FLAG_HOST_ONLY = 1 << 4
CS_FLAG_NO_FWD_QUARANTINE = 1 << 5

CS_D2H = 0
CS_H2D = 1
CS_PREFILL = 0
CS_DECODE = 1
CS_RECOMPUTE = 2


class cs_config(C.Structure):
    _fields_ = [
        ("num_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
        ("vocab", C.c_int32), ("rope_theta", C.c_float), ("rms_eps", C.c_float),
        ("weight_seed", C.c_uint64), ("token_seed", C.c_uint64),
        ("kv_bytes_per_token", C.c_int64), ("gpu_kv_capacity", C.c_int64),
        ("host_kv_capacity", C.c_int64), ("d2h_bandwidth", C.c_double),
        ("h2d_bandwidth", C.c_double), ("gather_cost_us", C.c_double),
        ("page_tokens", C.c_int32), ("safepoint_interval_layers", C.c_int32),
        ("max_batched_tokens", C.c_int64), ("incremental", C.c_int32),
        ("instrumented", C.c_int32), ("extra_blocks", C.c_int64),
        ("extra_host_slots", C.c_int64), ("max_entries", C.c_int32),
        ("layer_lookahead", C.c_int32), ("tp_rank", C.c_int32), ("tp_size", C.c_int32),
        ("device", C.c_int32), ("flags", C.c_int32),
    ]


class cs_alloc_result(C.Structure):
    _fields_ = [("ok", C.c_int32), ("shortfall_pages", C.c_int64)]


class cs_evict_stats(C.Structure):
    _fields_ = [("freed_pages", C.c_int64), ("pending_pages", C.c_int64), ("discarded_tokens", C.c_int64)]


class cs_resume_cost(C.Structure):
    _fields_ = [("host_only_pages", C.c_int64), ("host_only_bytes", C.c_int64), ("discarded_tokens", C.c_int64)]


class cs_transfer_job(C.Structure):
    _fields_ = [
        ("id", C.c_int64), ("direction", C.c_int32), ("bytes", C.c_int64),
        ("enqueue_time", C.c_int64), ("start_time", C.c_int64), ("done_time", C.c_int64),
        ("transfer_us", C.c_double), ("gather_us", C.c_double), ("moved_bytes", C.c_int64),
    ]


class cs_transfer_done(C.Structure):
    _fields_ = [("freed_pages", C.c_int64), ("n_became_resident", C.c_int32),
                ("became_resident", C.c_int64 * 4)]


class cs_kv_stats(C.Structure):
    _fields_ = [
        ("gpu_used_bytes", C.c_int64), ("gpu_free_bytes", C.c_int64), ("host_used_bytes", C.c_int64),
        ("gpu_free_pages", C.c_int64), ("page_bytes", C.c_int64), ("total_d2h_bytes", C.c_int64),
        ("total_h2d_bytes", C.c_int64), ("recompute_tagged_tokens", C.c_int64),
        ("transfers_inflight", C.c_int32), ("n_blocks", C.c_int64), ("free_blocks", C.c_int64),
        ("quarantined_blocks", C.c_int64), ("n_host_slots", C.c_int64), ("free_host_slots", C.c_int64),
        ("moved_d2h_bytes", C.c_int64), ("moved_h2d_bytes", C.c_int64), ("nonresident_reads", C.c_int64),
        ("moved_d2h_ms", C.c_double), ("moved_h2d_ms", C.c_double), ("kernel_launches", C.c_int64),
        ("host_lru_evicted_pages", C.c_int64), ("unbacked_reads", C.c_int64), ("host_numa_node", C.c_int32),
    ]


class cs_batch_entry(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("compute_tokens", C.c_int64), ("context_tokens", C.c_int64),
                ("kind", C.c_int32), ("online", C.c_int32)]


class cs_ktime(C.Structure):
    _fields_ = [("launches", C.c_int64), ("ms", C.c_double), ("units", C.c_double)]


CS_KT_K8, CS_KT_K2, CS_KT_K1, CS_KT_LIB, CS_KT_GRAPH = 0, 1, 2, 3, 4


class cs_iter_info(C.Structure):
    _fields_ = [("n_outputs", C.c_int32), ("preempted_at_layer", C.c_int32), ("n_entries_after", C.c_int32),
                ("done", C.c_int32), ("gpu_ms", C.c_double), ("preempt_signal_to_drop_us", C.c_double),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("gemm_trunc_layer", C.c_int32),
                ("pre_drop_layer_us", C.c_double)]


class cs_replay_stats(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("mismatches", C.c_int64), ("first_mismatch_op", C.c_int64),
                ("wall_ms", C.c_double), ("op_ms", C.c_double * 20)]


# (name, argtypes) for every export declared in include/conserve_b200.h
P = C.POINTER
E = C.c_void_p
EXPORTS = {
    "cs_last_error": ([], C.c_char_p),
    "cs_version": ([], C.c_char_p),
    "cs_config_default": ([P(cs_config)], None),
    "cs_create": ([P(cs_config), P(E)], C.c_int),
    "cs_destroy": ([E], C.c_int),
    "cs_nccl_unique_id": ([P(C.c_uint8)], C.c_int),
    "cs_nccl_init": ([E, P(C.c_uint8)], C.c_int),
    "cs_tp_exchange_ptr": ([E, P(C.c_void_p)], C.c_int),
    "cs_tp_exchange_ipc_handle": ([E, P(C.c_uint8)], C.c_int),
    "cs_tp_attach_peers": ([E, P(C.c_void_p), C.c_int32, C.c_int32], C.c_int),
    "cs_tp_attach_ipc": ([E, P(C.c_uint8), C.c_int32], C.c_int),
    "cs_kv_register_request": ([E, C.c_int64, C.c_int32], C.c_int),
    "cs_kv_allocate": ([E, C.c_int64, C.c_int64, C.c_int64, P(cs_alloc_result)], C.c_int),
    "cs_kv_commit": ([E, C.c_int64], C.c_int),
    "cs_kv_rollback": ([E, C.c_int64], C.c_int),
    "cs_kv_evict_request_gpu": ([E, C.c_int64, C.c_int64, C.c_int64, P(cs_evict_stats)], C.c_int),
    "cs_kv_discard_request": ([E, C.c_int64, C.c_int64, P(cs_evict_stats)], C.c_int),
    "cs_kv_release_offline_pages_on_demand": (
        [E, C.c_int64, C.c_int64, P(C.c_int64), P(C.c_int64), C.c_int64, P(C.c_int64)], C.c_int),
    "cs_kv_releasable_offline_pages_now": ([E, P(C.c_int64)], C.c_int),
    "cs_kv_stage_checkpoint": ([E, C.c_int64, C.c_int64, C.c_int64], C.c_int),
    "cs_kv_flush_checkpoints": ([E, C.c_int64, P(cs_transfer_job), P(C.c_int32)], C.c_int),
    "cs_kv_resume_cost": ([E, C.c_int64, P(cs_resume_cost)], C.c_int),
    "cs_kv_fully_resident": ([E, C.c_int64, P(C.c_int32)], C.c_int),
    "cs_kv_prefetch_inflight": ([E, C.c_int64, P(C.c_int32)], C.c_int),
    "cs_kv_start_prefetch": ([E, C.c_int64, C.c_int64, P(cs_transfer_job), P(C.c_int32)], C.c_int),
    "cs_kv_recompute_chunk": ([E, C.c_int64, C.c_int64, C.c_int64, P(C.c_int64)], C.c_int),
    "cs_kv_on_transfer_done": ([E, C.c_int64, C.c_int64, P(cs_transfer_done)], C.c_int),
    "cs_job_poll": ([E, C.c_int64, P(C.c_int32), P(C.c_double)], C.c_int),
    "cs_job_wait": ([E, C.c_int64, P(C.c_double)], C.c_int),
    "cs_kv_on_request_paused": ([E, C.c_int64, C.c_uint64], C.c_int),
    "cs_kv_on_request_active": ([E, C.c_int64], C.c_int),
    "cs_kv_release_request": ([E, C.c_int64], C.c_int),
    "cs_kv_note_written": ([E, C.c_int64, C.c_int64, C.c_int64], C.c_int),
    "cs_kv_stats_get": ([E, P(cs_kv_stats)], C.c_int),
    "cs_kv_request_info": ([E, C.c_int64, P(C.c_int64), P(C.c_int64), P(C.c_int64)], C.c_int),
    "cs_kv_audit": ([E], C.c_int),
    "cs_kv_page_table_json": ([E, C.c_int64, C.c_char_p, C.c_size_t, P(C.c_size_t)], C.c_int),
    "cs_kv_block_table": ([E, C.c_int64, P(C.c_int32), P(C.c_int32), C.c_int64, P(C.c_int64)], C.c_int),
    "cs_forward_launch": ([E, P(cs_batch_entry), C.c_int32, C.c_uint64], C.c_int),
    "cs_preempt_signal": ([E, C.c_uint64], C.c_int),
    "cs_iter_wait": ([E, P(cs_iter_info), P(C.c_int32), C.c_int32, P(C.c_float)], C.c_int),
    "cs_iter_poll": ([E, P(C.c_int32)], C.c_int),
    "cs_iter_progress": ([E, P(C.c_int32)], C.c_int),
    "cs_iter_elapsed": ([E, P(C.c_double)], C.c_int),
    "cs_iter_retro_drop": ([E, C.c_int32], C.c_int),
    "cs_set_kernel_timing": ([E, C.c_int32], C.c_int),
    "cs_kernel_timing": ([E, C.c_int32, P(cs_ktime)], C.c_int),
    "cs_debug_read_block": ([E, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "cs_debug_write_block": ([E, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "cs_debug_read_host_slot": ([E, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "cs_debug_fill_pool": ([E, C.c_uint64], C.c_int),
    "cs_debug_read_activation": ([E, C.c_int32, C.c_void_p, C.c_size_t], C.c_int),
    "cs_debug_read_weight": ([E, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, P(C.c_size_t)], C.c_int),
    "cs_sync": ([E], C.c_int),
    "cs_set_dry": ([E, C.c_int32], C.c_int),
    "cs_bench_attention": ([E, P(cs_batch_entry), C.c_int32, C.c_int32, P(C.c_double), P(C.c_int64),
                            P(C.c_int64)], C.c_int),
    "cs_bench_gemm": ([E, C.c_int32, C.c_int32, C.c_int32, C.c_int32, P(C.c_double), P(C.c_double),
                       P(C.c_double), P(C.c_double)], C.c_int),
    "cs_replay_run": ([E, P(C.c_int64), C.c_int64, C.c_int64, P(C.c_int64), P(C.c_double), P(C.c_double),
                       P(C.c_int32), P(C.c_double), P(C.c_double), P(C.c_int32), P(C.c_int64), P(C.c_int64),
                       P(cs_replay_stats)], C.c_int),
    "cs_token_id": ([C.c_uint64, C.c_int64, C.c_int64, C.c_int32], C.c_int32),
    "cs_hash_uniform": ([C.c_uint64, C.c_uint64, C.c_uint64], C.c_float),
}


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2410_01228_b200/csrc). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (argtypes, restype) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.argtypes = argtypes
        fn.restype = restype
    return lib
