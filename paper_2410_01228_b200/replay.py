"""Lockstep replay of a reference call log through the C-ABI.

A call log (tests/golden/<scenario>/calls.jsonl.gz, produced by the UNMODIFIED
reference SimEngine under oracle/lockstep/recorder.cpp) is the exact sequence
of hot-path calls the reference engine makes: KvCacheManager mutations with
their results, dispatched BatchPlans, preemption signals/drops and iteration
ends. This module encodes it into a flat op array and hands windows of it to
cs_replay_run (csrc/replay.cpp), which issues the same calls into the B200
engine and counts any result that differs from the reference's.
"""
from __future__ import annotations

import ctypes as C
import gzip
import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

from . import _ffi as F
from .engine import Engine, _check, lib

OPC = {"register": 0, "allocate": 1, "commit": 2, "rollback": 3, "evict": 4, "discard": 5,
       "release_on_demand": 6, "stage": 7, "flush": 8, "prefetch": 9, "done": 10, "paused": 11, "active": 12,
       "release": 13, "dispatch": 14, "signal": 15, "iter_end": 16, "build": 17, "drop": 18, "pt": 19}


@dataclass
class Trace:
    config: dict
    ops: np.ndarray              # [n_ops, 8] int64
    plans: np.ndarray            # [n_entries, 5] int64 (id, P, C, kind, online)
    bounds: np.ndarray           # [n_iter + 1] op index boundaries
    plan_of: List[np.ndarray]    # dispatched plan per iteration
    end_plan_of: List[np.ndarray]  # plan at iteration end (residual after a drop)
    end_now: np.ndarray          # reference iteration-end time (us)
    dropped: np.ndarray          # reference drop layer per iteration (-1)
    requests: Dict[int, dict] = field(default_factory=dict)
    audit: Optional[str] = None  # the reference's audit() verdict on its final state

    @property
    def n_iter(self) -> int:
        return len(self.plan_of)


def _job(j):
    if j is None:
        return 0, 0, 0, 0
    return 1, j["id"], j["bytes"], j["done"]


def load(calls_path: str, requests_path: Optional[str] = None) -> Trace:
    ops: List[List[int]] = []
    plans: List[List[int]] = []
    plan_of, end_plan_of, end_now, dropped = [], [], [], []
    config = {}
    audit = None
    opener = gzip.open if calls_path.endswith(".gz") else open
    with opener(calls_path, "rt") as f:
        for line in f:
            d = json.loads(line)
            if "config" in d:
                config = d["config"]
                continue
            op = d.get("op")
            if op == "audit":
                audit = d["result"]
                continue
            if op is None or op == "completed":
                continue
            c = OPC[op]
            r = [c, 0, 0, 0, 0, 0, 0, 0]
            if op == "register":
                r[1:3] = [d["id"], d["online"]]
            elif op == "allocate":
                r[1:6] = [d["id"], d["n"], d["now"], d["ok"], d["short"]]
            elif op in ("commit", "rollback", "active", "release"):
                r[1] = d["id"]
            elif op == "evict":
                r[1:7] = [d["id"], d["now"], d["max"], d["freed"], d["pending"], d["discarded"]]
            elif op == "discard":
                r[1:5] = [d["id"], d["now"], d["freed"], d["discarded"]]
            elif op == "release_on_demand":
                r[1:4] = [d["need"], d["now"], d["freed"]]
            elif op == "stage":
                r[1:4] = [d["id"], d["from"], d["to"]]
            elif op == "flush":
                r[1] = d["now"]
                r[2:6] = list(_job(d["job"]))
            elif op == "prefetch":
                r[1] = d["now"]
                r[2:6] = list(_job(d["job"]))
                r[7] = d["id"]
            elif op == "done":
                r[1:4] = [d["job"], d["now"], d["freed"]]
            elif op == "paused":
                r[1:3] = [d["id"], d["seq"]]
            elif op == "dispatch":
                r[1:3] = [len(plans), len(d["plan"])]
                plans.extend(d["plan"])
                plan_of.append(np.array(d["plan"], dtype=np.int64).reshape(-1, 5))
                end_plan_of.append(None)
                end_now.append(-1)
                dropped.append(-1)
            elif op == "iter_end":
                r[1] = d["now"]
                end_plan_of[-1] = np.array(d["plan"], dtype=np.int64).reshape(-1, 5)
                end_now[-1] = d["now"]
            elif op == "drop":
                r[1] = d["layer"]
                dropped[-1] = d["layer"]
            elif op == "build":
                r[1] = d["now"]
            elif op == "pt":
                h = int(d["hash"], 16)
                r[1:4] = [d["n"], h - (1 << 64) if h >= (1 << 63) else h, 1]
            ops.append(r)
    ops_a = np.array(ops, dtype=np.int64).reshape(-1, 8)
    disp = np.nonzero(ops_a[:, 0] == OPC["dispatch"])[0]
    # arm the preemption signal only for iterations the reference dropped,
    # with the layer it dropped at (1 + layer; 0 = no drop)
    for k, i in enumerate(disp):
        ops_a[i, 3] = 1 + dropped[k] if dropped[k] >= 0 else 0
    bounds = np.concatenate([[0], disp[1:], [len(ops_a)]]).astype(np.int64)
    tr = Trace(config, ops_a, np.array(plans, dtype=np.int64).reshape(-1, 5), bounds, plan_of, end_plan_of,
               np.array(end_now, dtype=np.int64), np.array(dropped, dtype=np.int32), audit=audit)
    if requests_path:
        opener = gzip.open if requests_path.endswith(".gz") else open
        with opener(requests_path, "rt") as f:
            for line in f:
                r = json.loads(line)
                tr.requests[r["id"]] = r
    return tr


@dataclass
class WindowResult:
    iterations: int
    mismatches: int
    first_mismatch_op: int
    wall_ms: float
    op_ms: np.ndarray  # host ms per replayed op kind (OPC codes)
    gpu_ms: np.ndarray
    wall_end_ms: np.ndarray
    dropped_layer: np.ndarray
    drop_latency_us: np.ndarray
    pre_drop_layer_us: np.ndarray
    gemm_trunc_layer: np.ndarray
    h2d_bytes: np.ndarray
    d2h_bytes: np.ndarray


def run(eng: Engine, tr: Trace, it_begin: int, it_end: int, dry: bool = False,
        check_page_tables: bool = False) -> WindowResult:
    """Executes the ops of iterations [it_begin, it_end) (see bounds).
    check_page_tables compares the logical page table of every live request
    with the reference's digest at every build (host work: off in benches)."""
    n = it_end - it_begin
    arrs = dict(gpu_ms=np.zeros(n), wall_end_ms=np.zeros(n), dropped_layer=np.full(n, -1, np.int32),
                drop_latency_us=np.zeros(n), pre_drop_layer_us=np.zeros(n), gemm_trunc_layer=np.full(n, -1, np.int32),
                h2d_bytes=np.zeros(n, np.int64), d2h_bytes=np.zeros(n, np.int64))
    ptr = {k: v.ctypes.data_as(C.POINTER({np.float64: C.c_double, np.int32: C.c_int32,
                                          np.int64: C.c_int64}[v.dtype.type])) for k, v in arrs.items()}
    st = F.cs_replay_stats()
    _check(lib().cs_set_dry(eng._h, 1 if dry else 0))
    ops = np.array(tr.ops)
    ops[ops[:, 0] == OPC["pt"], 3] = 1 if check_page_tables else 0
    plans = np.ascontiguousarray(tr.plans) if len(tr.plans) else np.zeros((1, 5), np.int64)
    rc = lib().cs_replay_run(eng._h, ops.ctypes.data_as(C.POINTER(C.c_int64)), int(tr.bounds[it_begin]),
                             int(tr.bounds[it_end]), plans.ctypes.data_as(C.POINTER(C.c_int64)),
                             ptr["gpu_ms"], ptr["wall_end_ms"], ptr["dropped_layer"], ptr["drop_latency_us"],
                             ptr["pre_drop_layer_us"], ptr["gemm_trunc_layer"], ptr["h2d_bytes"], ptr["d2h_bytes"], C.byref(st))
    if rc != F.CS_OK:
        msg = lib().cs_last_error().decode()
        raise RuntimeError(f"replay failed at op {st.first_mismatch_op} "
                           f"({tr.ops[st.first_mismatch_op].tolist()}): rc={rc} {msg}")
    _check(lib().cs_set_dry(eng._h, 0))
    return WindowResult(st.iterations, st.mismatches, st.first_mismatch_op, st.wall_ms, np.array(st.op_ms[:]), **arrs)


def engine_config_for(tr: Trace, preset: str, **overrides) -> F.cs_config:
    """Engine config whose cluster fields mirror the recorded RunConfig."""
    from .engine import model_config
    cl = tr.config["cluster"]
    pol = tr.config["policy"]
    cfg = model_config(preset, **overrides)
    cfg.num_layers = cl["num_layers"] if preset == "tiny" else cfg.num_layers
    cfg.kv_bytes_per_token = 2 * cfg.num_layers * cfg.n_kv_heads * cfg.head_dim * 2
    assert cfg.kv_bytes_per_token == cl["kv_bytes_per_token"], "trace KV size does not match the model shape"
    cfg.gpu_kv_capacity = cl["gpu_kv_capacity"]
    cfg.host_kv_capacity = cl["host_kv_capacity"]
    cfg.d2h_bandwidth = cl["d2h_bandwidth"]
    cfg.h2d_bandwidth = cl["h2d_bandwidth"]
    cfg.gather_cost_us = cl["gather_cost_us"]
    cfg.safepoint_interval_layers = cl["safepoint_interval_layers"]
    cfg.max_batched_tokens = cl["max_batched_tokens"]
    cfg.incremental = 1 if (pol["kind"] == "conserve" and pol["incremental_kv"]) else 0
    cfg.instrumented = 1 if (pol["kind"] == "conserve" and pol["layerwise_preemption"]) else 0
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


def token_progress(tr: Trace, k: int):
    """Useful tokens committed by iteration k (SimEngine::handle_iteration_end
    delta, sim_engine.cpp:190-199): per entry of the end plan, prefill adds P
    (+1 first token when the chunk completes the prompt), decode adds 1,
    recompute adds 0. Returns (offline, online, [(rid, n_new_output_tokens)])."""
    off = on = 0
    outs = []
    plan = tr.end_plan_of[k]
    if plan is None:
        return 0, 0, outs
    for rid, P, Cc, kind, online in plan:
        rq = tr.requests.get(int(rid))
        if kind == 0:
            got = int(P)
            if rq is not None and Cc + P >= rq["in"]:
                got += 1
                outs.append((int(rid), 1))
        elif kind == 1:
            got = 1
            outs.append((int(rid), 1))
        else:
            got = 0
        if online:
            on += got
        else:
            off += got
    return off, on, outs
