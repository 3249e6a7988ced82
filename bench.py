#!/usr/bin/env python
"""bench.py -- ConServe co-serving hot path on B200 (BASELINE.json configs[1]).

Workload (headline, `--workload llama8b`): tests/golden/llama8b_b200_spike, the
UNMODIFIED reference SimEngine's ConServe run recorded by
oracle/lockstep/recorder.cpp on a Llama-3.1-8B shape: the reference scheduler
planning on its own fit of the B200-measured latency grid, a bursty online
trace with a load spike (2 -> 8 req/s) against a 96-request offline backlog,
TTFT SLO 150 ms / TBT SLO 100 ms, a 32 GiB KV pool and a safepoint every layer,
so the run preempts layer-wise (7 drops), evicts, checkpoints and restores.
Synthetic random-init weights, teacher-forced synthetic token ids.

A STEP is one contiguous 1/K slice of the run: the first W iterations are
the warm-up steps (untimed), iterations [W, n) are cut into K slices and each
slice is replayed through the C-ABI (csrc/replay.cpp): the reference's
KvCacheManager calls, the 32-layer bf16 forward of every dispatched plan
(paged decode + prefill attention over the HBM block pool, tcgen05 GEMMs),
the preemption flag stored when the device reaches the layer the reference's
Alg. 1 fired in, and the incremental KV checkpoint / restore kernels.

  value  = offline tokens committed in the timed steps / summed device time
           of their forwards (plan metadata already resident)
  e2e    = the same tokens / wall time of the replay through the C-ABI with
           HOST plan buffers (H2D plan metadata + D2H sampled ids per iteration)
  roofline = the timed window's dominant hand-written kernel, algorithmic
           work of its launches / their CUDA-event time on the compute stream,
           measured over the timed region; the other kernel classes beside it

`--impl reference` times the reference path's CPU implementation on the host
cores. The reference computes no forward (its GPU is oracle_latency), so the
CPU arm is the fp32 CPU restatement of the forward (oracle/numeric.py,
"kind": "port") over a bounded sample of every step's slice, plus the
reference's own SimEngine control plane (oracle/_ref/time_engine) per
iteration. It never imports the product package.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "offline tok/s at online P99 TPOT SLO; preempt latency; KV ckpt GB/s"
UNIT = "tok/s"

WORKLOADS = {
    "llama8b": ("llama8b_b200_spike", "llama8b",
                "llama8b_b200_spike: Llama-3.1-8B shape bf16 on 1 B200 per rank, the reference's ConServe co-serving "
                "run (online Gamma 2 req/s with a 4 s spike to 8 req/s, 4096/256, 30 s, against a 96-request "
                "offline backlog; TTFT SLO 150 ms, TBT SLO 100 ms; chunked prefill, 8192-token batches, 32 GiB KV "
                "pool, safepoint every layer; 7 layer-wise drops, eviction, checkpoint and restore), scheduled with "
                "the reference's own fit of the B200-measured latency grid (profiles/b200_fit.json)"),
    "config1": ("config1", "tiny",
                "config1: the reference's tiny CPU co-serving trace (2 layers, SURVEY.md 8d config 1) -- a "
                "plumbing-size run, not a benchmark"),
    "llama8b_kv60": ("llama8b_b200_kv60", "llama8b",
                     "llama8b_b200_kv60: the same B200 schedule family on the reference's default 60 GiB KV pool "
                     "(online Gamma 3 req/s cv 2, 64-request offline backlog with replenish, no restores)"),
    "llama8b_pool24": ("llama8b_b200", "llama8b",
                       "llama8b_b200: online Gamma 3 req/s cv 2 + 64-request offline backlog on a 24 GiB KV pool "
                       "(eviction, checkpoint and restore)"),
    "qwen14b": ("qwen14b_b200", "qwen14b",
                "qwen14b_b200: Qwen-2.5-14B shape bf16 (48 layers, 40/8 heads), bursty online 2 req/s cv 2 "
                "(4096/256, 30 s) + 64-request offline backlog, 40 GiB KV pool, TBT SLO 200 ms, scheduled with the "
                "reference's fit of the B200 14B profile (profiles/b200_fit_14b.json)"),
    "llama70b": ("llama70b_b200", "llama70b",
                 "llama70b_b200: Llama-3.1-70B shape bf16 (80 layers, 141 GB of weights), online spike 0.5 -> 2 req/s "
                 "at 20 s (2048/128) against a 48-request offline backlog, 20 GiB KV pool, safepoint every layer, "
                 "scheduled with the reference's fit of the B200 70B profile (profiles/b200_fit_70b.json)"),
}
SHAPES = {  # SURVEY.md 8 model table (public HF configs)
    "llama8b": dict(num_layers=32, hidden=4096, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336, vocab=128256,
                    rope_theta=500000.0),
    "qwen14b": dict(num_layers=48, hidden=5120, n_heads=40, n_kv_heads=8, head_dim=128, ffn=13824, vocab=152064,
                    rope_theta=1000000.0),
    "llama70b": dict(num_layers=80, hidden=8192, n_heads=64, n_kv_heads=8, head_dim=128, ffn=28672, vocab=128256,
                     rope_theta=500000.0),
}


def peaks():
    """(HBM GB/s, bf16 TFLOP/s burst, bf16 TFLOP/s sustained, provenance). The
    burst figure is the roofline of a kernel timed alone (the fixed-shape
    probes); the sustained one (back-to-back GEMMs for 4 s, under the power
    cap) of a kernel timed inside the long co-serving run (the window's
    kernel classes)."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        burst = d.get("bf16_tflops", 1590.0)
        return (d.get("hbm_gbs", 6650.0), burst, d.get("bf16_tflops_sustained", burst),
                "measured (MEASURED_PEAKS.json): bf16 sustained for the in-window kernel classes, burst for the "
                "fixed-shape probes; HBM copy peak for both")
    return 6650.0, 1590.0, 1590.0, "fallback (B200_PROFILING.md)"


def percentile(xs, q):
    """Nearest-rank percentile (reference metrics.cpp:41-48)."""
    if not len(xs):
        return 0.0
    s = sorted(xs)
    r = min(max(int(math.ceil(q * len(s))), 1), len(s))
    return s[r - 1]


def slices(n_iter, warmup, steps):
    """[(it0, it1)] of the K timed steps: iterations [W, n) in K contiguous
    slices (a step is a 1/K slice of the run)."""
    W = min(max(warmup, 0), n_iter - 1)
    K = max(1, min(steps, n_iter - W))
    b = np.linspace(W, n_iter, K + 1).round().astype(int)
    return W, [(int(b[i]), int(b[i + 1])) for i in range(K)]


def mode_of(world, replicas):
    return f"tp{world} (KV-head groups, peer all-reduce)" if world > 1 and not replicas else f"{world} replicas"


def config_of(name, W, n_iter, K, n, mode):
    return {"workload": WORKLOADS[name][2], "trace": f"tests/golden/{WORKLOADS[name][0]}",
            "iterations": f"[{W}, {n_iter}) of {n_iter} in {K} steps (a step = one 1/{K} slice of the run)",
            "parallelism": mode if n > 1 else "single",
            "l2": "inputs larger than L2 (16 GB of weights + the KV pool stream every step)"}


# ------------------------------------------------------------ CPU arm (port) --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 9 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


_PORT = {}


def _port_model(shape):
    """fp32 numpy restatement (oracle/numeric.py) of ONE layer of the model
    plus embedding/lm_head, random weights (values do not change CPU time)."""
    if shape in _PORT:
        return _PORT[shape]
    from oracle import numeric as N
    sh = dict(SHAPES[shape])
    L = sh.pop("num_layers")
    s = N.ModelShape(num_layers=1, **sh)
    rng = np.random.default_rng(0)
    H, D = s.hidden, s.head_dim

    class W:
        pass
    w = W()
    w.s = s
    blk = rng.standard_normal((1024, H), dtype=np.float32) * 0.02  # tiled: values do not change CPU time
    w.emb = np.tile(blk, ((s.vocab + 1023) // 1024, 1))[: s.vocab]
    w.lm_head = np.ascontiguousarray(w.emb[::-1])
    w.final_norm = np.ones(H, np.float32)
    w.attn_norm = [np.ones(H, np.float32)]
    w.mlp_norm = [np.ones(H, np.float32)]
    w.wqkv = [rng.standard_normal(((s.n_heads + 2 * s.n_kv_heads) * D, H), dtype=np.float32) * 0.02]
    w.wo = [rng.standard_normal((H, s.n_heads * D), dtype=np.float32) * 0.02]
    w.wgu = [rng.standard_normal((2 * s.ffn, H), dtype=np.float32) * 0.02]
    w.wd = [rng.standard_normal((H, s.ffn), dtype=np.float32) * 0.02]
    _PORT[shape] = (N, s, w, L)
    return _PORT[shape]


def _cpu_cores():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        if info:
            return max(int(i.get("num_threads", 1)) for i in info)
    except Exception:
        pass
    return os.cpu_count()


def port_sample(log, k, shape):
    """CPU port of iteration k of the call log: one of the L layers (with the
    KV context of every entry) timed on the host cores and scaled to L layers,
    plus one lm_head pass over the sampled rows. Returns (offline tokens
    of the iteration, full-model-equivalent seconds, CPU seconds spent)."""
    N, s, w, L = _port_model(shape)
    orc = N.Oracle(s, weights=w, mimic_bf16=False)
    rng = np.random.default_rng(k)
    entries = []
    for rid, P, Cc, kind, online in log.plan_of[k]:
        if kind == 2:
            continue
        entries.append(N.Entry(int(rid), int(P), int(Cc), int(kind), bool(online)))
        ctx = int(Cc) if kind == 0 else int(Cc) - 1
        if ctx > 0:
            kk = rng.standard_normal((ctx, s.n_kv_heads, s.head_dim), dtype=np.float32)
            orc.kv.write(int(rid), 0, np.arange(ctx), kk, kk)
    t0 = time.perf_counter()
    orc.forward(entries)  # 1 layer + final norm + lm_head
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    _ = np.ones((len(entries), s.hidden), np.float32) @ w.lm_head.T
    t_head = time.perf_counter() - t1
    layer = max(dt - t_head, 1e-9)
    return log.offline_tokens(k), layer * L + t_head, dt + t_head


def pick_sample(log, it0, it1, max_tokens=512):
    """The iteration of [it0, it1) with the most offline tokens among those of
    at most max_tokens compute tokens (bounded CPU work); any iteration with
    offline work if none is that small."""
    best, best_off = None, -1
    for k in range(it0, it1):
        p = log.plan_of[k]
        if p[:, 1].sum() > max_tokens:
            continue
        off = log.offline_tokens(k)
        if off > best_off:
            best, best_off = k, off
    if best is None or best_off <= 0:
        cands = [k for k in range(it0, it1) if log.offline_tokens(k) > 0]
        best = min(cands, key=lambda k: log.plan_of[k][:, 1].sum()) if cands else it0
    return best


def control_plane(name, n_iter, min_s=2.0):
    """CPU path (a): the reference's own SimEngine control plane (oracle/_ref/
    time_engine, compiled from /root/reference) on the same RunConfig."""
    exe = os.path.join(ROOT, "oracle", "_ref", "time_engine")
    g = os.path.join(ROOT, "tests", "golden", WORKLOADS[name][0])
    if not os.path.exists(exe):
        return {"unavailable": "oracle/_ref/time_engine not built (make -C oracle time_engine)"}
    try:
        r = subprocess.run([exe, "run_config.json", str(n_iter), str(min_s)], cwd=g, capture_output=True, text=True,
                           timeout=300)
        d = json.loads(r.stdout.strip().splitlines()[-1])
        d["what"] = ("reference coserve::SimEngine::run() (proj/src/sim_engine.cpp:337-392) on this workload's "
                     "RunConfig, single thread, oracle_latency standing in for the forward; and KvCacheManager "
                     "bookkeeping per 16-token page (register/allocate/commit/stage/flush/done/evict/release)")
        return d
    except Exception as ex:
        return {"unavailable": f"time_engine failed: {ex}"}


def load_log(name):
    from oracle.lockstep import trace as T
    g = os.path.join(ROOT, "tests", "golden", WORKLOADS[name][0])
    return T.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))


def run_reference(args):
    """--impl reference: the CPU port over a bounded sample of every step's
    slice (same config, steps and warm-up as the GPU arm)."""
    name = args.workload
    shape = WORKLOADS[name][1]
    log = load_log(name)
    W, sl = slices(log.n_iter, args.warmup, args.steps)
    if args.warmup > 0:
        port_sample(log, pick_sample(log, 0, max(W, 1)), shape)  # page in weights / BLAS
    tok = secs = cpu = 0.0
    picked = []
    for it0, it1 in sl:
        k = pick_sample(log, it0, it1)
        o, full, spent = port_sample(log, k, shape)
        tok += o
        secs += full
        cpu += spent
        picked.append(k)
    v = tok / secs if secs > 0 else 0.0
    cores = _cpu_cores()
    cp = control_plane(name, log.n_iter)
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": len(sl), "warmup": W, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": config_of(name, W, log.n_iter, len(sl), args.gpus, mode_of(args.gpus, args.replicas)),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": (f"per step, the iteration of its slice with the most offline tokens among "
                                        f"those of <= 512 compute tokens (iterations {picked}); 1 of "
                                        f"{SHAPES[shape]['num_layers']} layers run by the fp32 numpy port "
                                        f"(oracle/numeric.py) and scaled, plus one lm_head pass; "
                                        f"{cpu:.1f} s of CPU work")},
            "control_plane": cp,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ------------------------------------------------------------------ GPU arm --
def host_link_peak(device: int):
    """Pinned cudaMemcpyAsync D2H / H2D GB/s (256 MiB, best of 3) on this box:
    the denominator of the checkpoint/restore fraction."""
    import torch
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    s = torch.cuda.Stream(device=device)
    out = {}
    for name in ("d2h", "h2d"):
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                (h.copy_(d, non_blocking=True) if name == "d2h" else d.copy_(h, non_blocking=True))
                e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = n / (best * 1e-3) / 1e9
    return out


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel
    from the committed `ncu --set full` captures (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    return json.load(open(p)) if os.path.exists(p) else {}


def window_tokens(R, tr, it0, it1, t_end_ms):
    """Offline/online tokens committed in [it0, it1) and the online TPOT/TBT
    samples on the given per-iteration clock (ms)."""
    off = on = 0
    times = {}
    for k in range(it0, it1):
        o, n, outs = R.token_progress(tr, k)
        off += o
        on += n
        for rid, _ in outs:
            if tr.requests.get(rid, {}).get("class") == "online":
                times.setdefault(rid, []).append(float(t_end_ms[k - it0]))
    tpot, tbt = [], []
    for rid, ts in times.items():
        if len(ts) >= 2:
            tpot.append((ts[-1] - ts[0]) / (len(ts) - 1))
            tbt.extend(np.diff(ts).tolist())
    return off, on, tpot, tbt


def attention_probe(cs, F, hbm_peak, bf16_peak):
    """K1 (decode) and K2 (prefill) timed alone on 8B attention shapes:
    64 sequences x 4224 context (1.107 GB/layer) and one
    2048-token chunk over a 4096-token context (1.72e11 flop/layer)."""
    import ctypes as C
    cfg = cs.model_config("llama8b", hidden=512, ffn=512, vocab=512, gpu_kv_capacity=80 << 30,
                          host_kv_capacity=1 << 30, max_batched_tokens=8192, instrumented=0)
    eng = cs.Engine(cfg)
    out = {}
    try:
        n, ctx = 64, 4224
        plan = []
        for r in range(n):
            eng.register_request(r, False)
            assert eng.allocate(r, ctx + 1).ok
            eng.commit_allocations(r)
            plan.append(F.cs_batch_entry(r, 1, ctx, F.CS_DECODE, 0))
        arr = (F.cs_batch_entry * n)(*plan)
        msv, bv, fv = C.c_double(), C.c_int64(), C.c_int64()
        cs.engine._check(cs.lib().cs_bench_attention(eng._h, arr, n, 20, C.byref(msv), C.byref(bv), C.byref(fv)))
        gbs = bv.value / (msv.value * 1e-3) / 1e9
        out["decode_64x4224"] = {"ms": msv.value, "bytes": bv.value, "gbs": gbs, "frac": gbs / hbm_peak}
        eng.register_request(1000, False)
        assert eng.allocate(1000, 4096 + 2048).ok
        eng.commit_allocations(1000)
        arr = (F.cs_batch_entry * 1)(F.cs_batch_entry(1000, 2048, 4096, F.CS_PREFILL, 0))
        cs.engine._check(cs.lib().cs_bench_attention(eng._h, arr, 1, 10, C.byref(msv), C.byref(bv), C.byref(fv)))
        tf = fv.value / (msv.value * 1e-3) / 1e12
        out["prefill_2048_over_4096"] = {"ms": msv.value, "flops": fv.value, "tflops": tf, "frac": tf / bf16_peak}
    finally:
        eng.close()
    return out


def safepoint_overhead(cs, F, reps=20, shard=None, attach=None, reduce_max=None):
    """SPEC.md acceptance #6: the same unpreempted mixed plan (online decode +
    offline 2048-token chunk) with a safepoint every layer vs none,
    alternating engines so clock drift hits both. Under the north-star split
    (`shard` = tp_size/tp_rank, every rank calls this) the instrumented engine
    also votes in every all-reduce tail, so `frac` is the g-rank agreement
    cost (reference model: preemption.cpp:15-22), max over ranks."""
    engs = []
    try:
        for instrumented in (0, 1):
            c = cs.model_config("llama8b", gpu_kv_capacity=8 << 30, host_kv_capacity=1 << 30,
                                max_batched_tokens=8192, safepoint_interval_layers=1, instrumented=instrumented,
                                max_entries=256, **(shard or {}))
            e = cs.Engine(c)
            if attach:
                attach(e)
            e.register_request(0, True)
            e.register_request(1, False)
            assert e.allocate(0, 2049).ok
            e.commit_allocations(0)
            engs.append(e)
        times = [[], []]
        for t in range(reps + 2):
            for i, e in enumerate(engs):
                assert e.allocate(1, 2048).ok
                plan = [cs.BatchEntry(0, 1, 2049, F.CS_DECODE, True), cs.BatchEntry(1, 2048, 0, F.CS_PREFILL, False)]
                ms = e.forward(plan, epoch=20_000 + 10 * t + i).gpu_ms
                e.rollback_allocations(1)
                if t >= 2:
                    times[i].append(ms)
        a, b = float(np.median(times[0])), float(np.median(times[1]))
        if reduce_max:
            a, b = reduce_max(a), reduce_max(b)
        g = (shard or {}).get("tp_size", 1)
        return {"ms_without": a, "ms_with": b, "frac": b / a - 1.0, "reps": reps, "tp": g,
                "plan": "online decode (C=2049) + offline 2048-token prefill chunk, 32 layers, 31 safepoints"
                        + (f", vote in every all-reduce tail of {g} ranks (max over ranks)" if g > 1 else "")}
    except Exception as ex:  # never hide the main numbers
        return {"error": str(ex)}
    finally:
        for e in engs:
            e.close()


def live_leg(name, device, margin=None):
    """Live mode (oracle/lockstep/live.cpp): the UNMODIFIED reference SimEngine
    schedules on its fit, but its clock advances by the measured device time
    of each real forward on this GPU (KV calls on the HBM pool). Returns the
    reference's own metrics.json of that run (offline tok/s at its measured
    TBT) plus the tool's summary."""
    import tempfile
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter", "live")
    if not os.path.exists(exe):
        return {"unavailable": "oracle/_ref/adapter/live not built (make -C oracle live)"}
    trace, preset, _ = WORKLOADS[name]
    g = os.path.join(ROOT, "tests", "golden", trace)
    c = json.load(open(os.path.join(g, "run_config.json")))
    wl = c.get("workload", {})
    if isinstance(wl.get("trace"), str):
        wl["trace"] = os.path.join(g, wl["trace"])
    if margin is not None:
        c.setdefault("slo", {})["safety_margin"] = margin
    with tempfile.TemporaryDirectory() as tmp:
        cp = os.path.join(tmp, "run_config.json")
        json.dump(c, open(cp, "w"))
        try:
            r = subprocess.run([exe, cp, tmp, preset, "--device", str(device)], capture_output=True, text=True,
                               timeout=900)
        except Exception as ex:
            return {"error": str(ex)}
        if r.returncode != 0:
            return {"error": r.stderr[-500:]}
        summ = json.loads(r.stdout.strip().splitlines()[-1])
        m = json.load(open(os.path.join(tmp, "metrics.json")))
    slo = c.get("slo", {})
    return {"offline_tok_s": m["offline_throughput"], "online_p99_tbt_ms": 1e3 * m["tbt"]["p99"],
            "online_p99_ttft_ms": 1e3 * m["ttft"]["p99"], "tbt_attainment": m["tbt_attainment"],
            "ttft_attainment": m["ttft_attainment"], "slo_tbt_ms": 1e3 * slo.get("tbt_slo_s", 0.1),
            "slo_ttft_ms": 1e3 * slo.get("ttft_slo_s", 0.5), "safety_margin": slo.get("safety_margin", 0.05),
            "preemptions": m["preemptions"], "iterations": summ["iterations"], "horizon_s": m["horizon_s"],
            "measured_over_predicted_median": summ["measured_over_predicted_median"],
            "transferred_bytes": m["transferred_bytes"], "wall_s": summ["wall_s"]}


def ckpt_ranks(rows):
    """N>1: per-rank checkpoint / restore GB/s (each rank's shard over its own
    host link) and the aggregate (all ranks' bytes over the slowest rank's
    summed copy time)."""
    if not rows:
        return {}
    gbs = lambda b, ms: b / (ms * 1e-3) / 1e9 if ms > 0 else None
    per = [{"rank": i, "d2h_gbs": gbs(r[0], r[1]), "h2d_gbs": gbs(r[2], r[3]), "d2h_bytes": int(r[0]),
            "h2d_bytes": int(r[2]), "host_numa_node": int(r[4])} for i, r in enumerate(rows)]
    return {"per_rank": per,
            "aggregate_d2h_gbs": gbs(sum(r[0] for r in rows), max(r[1] for r in rows)),
            "aggregate_h2d_gbs": gbs(sum(r[2] for r in rows), max(r[3] for r in rows))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20, help="timed steps: 1/K slices of the run after the warm-up")
    ap.add_argument("--warmup", type=int, default=5, help="warm-up steps: the run's first W iterations, untimed")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="llama8b", choices=sorted(WORKLOADS))
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: N independent replicas of the run (one per GPU) instead of the north-star split "
                         "(ONE model sharded over the N GPUs by KV-head groups, peer-memory all-reduce)")
    ap.add_argument("--legs", default="llama8b_kv60",
                    help="comma list of extra full-run workloads reported beside the headline ('' for none)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-probes", action="store_true")
    ap.add_argument("--dump", default=None, help="write per-iteration device times + plan shapes (.npz)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args)
        return

    import torch  # plumbing: device selection, barrier, max-over-ranks
    dist = None
    one_device = os.environ.get("CS_BENCH_ONE_DEVICE") == "1"
    red_dev = "cpu" if one_device else "cuda"  # device of the few reduced scalars
    if world > 1:
        import torch.distributed as dist
        # CS_BENCH_ONE_DEVICE=1: every rank on GPU 0 (plumbing check of the
        # sharded path on a one-GPU box; NCCL refuses two ranks per device, so
        # the process group is gloo and the ranks time-slice the GPU)
        if one_device:
            local = 0
        torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() and not one_device else "gloo")

    import paper_2410_01228_b200 as cs
    from paper_2410_01228_b200 import _ffi as F
    from paper_2410_01228_b200 import replay as R
    hbm_peak, bf16_peak, bf16_sus, peak_kind = peaks()
    tp = world > 1 and not args.replicas
    mode = mode_of(world, args.replicas)

    def attach_tp(eng):
        """One process per GPU: all-gather the exchange regions' IPC handles
        and map every peer's (cs_tp_attach_ipc)."""
        import ctypes as C
        h = (C.c_uint8 * 64)()
        cs.engine._check(cs.lib().cs_tp_exchange_ipc_handle(eng._h, h))
        handles = [None] * world
        dist.all_gather_object(handles, bytes(h))
        allh = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(handles))
        cs.engine._check(cs.lib().cs_tp_attach_ipc(eng._h, allh, world))

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def replay(name, timed=True):
        """Replays tests/golden/<trace> on one engine: W warm-up iterations,
        then the K step slices (timed region: barrier + sync on both sides)."""
        trace, preset, _ = WORKLOADS[name]
        g = os.path.join(ROOT, "tests", "golden", trace)
        tr = R.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))
        W, sl = slices(tr.n_iter, args.warmup, args.steps)
        shard = dict(tp_size=world, tp_rank=rank) if tp else {}
        cfg = R.engine_config_for(tr, preset, device=local, max_entries=256, **shard)
        t_setup = time.time()
        eng = cs.Engine(cfg)
        if shard:
            attach_tp(eng)
        setup_s = time.time() - t_setup
        R.run(eng, tr, 0, W)
        s0 = eng.stats()
        eng.set_kernel_timing(timed)
        sampler = ClockSampler(local)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        sampler.start()
        prof = os.environ.get("CS_PROFILE_REGION") == "1" and timed
        if prof:  # launch lists: ncu --profile-from-start off records the timed region only
            torch.cuda.profiler.start()
        parts = [R.run(eng, tr, a, b) for a, b in sl]
        torch.cuda.synchronize()
        if prof:
            torch.cuda.profiler.stop()
        if dist:
            dist.barrier()
        clocks = sampler.stop()
        s1 = eng.stats()
        kt = {c: eng.kernel_timing(c) for c in (F.CS_KT_K8, F.CS_KT_K2, F.CS_KT_K1, F.CS_KT_LIB, F.CS_KT_GRAPH)}
        eng.set_kernel_timing(False)
        for p in parts:
            assert p.mismatches == 0, f"replay diverged from the reference at op {p.first_mismatch_op}"
        cat = lambda f: np.concatenate([getattr(p, f) for p in parts])
        wall_ms = np.array([p.wall_ms for p in parts])
        op_ms = np.sum([p.op_ms for p in parts], axis=0)
        # per-iteration wall clock of the whole window (each step restarts its clock)
        t_end = np.concatenate([p.wall_end_ms + (wall_ms[:i].sum()) for i, p in enumerate(parts)])
        it0, it1 = sl[0][0], sl[-1][1]
        off, on, tpot, tbt = window_tokens(R, tr, it0, it1, t_end)
        gpu_ms = cat("gpu_ms")
        step_ms = np.array([p.gpu_ms.sum() for p in parts])
        gpu_s, wall_s = float(gpu_ms.sum()) / 1e3, float(wall_ms.sum()) / 1e3
        ranks_ckpt = None
        if dist:
            t = torch.tensor([gpu_s, wall_s], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            gpu_s, wall_s = float(t[0]), float(t[1])
            # per-rank checkpoint traffic: every rank moves its own KV-head shard
            # over its own host link, concurrently (config 5)
            mine = torch.tensor([s1.moved_d2h_bytes - s0.moved_d2h_bytes, s1.moved_d2h_ms - s0.moved_d2h_ms,
                                 s1.moved_h2d_bytes - s0.moved_h2d_bytes, s1.moved_h2d_ms - s0.moved_h2d_ms,
                                 s1.host_numa_node], dtype=torch.float64, device=red_dev)
            allr = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(allr, mine)
            ranks_ckpt = [x.tolist() for x in allr]
        eng.close()
        return dict(tr=tr, W=W, sl=sl, s0=s0, s1=s1, off=off, on=on, tpot=tpot, tbt=tbt, gpu_s=gpu_s, wall_s=wall_s,
                    clocks=clocks, setup_s=setup_s, kt=kt, gpu_ms=gpu_ms, step_ms=step_ms,
                    dropped=cat("dropped_layer"), drop_us=cat("drop_latency_us"), pre_drop=cat("pre_drop_layer_us"),
                    h2d=cat("h2d_bytes"), d2h=cat("d2h_bytes"), iters=int(sum(p.iterations for p in parts)),
                    ranks_ckpt=ranks_ckpt, op_ms=op_ms, wall_end_ms=t_end)

    rp = replay(args.workload)
    reps = world if (world > 1 and not tp) else 1
    tr, W, sl, s0, s1 = rp["tr"], rp["W"], rp["sl"], rp["s0"], rp["s1"]
    K = len(sl)
    if args.dump and rank == 0:
        shapes = []
        for k in range(sl[0][0], sl[-1][1]):
            pl = tr.plan_of[k]
            pre, dec = pl[pl[:, 3] != 1], pl[pl[:, 3] == 1]
            shapes.append([len(pl), int(pre[:, 1].sum()), int((pre[:, 1] * (pre[:, 1] + pre[:, 2])).sum()),
                           len(dec), int(dec[:, 2].sum())])
        np.savez(args.dump, gpu_ms=rp["gpu_ms"], shapes=np.array(shapes, np.int64), wall_end_ms=rp["wall_end_ms"])

    legs = {}
    if not args.no_probes:
        for leg in [x for x in args.legs.split(",") if x and x != args.workload]:
            o = replay(leg, timed=False)
            d2h_b = o["s1"].moved_d2h_bytes - o["s0"].moved_d2h_bytes
            h2d_b = o["s1"].moved_h2d_bytes - o["s0"].moved_h2d_bytes
            legs[leg] = {"workload": WORKLOADS[leg][2], "value": reps * o["off"] / o["gpu_s"],
                         "e2e": reps * o["off"] / o["wall_s"],
                         "online_p99_tpot_ms": percentile(o["tpot"], 0.99),
                         "online_p99_tbt_ms": percentile(o["tbt"], 0.99),
                         "slo_tbt_ms": 1e3 * o["tr"].config.get("slo", {}).get("tbt_slo_s", 0.1),
                         "offline_tokens": o["off"], "iterations": o["iters"], "d2h_bytes": d2h_b,
                         "h2d_bytes": h2d_b, "drops": int((o["dropped"] >= 0).sum())}

    live = {}
    if not args.no_probes and rank == 0 and world == 1:
        live["recorded_margin"] = live_leg(args.workload, local)
        live["margin_0"] = live_leg(args.workload, local, margin=0.0)

    probes = {}
    if not args.no_probes and tp:  # every rank: the agreement cost at g = world
        probes["safepoint_overhead"] = safepoint_overhead(cs, F, shard=dict(tp_size=world, tp_rank=rank),
                                                          attach=attach_tp, reduce_max=reduce_max)
    if not args.no_probes and rank == 0:
        probes["attention"] = attention_probe(cs, F, hbm_peak, bf16_peak)
        if not tp:
            probes["safepoint_overhead"] = safepoint_overhead(cs, F)
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    off, on, tpot, tbt = rp["off"], rp["on"], rp["tpot"], rp["tbt"]
    gpu_s, wall_s = rp["gpu_s"], rp["wall_s"]
    value = reps * off / gpu_s
    e2e = reps * off / wall_s
    slo_tbt = 1e3 * tr.config.get("slo", {}).get("tbt_slo_s", 0.1)
    d2h_b = s1.moved_d2h_bytes - s0.moved_d2h_bytes
    d2h_ms = s1.moved_d2h_ms - s0.moved_d2h_ms
    h2d_b = s1.moved_h2d_bytes - s0.moved_h2d_bytes
    h2d_ms = s1.moved_h2d_ms - s0.moved_h2d_ms
    link_peak = host_link_peak(local)
    traffic = ncu_traffic()

    # kernel classes timed live over the timed region (CUDA events on the
    # compute stream around each non-graph launch)
    kinfo = {}
    for cls, key, bound, unit, scale, peak, tkey in (
            (F.CS_KT_K8, "K8 gemm_pf_kernel (layer projections, tcgen05 cta_group::2)", "tensor", "TFLOP/s", 1e12,
             bf16_sus, "K8"),
            (F.CS_KT_K2, "K2 attn_prefill_tc_kernel (prefill paged attention, tcgen05)", "tensor", "TFLOP/s", 1e12,
             bf16_sus, "K2"),
            (F.CS_KT_K1, "K1 attn_decode_kernel (decode paged attention)", "hbm", "GB/s", 1e9, hbm_peak, "K1")):
        t = rp["kt"][cls]
        if t.launches == 0 or t.ms <= 0:
            continue
        per = t.units / t.launches
        ach = per / (t.ms / t.launches * 1e-3) / scale
        kinfo[tkey] = {"kernel": key, "bound": bound, "achieved": ach, "peak": peak, "unit": unit,
                       "frac": ach / peak, "traffic": traffic.get(tkey, {}).get("dram_bytes"),
                       "traffic_source": traffic.get(tkey, {}).get("source"),
                       "launches": int(t.launches), "ms_total": t.ms, "avg_launch_ms": t.ms / t.launches,
                       "algorithmic_per_launch": per,
                       "share_of_window": t.ms / (gpu_s * 1e3)}
    dom = max(kinfo, key=lambda k: kinfo[k]["ms_total"]) if kinfo else None
    # where the rest of the window goes: library GEMMs of non-graph forwards,
    # whole decode-graph forwards (cuBLAS GEMMs + K1 + norms inside)
    lib, gr = rp["kt"][F.CS_KT_LIB], rp["kt"][F.CS_KT_GRAPH]
    breakdown = {k: v["share_of_window"] for k, v in kinfo.items()}
    breakdown["cublas_gemm_nongraph"] = lib.ms / (gpu_s * 1e3)
    breakdown["cublas_gemm_nongraph_tflops"] = lib.units / (lib.ms * 1e-3) / 1e12 if lib.ms > 0 else None
    breakdown["decode_graph_forwards"] = gr.ms / (gpu_s * 1e3)
    breakdown["decode_graph_iterations"] = int(gr.launches)
    breakdown["other"] = 1.0 - sum(v for k, v in breakdown.items()
                                   if k in kinfo or k in ("cublas_gemm_nongraph", "decode_graph_forwards"))
    roofline = dict(kinfo[dom]) if dom else {}
    if dom:
        roofline["peak_kind"] = peak_kind
        roofline["others"] = {k: {x: v[x] for x in ("achieved", "unit", "frac", "share_of_window", "launches")}
                              for k, v in kinfo.items() if k != dom}
        roofline["probes"] = probes.get("attention")
        roofline["window_breakdown"] = breakdown

    dl = rp["dropped"]
    drops = []
    for i in np.nonzero(dl >= 0)[0]:
        k = sl[0][0] + int(i)
        drops.append({"iteration": k, "reference_layer": int(tr.dropped[k]), "device_layer": int(dl[i]),
                      "flag_to_drop_us": float(rp["drop_us"][i]), "layer_time_us": float(rp["pre_drop"][i]),
                      "under_one_layer": bool(rp["drop_us"][i] < rp["pre_drop"][i])})
    ref_drops = int(sum(1 for k in range(sl[0][0], sl[-1][1]) if tr.dropped[k] >= 0))
    cpu = None
    if not args.no_cpu and world == 1:  # the CPU baseline is an N = 1 measurement (rank 0)
        try:
            log = load_log(args.workload)
            k = pick_sample(log, sl[0][0], sl[-1][1])
            o, full, spent = port_sample(log, k, WORKLOADS[args.workload][1])
            cpu = {"value": o / full, "unit": UNIT, "cores": _cpu_cores(), "kind": "port",
                   "sample": f"iteration {k} of the run ({len(log.plan_of[k])} entries): 1 of the model's layers by "
                             f"the fp32 numpy port (oracle/numeric.py) scaled to all layers + one lm_head pass; "
                             f"{spent:.1f} s of CPU work",
                   "control_plane": control_plane(args.workload, log.n_iter)}
        except Exception as ex:  # the CPU sample must never hide the GPU number
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "sample": f"failed: {ex}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": 1e3 * gpu_s / K, "higher_is_better": True,
        "scaling": "strong" if tp else "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, teacher-forced hashed token ids, the reference's recorded schedule)",
        "config": config_of(args.workload, W, tr.n_iter, K, world, mode),
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": float(rp["h2d"].sum()) / K,
                "d2h_bytes_per_step": float(rp["d2h"].sum()) / K,
                "what": "offline tokens / wall time of the replay through the C-ABI (host plan buffers: H2D plan "
                        "metadata, D2H sampled ids, every iteration)",
                "wall_s": wall_s, "device_s": gpu_s,
                "host_ms_by_op": {k: round(float(rp["op_ms"][c]), 1) for k, c in R.OPC.items()
                                  if float(rp["op_ms"][c]) >= 0.05}},
        "online_p99_tpot_ms": percentile(tpot, 0.99), "online_p99_tbt_ms": percentile(tbt, 0.99),
        "slo_tbt_ms": slo_tbt, "slo_met": bool(percentile(tbt, 0.99) <= slo_tbt),
        "offline_tokens": off, "online_tokens": on, "iterations": rp["iters"],
        "step_ms": {"min": float(rp["step_ms"].min()), "median": float(np.median(rp["step_ms"])),
                    "max": float(rp["step_ms"].max())},
        "preempt": {"drops": drops, "reference_drops_in_window": ref_drops,
                    "max_flag_to_drop_us": max((d["flag_to_drop_us"] for d in drops), default=None),
                    "all_under_one_layer": bool(drops) and all(d["under_one_layer"] for d in drops),
                    "what": "host flag store (when the device enters the layer the reference's Alg. 1 fired in) -> "
                            "the next layer-head kernel truncating the batch on the device; every later kernel of "
                            "the forward (K8 GEMMs included, device-side M) runs on the online rows",
                    "safepoint_overhead": probes.get("safepoint_overhead")},
        "kv_ckpt": {"d2h_gbs": d2h_b / (d2h_ms * 1e-3) / 1e9 if d2h_ms > 0 else None,
                    "h2d_gbs": h2d_b / (h2d_ms * 1e-3) / 1e9 if h2d_ms > 0 else None,
                    "d2h_bytes": d2h_b, "h2d_bytes": h2d_b, "host_link_peak_gbs": link_peak,
                    "frac_d2h": (d2h_b / (d2h_ms * 1e-3) / 1e9) / link_peak["d2h"] if d2h_ms > 0 else None,
                    "frac_h2d": (h2d_b / (h2d_ms * 1e-3) / 1e9) / link_peak["h2d"] if h2d_ms > 0 else None,
                    "host_numa_node": s1.host_numa_node,
                    **ckpt_ranks(rp["ranks_ckpt"])},
        "nonresident_reads": s1.nonresident_reads,
        "legs": legs,
        "live": dict(live, what="live mode (oracle/lockstep/live.cpp): the unmodified reference SimEngine schedules "
                                "on its B200 fit while its clock advances by the measured device time of each "
                                "real forward on this GPU; metrics are the reference's own metrics.json") if live
        else None,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": rp["clocks"],
        "gpu_launches": int(s1.kernel_launches - s0.kernel_launches),
        "setup_s": rp["setup_s"],
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
