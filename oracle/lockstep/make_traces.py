"""Generates the golden lockstep call logs from the UNMODIFIED reference
(oracle/_ref/recorder, built by `make -C oracle recorder`) -- test/bench
infrastructure only. Output: tests/golden/<scenario>/{run_config.json,
trace.jsonl, calls.jsonl.gz, metrics.json, requests.jsonl.gz}.

Scenarios:
  config1  -- tiny CPU co-serving trace: 16 offline (in=96+16i, out=8+i) at
              t=0 and 4 online (in=64+32i, out=12) at 10/12/40/41 ms; L=2,
              interval 1, 2048 B/token, 64-page GPU pool, 512-token batches,
              oracle k1=0.0214 k2=8.36e-7 k4=7e-5 k5=3.5, SLO 50 ms / 20 ms.
  llama8b  -- Llama-3.1-8B shape (real 131072 B/token, 32 layers), 8192-token
              batches, a 24 GiB KV pool (so the run evicts, checkpoints and
              restores), bursty Gamma online trace (rate 3/s, cv 2) 4096/256
              over 30 s plus a 64-request offline backlog with replenish,
              8B-preset oracle coefficients (coserve_cli.cpp:45-53), SLO
              TTFT 0.5 s / TBT 0.1 s, a safepoint every layer.
"""
from __future__ import annotations

import gzip
import json
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
RECORDER = os.path.join(ROOT, "oracle", "_ref", "recorder")
GOLDEN = os.path.join(ROOT, "tests", "golden")


def _8b_oracle():
    # calibrate_preset("8b") (coserve_cli.cpp:45-53)
    chunk, ctx, fresh, deep = 2048.0, 40960.0, 51.0, 124.0
    k4, k5, k3 = 7e-5, 3.5, 0.0
    k2 = (deep - fresh - k4 * ctx) / (chunk * ctx)
    k1 = (fresh - k2 * chunk * chunk - k4 * chunk - k5) / chunk - k3
    return {"k1": k1, "k2": k2, "k3": k3, "k4": k4, "k5": k5, "noise_cv": 0.0}


def scenario(name: str):
    if name == "config1":
        trace = [{"t": 0.0, "class": "offline", "in": 96 + 16 * i, "out": 8 + i} for i in range(16)]
        for i, t in enumerate([0.010, 0.012, 0.040, 0.041]):
            trace.append({"t": t, "class": "online", "in": 64 + 32 * i, "out": 12})
        cfg = {
            "cluster": {"num_layers": 2, "safepoint_interval_layers": 1, "kv_bytes_per_token": 2048,
                        "gpu_kv_capacity": 64 * 16 * 2048, "host_kv_capacity": 4096 * 16 * 2048,
                        "d2h_bandwidth": 38797312000.0, "h2d_bandwidth": 38797312000.0,
                        "safepoint_check_cost_us": 21.0, "gather_cost_us": 500.0, "max_batched_tokens": 512},
            "oracle": {"k1": 0.0214, "k2": 8.36e-7, "k4": 7e-5, "k5": 3.5},
            "policy": {"kind": "conserve"},
            "slo": {"ttft_slo_s": 0.05, "tbt_slo_s": 0.02, "safety_margin": 0.0},
            "workload": {"trace": "TRACE"},
            "seed": 1, "audit": True,
        }
        return cfg, trace
    if name == "llama8b":
        cfg = {
            "cluster": {"num_layers": 32, "safepoint_interval_layers": 1, "kv_bytes_per_token": 131072,
                        "gpu_kv_capacity": 24 << 30, "host_kv_capacity": 64 << 30,
                        "safepoint_check_cost_us": 5.0, "max_batched_tokens": 8192},
            "oracle": _8b_oracle(),
            "policy": {"kind": "conserve"},
            "slo": {"ttft_slo_s": 0.5, "tbt_slo_s": 0.1},
            "workload": {"online": {"rate": 3.0, "cv": 2.0, "input_tokens": 4096, "output_tokens": 256,
                                    "duration_s": 30.0},
                         "offline": {"backlog": 64, "input_tokens": 4096, "output_tokens": 256, "replenish": True}},
            "seed": 1,
        }
        return cfg, None
    if name == "llama8b_b200":
        # the llama8b scenario with the reference scheduler planning on
        # B200-measured latencies: oracle coefficients = the reference's own
        # fit (oracle/_ref/fit_profile) of the engine profiled on a B200 over
        # default_profile_grid (tools/profile_b200.py -> profiles/b200_fit.json)
        cfg, _ = scenario("llama8b")
        fit = json.load(open(os.path.join(ROOT, "profiles", "b200_fit.json")))["coeffs"]
        cfg["oracle"] = {"k1": fit["a_lin"], "k2": fit["a_quad"], "k3": 0.0, "k4": fit["a_mem"],
                         "k5": fit["a_const"], "noise_cv": 0.0}
        # the single-entry fit underpredicts some mixed batches (measured P99
        # TBT 112 ms at the default 5% margin, profiles/r1/bench_r1g.json):
        # the scheduler budgets TBT x (1 - margin) (config.hpp:17-28)
        cfg["slo"]["safety_margin"] = 0.2
        return cfg, None
    if name == "llama8b_b200_kv60":
        # the same B200 schedule with the reference's default 60 GiB KV pool
        # (config.hpp:37): offline requests stay resident (no restores), every
        # new KV token is still checkpointed
        cfg, _ = scenario("llama8b_b200")
        cfg["cluster"]["gpu_kv_capacity"] = 60 << 30
        return cfg, None
    if name == "llama8b_b200_spike":
        # BASELINE config 2 with the pieces the driver-timed window must hold
        # (VERDICT r1): the B200-fitted llama8b schedule, an online load spike
        # (2 -> 8 req/s for 4 s at t = 12 s, frozen as a trace like config 4)
        # against a 96-request offline backlog, and a 32 GiB KV pool, so the
        # run preempts layer-wise, evicts, checkpoints AND restores.
        import numpy as np
        cfg, _ = scenario("llama8b_b200")
        cfg["cluster"]["gpu_kv_capacity"] = 32 << 30
        rng = np.random.default_rng(8)
        trace = [{"t": 0.0, "class": "offline", "in": 4096, "out": 256} for _ in range(96)]
        t = 0.0
        while True:
            t += float(rng.exponential(1.0 / (8.0 if 12.0 <= t < 16.0 else 2.0)))
            if t >= 30.0:
                break
            trace.append({"t": round(t, 6), "class": "online", "in": 4096, "out": 256})
        cfg["workload"] = {"trace": "TRACE"}
        # a latency-critical online class: TTFT SLO 150 ms (a 4096-token
        # prefill is ~55 ms on the B200), so an arrival during a large
        # offline batch trips Alg. 1 (preemption.cpp:24-32): 7 layer-wise
        # drops in the reference run (0 at the 0.5 s SLO)
        cfg["slo"]["ttft_slo_s"] = 0.15
        return cfg, trace
    if name == "qwen14b_b200":
        # BASELINE config 3's model (Qwen-2.5-14B shape: 48 layers, 40/8 heads,
        # 196608 B/token -- the reference presets' own KV unit) on ONE B200,
        # the llama8b workload at 2 req/s online, a 40 GiB KV pool, scheduled
        # on the reference-fitted B200 14B profile (profiles/b200_fit_14b.json)
        cfg, _ = scenario("llama8b")
        fit = json.load(open(os.path.join(ROOT, "profiles", "b200_fit_14b.json")))["coeffs"]
        cfg["cluster"]["num_layers"] = 48
        cfg["cluster"]["kv_bytes_per_token"] = 196608
        cfg["cluster"]["gpu_kv_capacity"] = 40 << 30
        # 3 req/s of 4096/256 online work exceeds a 14B on one GPU: the
        # reference scheduler then stops dispatching ("event queue drained")
        cfg["workload"]["online"]["rate"] = 2.0
        cfg["oracle"] = {"k1": fit["a_lin"], "k2": fit["a_quad"], "k3": 0.0, "k4": fit["a_mem"],
                         "k5": fit["a_const"], "noise_cv": 0.0}
        # the 14B single-entry fit prices a decode at ~1 ms of KV traffic at 4K
        # context; 90 online decodes then exceed a 100 ms budget and the
        # reference scheduler drains its queue -> a 200 ms TBT SLO
        cfg["slo"] = {"ttft_slo_s": 1.0, "tbt_slo_s": 0.2, "safety_margin": 0.2}
        return cfg, None
    if name == "llama70b_b200":
        # BASELINE config 4 on ONE B200 (141 GB of bf16 weights + a 20 GiB KV
        # pool fit in 179 GiB): Llama-3.1-70B shape (80 layers, 327680 B/token),
        # safepoint every layer, an online load spike (0.5 -> 2 req/s at 20 s,
        # frozen as a trace) against a 48-request offline backlog, scheduled by
        # the reference on the reference-fitted B200 70B profile
        # (profiles/b200_fit_70b.json); host link at the measured pinned peaks.
        import numpy as np
        fit = json.load(open(os.path.join(ROOT, "profiles", "b200_fit_70b.json")))["coeffs"]
        rng = np.random.default_rng(70)
        trace = [{"t": 0.0, "class": "offline", "in": 2048, "out": 128} for _ in range(48)]
        t = 0.0
        while True:
            t += float(rng.exponential(1.0 / (0.5 if t < 20.0 else 2.0)))
            if t >= 40.0:
                break
            trace.append({"t": round(t, 6), "class": "online", "in": 2048, "out": 128})
        cfg = {
            "cluster": {"num_layers": 80, "safepoint_interval_layers": 1, "kv_bytes_per_token": 327680,
                        "gpu_kv_capacity": 20 << 30, "host_kv_capacity": 64 << 30,
                        "d2h_bandwidth": 57.1e9, "h2d_bandwidth": 55.6e9,
                        "safepoint_check_cost_us": 5.0, "max_batched_tokens": 8192},
            "oracle": {"k1": fit["a_lin"], "k2": fit["a_quad"], "k3": 0.0, "k4": fit["a_mem"],
                       "k5": fit["a_const"], "noise_cv": 0.0},
            "policy": {"kind": "conserve"},
            "slo": {"ttft_slo_s": 0.6, "tbt_slo_s": 0.3, "safety_margin": 0.2},
            "workload": {"trace": "TRACE"},
            "seed": 1,
        }
        return cfg, trace
    if name.startswith("config1_"):
        # the config-1 trace under the other policies / ablations
        # (policy kinds: config.cpp:38-44; ablation switches: config.hpp:76-82)
        cfg, trace = scenario("config1")
        variant = name[len("config1_"):]
        pol = {"nonpreemptive": {"kind": "non_preemptive"}, "onlineonly": {"kind": "online_only"},
               "sarathi": {"kind": "sarathi_preemptive"},
               "noincr": {"kind": "conserve", "incremental_kv": False},
               "nolayerwise": {"kind": "conserve", "layerwise_preemption": False},
               "pool48": {"kind": "conserve"}, "pool80": {"kind": "conserve"},
               **{f"host{h}": {"kind": "conserve"} for h in (32, 40, 48)}}[variant]
        cfg["policy"] = pol
        if variant.startswith("pool"):
            cfg["cluster"]["gpu_kv_capacity"] = int(variant[4:]) * 16 * 2048
        if variant.startswith("host"):
            # host-memory-limited regime:
            # flush_checkpoints must LRU-evict host copies and tag recompute
            # (kv_cache.cpp:326-362, 379-384); a 48-page GPU pool so evicted
            # requests restore from, or recompute past, the small host pool
            cfg["cluster"]["host_kv_capacity"] = int(variant[4:]) * 16 * 2048
            cfg["cluster"]["gpu_kv_capacity"] = 48 * 16 * 2048
            # the reference's own per-event audit trips on this regime ("host
            # byte accounting drifted" / "interior page is partial", reference
            # defects); record without it -- the final audit verdict is kept
            # and must be reproduced by the replay
            cfg["audit"] = False
        return cfg, trace
    if name.startswith("fuzz"):
        # test_sim_engine.cpp:166-187 ("fuzzed co-serving runs"): base_config
        # (:14-35) with a 160-page GPU pool at 196608 B/token (= the real
        # Qwen-2.5-14B shape, 48 layers x 8 KV heads x 128), audit after every
        # event. Seed 1 is the reference's own crash -> skipped.
        seed = int(name[4:])
        pol = {"kind": "conserve"}
        if seed % 3 == 0:
            pol = {"kind": "sarathi_preemptive"}
        if seed % 3 == 1:
            pol["incremental_kv"] = seed % 2 == 0
        cfg = {
            "cluster": {"num_layers": 48, "kv_bytes_per_token": 196608, "gpu_kv_capacity": 196608 * 16 * 160,
                        "host_kv_capacity": 196608 * 16 * 256},
            "oracle": {"k1": 0.0214, "k2": 8.36e-7, "k4": 7e-5, "k5": 3.5},
            "policy": pol,
            "slo": {"ttft_slo_s": 1.0, "tbt_slo_s": 0.1, "safety_margin": 0.0},
            "workload": {"online": {"rate": 6.0, "cv": 0.5, "input_tokens": 320, "output_tokens": 24,
                                    "duration_s": 6.0},
                         "offline": {"backlog": 6, "input_tokens": 512, "output_tokens": 16}},
            "seed": seed, "audit": True, "max_sim_time_s": 300.0,
        }
        return cfg, None
    raise SystemExit(f"unknown scenario {name}")


def record(name: str) -> str:
    if not os.path.exists(RECORDER):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "recorder"], check=True)
    cfg, trace = scenario(name)
    out = os.path.join(GOLDEN, name)
    os.makedirs(out, exist_ok=True)
    with tempfile.TemporaryDirectory() as tmp:
        if trace is not None:
            tpath = os.path.join(out, "trace.jsonl")
            with open(tpath, "w") as f:
                for t in trace:
                    f.write(json.dumps(t) + "\n")
            cfg["workload"]["trace"] = tpath
        cpath = os.path.join(tmp, "run_config.json")
        with open(cpath, "w") as f:
            json.dump(cfg, f, indent=1)
        r = subprocess.run([RECORDER, cpath, tmp], capture_output=True, text=True)
        print(r.stdout.strip(), r.stderr.strip())
        if r.returncode != 0:
            raise SystemExit(r.returncode)
        if trace is not None:
            cfg["workload"]["trace"] = "trace.jsonl"
        with open(os.path.join(out, "run_config.json"), "w") as f:
            json.dump(cfg, f, indent=1)
        for fn in ["calls.jsonl", "requests.jsonl"]:
            with open(os.path.join(tmp, fn), "rb") as src, gzip.open(os.path.join(out, fn + ".gz"), "wb") as dst:
                shutil.copyfileobj(src, dst)
        shutil.copy(os.path.join(tmp, "metrics.json"), os.path.join(out, "metrics.json"))
        with open(os.path.join(out, "summary.txt"), "w") as f:
            f.write(r.stdout)
    return out


if __name__ == "__main__":
    ALL = ["config1", "llama8b"] + [f"config1_{v}" for v in
                                    ("nonpreemptive", "onlineonly", "sarathi", "noincr", "nolayerwise", "pool48",
                                     "pool80")] + [f"fuzz{s}" for s in range(2, 7)]
    for n in sys.argv[1:] or ALL:
        print(n, "->", record(n))
