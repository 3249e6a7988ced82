"""Decode-step probe (tools only): one decode-only plan shaped like the
headline trace's decode iterations (n sequences at ~4.3K context, Llama-3.1-8B
shape, CUDA-graph path) run `reps` times; prints the event-timed step and its
HBM roofline (weights + K/V bytes). Run under `ncu --metrics
gpu__time_duration.sum` for the per-kernel breakdown of one step.
    python tools/decode_probe.py [n_seqs] [ctx] [reps]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2410_01228_b200 as cs  # noqa: E402
from paper_2410_01228_b200 import _ffi as F  # noqa: E402


def main(n=36, ctx=4300, reps=10):
    cfg = cs.model_config("llama8b", gpu_kv_capacity=(n * (ctx + 64) * 131072) + (1 << 30), host_kv_capacity=1 << 30,
                          max_batched_tokens=8192, instrumented=1, max_entries=256)
    eng = cs.Engine(cfg)
    plan = []
    for r in range(n):
        eng.register_request(r, r < n // 4)
        assert eng.allocate(r, ctx + r).ok
        eng.commit_allocations(r)
    ms = []
    for t in range(reps):
        plan = [cs.BatchEntry(r, 1, ctx + r, F.CS_DECODE, r < n // 4) for r in range(n)]
        info = eng.forward(plan, epoch=100 + t)
        ms.append(info.gpu_ms)
    W = 2 * (32 * (4096 * 6144 + 4096 * 4096 + 4096 * 28672 + 14336 * 4096) + 128256 * 4096)
    kv = sum((ctx + r) * 8 * 128 * 4 * 32 for r in range(n)) + n * 32 * 128 * 4 * 32
    med = float(np.median(ms[2:]))
    print(json.dumps({"n": n, "ctx": ctx, "step_ms": med, "weights_gb": W / 1e9, "kv_gb": kv / 1e9,
                      "ideal_ms_at_6500": (W + kv) / 6.5e12 * 1e3, "frac": (W + kv) / 6.5e12 * 1e3 / med,
                      "all_ms": [round(x, 3) for x in ms]}))
    eng.close()


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
