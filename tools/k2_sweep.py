"""K2 (prefill attention) event-timed over several plan shapes, Llama-3.1-8B
heads (32 q / 8 KV, d=128): single chunks over cached contexts and multi-entry
mixes like the bench's prefill iterations. Prints one JSON line per shape.

  python tools/k2_sweep.py [reps]
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01228_b200 as cs  # noqa: E402
from paper_2410_01228_b200 import _ffi as F  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_targets import bench_attention  # noqa: E402

SHAPES = [
    [(2048, 4096)],
    [(2048, 0)],
    [(1024, 3072)],
    [(4096, 0)],
    [(512, 8192)],
    [(256, 4000)],
    [(1500, 2000), (1800, 500), (1400, 0)],
    [(2000, 2200), (2000, 200)],
]


def main(reps=20):
    cfg = cs.model_config("llama8b", hidden=512, ffn=512, vocab=512, gpu_kv_capacity=40 << 30,
                          host_kv_capacity=1 << 30, max_batched_tokens=8192, instrumented=0)
    eng = cs.Engine(cfg)
    rid = 0
    peak = 1668.5
    for shape in SHAPES:
        plan, ids = [], []
        for P, C in shape:
            ids.append(rid)
            eng.register_request(rid, False)
            assert eng.allocate(rid, P + C).ok
            eng.commit_allocations(rid)
            plan.append(F.cs_batch_entry(rid, P, C, F.CS_PREFILL, 0))
            rid += 1
        ms, _, f = bench_attention(eng, plan, reps)
        print(json.dumps({"shape": shape, "ms": round(ms, 4), "tflops": round(f / ms / 1e9, 1),
                          "frac": round(f / ms / 1e9 / peak, 3)}), flush=True)
        for r in ids:
            eng.release_request(r)
    eng.close()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
