"""Profiles the B200 engine over the reference's latency grid
(default_profile_grid, perf_model.cpp:98-108: P in {1,16,64,256,512,1024,2048,
4096} x C in {0,1K,4K,16K,40K,64K}) -- one single-entry prefill plan per point,
exactly what coserve::profile measures on its oracle (perf_model.cpp:110-123),
but timed as the real Llama-3.1-8B forward on the device (CUDA events,
median of 3 after a warm-up). Writes {"grid": [[P, C, ms], ...]}, the format
coserve::profile_from_json_text reads; oracle/_ref/fit_profile then fits the
reference's own model to it (the closed loop).

  python tools/profile_b200.py [--out profiles/b200_profile.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01228_b200 as cs  # noqa: E402

P_VALUES = (1, 16, 64, 256, 512, 1024, 2048, 4096)
C_VALUES = (0, 1024, 4096, 16384, 40960, 65536)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "b200_profile.json"))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--p-values", type=int, nargs="*", default=list(P_VALUES))
    ap.add_argument("--c-values", type=int, nargs="*", default=list(C_VALUES))
    ap.add_argument("--preset", default="llama8b")
    args = ap.parse_args()
    kv_gib = 12 if args.preset == "llama8b" else 24
    # forwards here are synchronous, so freed blocks need no quarantine
    cfg = cs.model_config(args.preset, gpu_kv_capacity=kv_gib << 30, host_kv_capacity=1 << 30,
                          max_batched_tokens=8192, instrumented=0, max_entries=64,
                          flags=cs._ffi.CS_FLAG_NO_FWD_QUARANTINE)
    eng = cs.Engine(cfg)
    grid = []
    rid = 0
    try:
        for c in args.c_values:
            # context of c tokens, written once (its values do not change timing)
            ctx_id = None
            if c > 0:
                ctx_id = rid
                rid += 1
                eng.register_request(ctx_id, False)
                assert eng.allocate(ctx_id, c).ok
                eng.commit_allocations(ctx_id)
            for p in args.p_values:
                times = []
                for rep in range(args.reps + 1):
                    if ctx_id is None:
                        r = rid
                        rid += 1
                        eng.register_request(r, False)
                        assert eng.allocate(r, p).ok
                        entry = cs.BatchEntry(r, p, 0, cs.CS_PREFILL, False)
                    else:
                        r = ctx_id
                        assert eng.allocate(r, p).ok
                        entry = cs.BatchEntry(r, p, c, cs.CS_PREFILL, False)
                    info = eng.forward([entry], epoch=rid)
                    eng.rollback_allocations(r)
                    if ctx_id is None:
                        eng.release_request(r)
                    if rep > 0:
                        times.append(info.gpu_ms)
                ms = float(np.median(times))
                grid.append([p, c, ms])
                print(f"P={p:5d} C={c:6d} {ms:8.3f} ms", flush=True)
            if ctx_id is not None:
                eng.release_request(ctx_id)
    finally:
        eng.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"grid": grid, "model": f"{args.preset} bf16, 1 B200", "timing": "CUDA events, median of %d" % args.reps},
              open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
