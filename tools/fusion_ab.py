"""A/B (tools only): one Llama-3.1-8B prefill forward (the K8 path) with the
K8 epilogue fusions on and off (CS_NO_FUSE), median device ms of `reps`
forwards per mode, for chunk sizes covering the bench's prefill iterations.
    python tools/fusion_ab.py [reps]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(P, reps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2410_01228_b200 as cs
    cfg = cs.model_config("llama8b", gpu_kv_capacity=8 << 30, host_kv_capacity=1 << 28, max_batched_tokens=8192,
                          instrumented=0, max_entries=64)
    eng = cs.Engine(cfg)
    ms = []
    for rep in range(reps + 1):
        eng.register_request(rep, False)
        assert eng.allocate(rep, P).ok
        info = eng.forward([cs.BatchEntry(rep, P, 0, cs.CS_PREFILL, False)], epoch=rep + 1)
        eng.commit_allocations(rep)
        eng.release_request(rep)
        if rep:
            ms.append(info.gpu_ms)
    eng.close()
    print(json.dumps({"P": P, "fused": os.environ.get("CS_NO_FUSE") != "1", "ms": float(np.median(ms))}), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    for P in (2048, 4096, 6144, 8192):
        for nf in ("1", "0"):
            env = dict(os.environ, CS_NO_FUSE=nf)
            subprocess.run([sys.executable, os.path.abspath(__file__), "child", str(P), str(reps)], env=env, check=True)
