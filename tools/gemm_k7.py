"""K7 (tcgen05 weight-streaming GEMM) against cuBLASLt on the decode-step
projection shapes of Llama-3.1-8B: ms per launch, achieved weight-stream
GB/s, and the max |K7 - cuBLAS| relative to max |cuBLAS|. One JSON line per
shape.   python tools/gemm_k7.py [reps]
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01228_b200 as cs  # noqa: E402

SHAPES = [  # (name, N, K)
    ("qkv", 6144, 4096), ("o_proj", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336),
    ("lm_head", 128256, 4096)]


def main(reps=50, only=None):
    cfg = cs.model_config("llama8b", hidden=512, ffn=512, vocab=512, gpu_kv_capacity=1 << 30,
                          host_kv_capacity=1 << 28, max_batched_tokens=1024, instrumented=0)
    eng = cs.Engine(cfg)
    cases = [(M, s) for M in (8, 32, 64, 128, 256) for s in SHAPES] if only is None else [(only[0], ("one",) + only[1:])]
    for M, (name, N, K) in cases:
        if True:
            a, b, d, r = C.c_double(), C.c_double(), C.c_double(), C.c_double()
            cs.engine._check(cs.lib().cs_bench_gemm(eng._h, M, N, K, reps, C.byref(a), C.byref(b), C.byref(d),
                                                    C.byref(r)))
            wbytes = N * K * 2
            print(json.dumps({"M": M, "shape": name, "N": N, "K": K, "k7_ms": round(a.value, 4),
                              "cublas_ms": round(b.value, 4), "k7_gbs": round(wbytes / a.value / 1e6),
                              "cublas_gbs": round(wbytes / b.value / 1e6),
                              "rel_diff": d.value / max(r.value, 1e-30)}), flush=True)
    eng.close()


if __name__ == "__main__":
    # python tools/gemm_k7.py [reps [M N K]]
    a = [int(x) for x in sys.argv[1:]]
    main(a[0] if a else 50, tuple(a[1:4]) if len(a) >= 4 else None)
