"""Short, single-GPU drivers for ncu captures of the hot-path kernels.

  python tools/ncu_targets.py decode    # K1: 64 seqs x 4224 ctx, Llama-3.1-8B heads
  python tools/ncu_targets.py prefill   # K2: one 2048-token chunk over 4096 cached
  python tools/ncu_targets.py gather    # K4: checkpoint gather of 1024 whole blocks
  python tools/ncu_targets.py gemm      # K8: 8192-token prefill forwards of the full 8B

Each target launches its kernel a handful of times (ncu replays each launch);
the numbers printed here are NOT bench values.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01228_b200 as cs  # noqa: E402
from paper_2410_01228_b200 import _ffi as F  # noqa: E402


def _engine(**kw):
    cfg = cs.model_config("llama8b", hidden=512, ffn=512, vocab=512, gpu_kv_capacity=80 << 30,
                          host_kv_capacity=4 << 30, max_batched_tokens=8192, instrumented=0, **kw)
    return cs.Engine(cfg)


def bench_attention(eng, plan, reps):
    arr = (F.cs_batch_entry * len(plan))(*plan)
    ms, b, f = C.c_double(), C.c_int64(), C.c_int64()
    cs.engine._check(cs.lib().cs_bench_attention(eng._h, arr, len(plan), reps, C.byref(ms), C.byref(b), C.byref(f)))
    return ms.value, b.value, f.value


def decode(reps=3, n=64, ctx=4224):
    eng = _engine()
    plan = []
    for r in range(n):
        eng.register_request(r, False)
        assert eng.allocate(r, ctx + 1).ok
        eng.commit_allocations(r)
        plan.append(F.cs_batch_entry(r, 1, ctx, F.CS_DECODE, 0))
    ms, b, _ = bench_attention(eng, plan, reps)
    print(f"decode: {ms:.4f} ms/launch, {b} B, {b / ms / 1e6:.1f} GB/s")
    eng.close()


def prefill(reps=3, P=2048, ctx=4096):
    eng = _engine()
    eng.register_request(0, False)
    assert eng.allocate(0, ctx + P).ok
    eng.commit_allocations(0)
    ms, _, f = bench_attention(eng, [F.cs_batch_entry(0, P, ctx, F.CS_PREFILL, 0)], reps)
    print(f"prefill: {ms:.4f} ms/launch, {f} flop, {f / ms / 1e9:.1f} TFLOP/s")
    eng.close()


def gather(n_blocks=1024):
    eng = _engine()
    eng.register_request(0, False)
    assert eng.allocate(0, n_blocks * 16).ok
    eng.commit_allocations(0)
    eng.note_written(0, 0, n_blocks * 16)
    eng.stage_checkpoint(0, 0, n_blocks * 16)
    job = eng.flush_checkpoints(0)
    eng.job_wait(job.id)
    eng.on_transfer_done(job.id, job.done_time)
    s = eng.stats()
    print(f"gather: {s.moved_d2h_bytes} B in {s.moved_d2h_ms:.3f} ms = {s.moved_d2h_bytes / s.moved_d2h_ms / 1e6:.1f} GB/s")
    eng.close()


def step(n=32, ctx=4096, reps=3):
    """A decode-only forward of the full Llama-3.1-8B (the CUDA-graph path):
    n sequences at ctx tokens of context."""
    cfg = cs.model_config("llama8b", gpu_kv_capacity=60 << 30, host_kv_capacity=1 << 30, max_batched_tokens=8192,
                          instrumented=0, max_entries=256)
    eng = cs.Engine(cfg)
    for r in range(n):
        eng.register_request(r, False)
        assert eng.allocate(r, ctx).ok
        eng.commit_allocations(r)
    for rep in range(reps):
        for r in range(n):
            assert eng.allocate(r, 1).ok
        info = eng.forward([cs.BatchEntry(r, 1, ctx + rep + 1, cs.CS_DECODE, False) for r in range(n)], epoch=rep + 1)
        for r in range(n):
            eng.commit_allocations(r)
        print(f"step rep {rep}: {info.gpu_ms:.3f} ms", flush=True)
    eng.close()


def gemm(P=8192, reps=2):
    """Prefill forwards of the full Llama-3.1-8B over one P-token chunk: the
    layer projections run on K8 (gemm_pf_kernel, gate|up with the fused
    SwiGLU epilogue)."""
    cfg = cs.model_config("llama8b", gpu_kv_capacity=8 << 30, host_kv_capacity=1 << 30, max_batched_tokens=8192,
                          instrumented=0, max_entries=256)
    eng = cs.Engine(cfg)
    for rep in range(reps):
        eng.register_request(rep, False)
        assert eng.allocate(rep, P).ok
        info = eng.forward([cs.BatchEntry(rep, P, 0, cs.CS_PREFILL, False)], epoch=rep + 1)
        eng.commit_allocations(rep)
        print(f"prefill forward {P} tokens: {info.gpu_ms:.3f} ms", flush=True)
    eng.close()


if __name__ == "__main__":
    # optional integer arguments are passed through, e.g. `step 92 4130`
    {"decode": decode, "prefill": prefill, "gather": gather, "step": step, "gemm": gemm}[sys.argv[1]](*map(int, sys.argv[2:]))
