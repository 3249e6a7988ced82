"""K8 epilogue fusions (csrc/gemm_pf.cu): on single-rank
prefill layers the qkv projection applies RoPE and appends k / v to the KV
pool in its epilogue (no rope_append launch), and o_proj / down add the
residual in place (no separate add). Both are designed to round exactly
where the unfused kernels store (bf16 qkv / projection outputs, the same
fma/mul rotation), so a fused engine must reproduce the unfused engine BIT
FOR BIT: logits and every written KV block, over a Llama-3.1-8B-width
2-layer model, a 2048-token prefill chunk (K8 path) followed by a chunk over
that cached context, a mixed decode+prefill iteration, and decode-only
CUDA-graph steps (where K1 rotates q and appends the new token's k / v)."""
import os

import numpy as np
import pytest

import paper_2410_01228_b200 as cs

pytestmark = pytest.mark.gpu


def _engine(fused):
    # both engines must run the same, deterministic GEMM kernels: K7 for
    # every M <= 256 projection (a fixed-order DSMEM reduction), K8 above; no
    # start-up timing (which may choose differently per engine) and no
    # cuBLASLt (whose split-K reductions need not be bitwise reproducible)
    env = {"CS_NO_FUSE": "0" if fused else "1", "CS_NO_GEMM_TUNE": "1", "CS_WGEMM": "1"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        cfg = cs.model_config("llama8b", num_layers=2, gpu_kv_capacity=2 << 30, host_kv_capacity=1 << 28,
                              max_batched_tokens=8192, max_entries=64, instrumented=0)
        return cs.Engine(cfg)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v


def _run(eng):
    outs = []
    eng.register_request(0, False)
    eng.register_request(1, True)
    steps = [
        ([cs.BatchEntry(0, 2048, 0, cs.CS_PREFILL, False)], [(0, 2048)]),
        ([cs.BatchEntry(0, 2100, 2048, cs.CS_PREFILL, False)], [(0, 2101)]),
        ([cs.BatchEntry(1, 2200, 0, cs.CS_PREFILL, True), cs.BatchEntry(0, 1, 4149, cs.CS_DECODE, False)],
         [(1, 2201), (0, 1)]),
    ]
    # decode-only steps (CUDA graphs): RoPE of q and the new token's K/V
    # append run inside K1 instead of rope_append
    for k in range(3):
        steps.append(([cs.BatchEntry(1, 1, 2201 + k, cs.CS_DECODE, True),
                       cs.BatchEntry(0, 1, 4150 + k, cs.CS_DECODE, False)], [(1, 1), (0, 1)]))
    for ep, (plan, allocs) in enumerate(steps):
        for rid, n in allocs:
            assert eng.allocate(rid, n).ok
        eng.forward_launch(plan, ep + 1)
        _, logits = eng.iter_wait(want_logits=True)
        for rid, _ in allocs:
            eng.commit_allocations(rid)
        outs.append(np.array(logits))
    blocks = {}
    for rid in (0, 1):
        b, _ = eng.block_table(rid)
        blocks[rid] = [np.array(eng.read_block(x)) for x in b if x >= 0]
    return outs, blocks


def test_fused_epilogues_are_bit_identical_to_unfused_kernels():
    a = _engine(fused=False)
    try:
        la, ba = _run(a)
    finally:
        a.close()
    b = _engine(fused=True)
    try:
        lb, bb = _run(b)
    finally:
        b.close()
    for x, y in zip(la, lb):
        assert x.shape == y.shape
        assert np.array_equal(x, y)
    for rid in (0, 1):
        assert len(ba[rid]) == len(bb[rid])
        for x, y in zip(ba[rid], bb[rid]):
            assert np.array_equal(x, y)
