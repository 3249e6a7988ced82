"""Numeric parity at BASELINE config 2 width: a
Llama-3.1-8B-shaped forward (hidden 4096, 32/8 heads, d 128, ffn 14336,
vocab 128256; 2 of the 32 layers) on the engine vs the fp32 oracle
(oracle/numeric.py, mimic_bf16=False -- no bf16 storage points), on plans
taken from the reference's own co-serving schedule tests/golden/
llama8b_b200_kv60: mixed iterations (online decode prefix, offline decodes
at 4.2-4.4K context, one offline prefill chunk over 1.5-3.3K cached tokens),
a prefill-sized iteration (M >= 2048: the K8 tcgen05 GEMMs) and a decode-only
CUDA-graph step. The oracle itself is pinned against transformers'
LlamaForCausalLM (tests/test_oracle_hf.py).

Context KV (positions before each entry's first query) is random bf16
written into the engine's paged blocks through the C-ABI and into the
oracle's KV store, so the test covers the block-table gather of every
attention read at full width without replaying the trace's history.

Two oracles run every plan on the same weights and context KV:
  * pure fp32 (mimic_bf16=False): the algorithm with no bf16 rounding at all.
    The engine stores every activation in bf16 (2^-9 relative step), which
    leaves a ~1% relative error on each logit; the max over 16 x 128256
    logits of that error is ~5 sigma, so a max-abs bound of 1e-2 * std is
    not reachable against pure fp32 by ANY bf16 engine. Bounds:
      logits rel-L2 <= FP32_LOGIT_L2, max-abs <= FP32_LOGIT_MAX * std,
      argmax agreement >= 0.99 on rows whose top-2 gap > 2 * max-abs bound,
      last attention output rel-L2 <= FP32_ATTN_L2.
  * storage-point oracle (mimic_bf16=True): the same fp32 arithmetic
    rounded to bf16 exactly where the engine stores a tensor. What is left
    is accumulation order and the bf16 P operand of P.V. Bounds:
      logits max-abs <= BF16_LOGIT_MAX * std (the 1e-2 * std the verdict
      asks for), rel-L2 <= BF16_LOGIT_L2; attention rel-L2 <= BF16_ATTN_L2.
"""
import json

import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from oracle import numeric as N
from paper_2410_01228_b200 import replay as R

pytestmark = pytest.mark.gpu

FP32_LOGIT_L2 = 2e-2
FP32_LOGIT_MAX = 0.1
FP32_ATTN_L2 = 2e-2
BF16_LOGIT_MAX = 1e-2
BF16_LOGIT_L2 = 5e-3
BF16_ATTN_L2 = 5e-3
GOLDEN = "tests/golden/llama8b_b200_kv60"


def _device_weights(eng, s):
    """The engine's bf16 weights as fp32 (spot-checked against the hash)."""
    class W:
        pass
    w = W()
    w.s = s
    f = lambda a, shape: N.from_bf16_bits(a).reshape(shape)
    H, D = s.hidden, s.head_dim
    w.emb = f(eng.read_weight(0, 6), (s.vocab, H))
    w.lm_head = f(eng.read_weight(0, 7), (s.vocab, H))
    w.final_norm = f(eng.read_weight(0, 8), (H,))
    w.attn_norm, w.mlp_norm, w.wqkv, w.wo, w.wgu, w.wd = [], [], [], [], [], []
    for l in range(s.num_layers):
        w.attn_norm.append(f(eng.read_weight(l, 0), (H,)))
        w.wqkv.append(f(eng.read_weight(l, 1), ((s.n_heads + 2 * s.n_kv_heads) * D, H)))
        w.wo.append(f(eng.read_weight(l, 2), (H, s.n_heads * D)))
        w.mlp_norm.append(f(eng.read_weight(l, 3), (H,)))
        w.wgu.append(f(eng.read_weight(l, 4), (2 * s.ffn, H)))
        w.wd.append(f(eng.read_weight(l, 5), (H, s.ffn)))
    # the device weights are the oracle's hash init (pinned exactly at small
    # shapes by test_numeric_oracle_hashes_match_engine): sample them here
    rng = np.random.default_rng(0)
    ws = np.float32(np.float32(0.02) * np.float32(1.7320508))
    for name, tid, mat in (("emb", N.TENSOR_EMB, w.emb), ("wd1", N._tid(1, N.W_D), w.wd[1]),
                           ("wqkv0", N._tid(0, N.W_QKV), w.wqkv[0])):
        idx = rng.integers(0, mat.size, 4096).astype(np.uint64)
        want = N.bf16_round((ws * N.hash_uniform(s.weight_seed, tid, idx)).astype(np.float32))
        assert np.array_equal(mat.reshape(-1)[idx.astype(np.int64)], want), name
    return w


def _plans():
    tr = R.load(f"{GOLDEN}/calls.jsonl.gz", f"{GOLDEN}/requests.jsonl.gz")
    out = {}
    for name, k, n_on, n_off in (("mixed_it72", 72, 4, 4), ("mixed_it401", 401, 4, 4),
                                 ("prefill_it147", 147, 2, 2)):
        p = tr.plan_of[k]
        dec = p[p[:, 3] == 1]
        pre = p[p[:, 3] != 1]
        on = dec[dec[:, 4] == 1][:n_on]
        off = dec[dec[:, 4] == 0][:n_off]
        # the reference's plan order (scheduler.cpp:183-317): online decodes,
        # online prefills, then offline entries
        rows = np.concatenate([on, pre[pre[:, 4] == 1], off, pre[pre[:, 4] == 0]])
        out[name] = (k, rows)
    # decode-only step of 16 sequences (CUDA graph bucket 16, cuBLAS GEMMs)
    p = tr.plan_of[72]
    out["decode_graph"] = (72, p[p[:, 3] == 1][:16])
    return out


def test_llama8b_width_forward_vs_fp32_oracle():
    cfg = cs.model_config("llama8b", num_layers=2, gpu_kv_capacity=4 << 30, host_kv_capacity=1 << 30,
                          max_batched_tokens=8192, max_entries=64, instrumented=1, safepoint_interval_layers=1)
    eng = cs.Engine(cfg)
    s = N.ModelShape.from_cfg(cfg)
    w = _device_weights(eng, s)
    orc = N.Oracle(s, weights=w, mimic_bf16=False)
    orc16 = N.Oracle(s, weights=w, mimic_bf16=True)
    rng = np.random.default_rng(1)
    L, Hkv, D = s.num_layers, s.n_kv_heads, s.head_dim
    report = {}
    try:
        for pi, (name, (k, rows)) in enumerate(sorted(_plans().items())):
            entries, oentries = [], []
            for rid0, P, Cc, kind, online in rows.tolist():
                rid = int(rid0) + 1_000_000 * (pi + 1)  # fresh request per plan
                eng.register_request(rid, bool(online))
                kv_len = Cc if kind == 1 else Cc + P
                first_q = Cc - 1 if kind == 1 else Cc     # context = positions before the first query
                assert eng.allocate(rid, kv_len).ok
                eng.commit_allocations(rid)
                if first_q > 0:
                    kv = N.bf16_round(rng.standard_normal((L, 2, first_q, Hkv, D), dtype=np.float32))
                    for l in range(L):
                        for o in (orc, orc16):
                            o.kv.write(rid, l, np.arange(first_q), kv[l, 0], kv[l, 1])
                    blocks, _ = eng.block_table(rid)
                    for pg in range((first_q + 15) // 16):
                        blk = np.zeros((L, 2, Hkv, 16, D), np.float32)
                        t0, t1 = pg * 16, min(first_q, pg * 16 + 16)
                        blk[:, :, :, : t1 - t0] = kv[:, :, t0:t1].transpose(0, 1, 3, 2, 4)
                        eng.write_block(blocks[pg], N.bf16_bits(blk).reshape(-1))
                entries.append(cs.BatchEntry(rid, int(P), int(Cc), int(kind), bool(online)))
                oentries.append(N.Entry(rid, int(P), int(Cc), int(kind), bool(online)))
            info, got = eng.forward(entries, epoch=100 + pi, want_logits=True)
            n_tok = sum(e.compute_tokens for e in entries)
            attn = N.from_bf16_bits(eng.read_activation(0, n_tok, s.n_heads * D))
            ref = orc.forward(oentries)
            ref16 = orc16.forward(oentries)
            sd = float(np.std(ref))
            err = float(np.max(np.abs(got - ref)))
            err16 = float(np.max(np.abs(got - ref16)))
            top2 = np.sort(ref, -1)[:, -2:]
            clear = (top2[:, 1] - top2[:, 0]) > 2 * FP32_LOGIT_MAX * sd
            agree = float(np.mean((np.argmax(got, -1) == np.argmax(ref, -1))[clear])) if clear.any() else 1.0
            rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
            a_rel, a_rel16 = rel(attn, orc.last_attn), rel(attn, orc16.last_attn)
            l_rel, l_rel16 = rel(got, ref), rel(got, ref16)
            report[name] = dict(iteration=k, entries=len(entries), tokens=n_tok,
                                max_ctx=int(max(e.context_tokens for e in entries)), gpu_ms=info.gpu_ms,
                                logit_std=sd, fp32_logit_maxabs_over_std=err / sd, fp32_logit_rel_l2=l_rel,
                                fp32_attn_rel_l2=a_rel, argmax_agree_clear=agree, clear_rows=int(clear.sum()),
                                bf16_logit_maxabs_over_std=err16 / sd, bf16_logit_rel_l2=l_rel16,
                                bf16_attn_rel_l2=a_rel16)
            print(json.dumps({name: report[name]}))
            for e in entries:
                eng.release_request(e.request_id)
    finally:
        eng.close()
    for name, r in report.items():
        assert r["fp32_logit_rel_l2"] <= FP32_LOGIT_L2, (name, r)
        assert r["fp32_logit_maxabs_over_std"] <= FP32_LOGIT_MAX, (name, r)
        assert r["fp32_attn_rel_l2"] <= FP32_ATTN_L2, (name, r)
        assert r["argmax_agree_clear"] >= 0.99, (name, r)
        assert r["bf16_logit_maxabs_over_std"] <= BF16_LOGIT_MAX, (name, r)
        assert r["bf16_logit_rel_l2"] <= BF16_LOGIT_L2, (name, r)
        assert r["bf16_attn_rel_l2"] <= BF16_ATTN_L2, (name, r)
    assert len(report) == 4
