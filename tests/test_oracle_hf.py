"""Pins the numeric oracle (oracle/numeric.py, builder-authored because the
reference computes no numbers -- SURVEY.md 8c) against a published
implementation of the same algorithm: transformers' LlamaForCausalLM
(transformers 5.5.0, default RoPE, SiLU-gated MLP, RMSNorm, GQA) in fp32,
loaded with the oracle's own hashed weights. The oracle runs the BatchPlan
semantics the B200 engine runs (prefill chunks over cached context, decode
entries at position C-1, a paged KV store keyed by position); HF runs the
whole token sequence at once with causal masking. In fp32 the two must agree
to float rounding: logits max-abs <= 1e-4 * max|logit| + 1e-5.

This is CPU-only test infrastructure: it pins the checker, the product never
imports transformers or the oracle."""
import numpy as np
import pytest

from oracle import numeric as N

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")

SHAPES = {
    # BASELINE config 1: 2 layers, d=256, 4 heads
    "config1": N.ModelShape(),
    # GQA G=4 and d=128 as at the Llama-3.1-8B shape (32/8 heads, theta 5e5), narrowed
    "gqa_d128": N.ModelShape(num_layers=2, hidden=512, n_heads=8, n_kv_heads=2, head_dim=128, ffn=1024, vocab=2048,
                             rope_theta=500000.0),
}


def hf_model(s: N.ModelShape, w: N.Weights):
    from transformers import LlamaConfig, LlamaForCausalLM
    cfg = LlamaConfig(vocab_size=s.vocab, hidden_size=s.hidden, intermediate_size=s.ffn, num_hidden_layers=s.num_layers,
                      num_attention_heads=s.n_heads, num_key_value_heads=s.n_kv_heads, head_dim=s.head_dim,
                      rms_norm_eps=s.rms_eps, rope_theta=s.rope_theta, tie_word_embeddings=False, attention_bias=False,
                      mlp_bias=False, max_position_embeddings=1 << 16, hidden_act="silu")
    m = LlamaForCausalLM(cfg).eval().float()
    H, D, Hq, Hkv = s.hidden, s.head_dim, s.n_heads, s.n_kv_heads
    sd = {"model.embed_tokens.weight": w.emb, "lm_head.weight": w.lm_head, "model.norm.weight": w.final_norm}
    for l in range(s.num_layers):
        p = f"model.layers.{l}."
        q = w.wqkv[l]
        sd[p + "self_attn.q_proj.weight"] = q[: Hq * D]
        sd[p + "self_attn.k_proj.weight"] = q[Hq * D: (Hq + Hkv) * D]
        sd[p + "self_attn.v_proj.weight"] = q[(Hq + Hkv) * D:]
        sd[p + "self_attn.o_proj.weight"] = w.wo[l]
        sd[p + "mlp.gate_proj.weight"] = w.wgu[l][: s.ffn]
        sd[p + "mlp.up_proj.weight"] = w.wgu[l][s.ffn:]
        sd[p + "mlp.down_proj.weight"] = w.wd[l]
        sd[p + "input_layernorm.weight"] = w.attn_norm[l]
        sd[p + "post_attention_layernorm.weight"] = w.mlp_norm[l]
    m.load_state_dict({k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)) for k, v in sd.items()},
                      strict=True)
    return m


@pytest.mark.parametrize("shape", sorted(SHAPES))
def test_oracle_matches_transformers_llama(shape):
    s = SHAPES[shape]
    w = N.Weights(s)
    m = hf_model(s, w)
    # two requests: A in three prefill chunks then two decodes (each plan
    # entry's last row = the logits HF gives at that position); B interleaved
    # in the same plans, so batching across entries is exercised too
    orc = N.Oracle(s, weights=w, mimic_bf16=False)
    plans = [
        [N.Entry(1, 40, 0, 0, True), N.Entry(0, 64, 0, 0, False)],
        [N.Entry(1, 30, 40, 0, True), N.Entry(0, 50, 64, 0, False)],
        [N.Entry(1, 1, 71, 1, True), N.Entry(0, 36, 114, 0, False)],
        [N.Entry(1, 1, 72, 1, True), N.Entry(0, 1, 151, 1, False)],
        [N.Entry(0, 1, 152, 1, False)],
    ]
    got, want = [], []
    n_tok = {0: 153, 1: 73}
    full = {}
    with torch.no_grad():
        for rid, n in n_tok.items():
            ids = N.token_id(s.token_seed, np.full(n, rid), np.arange(n), s.vocab)
            full[rid] = m(input_ids=torch.from_numpy(ids[None]).long()).logits[0].numpy()
    for plan in plans:
        lg = orc.forward(plan)
        for e, row in zip(plan, lg):
            last = int(N.entry_positions(e)[-1])
            got.append(row)
            want.append(full[e.request_id][last])
    got, want = np.array(got), np.array(want)
    err = float(np.max(np.abs(got - want)))
    assert err <= 1e-4 * float(np.max(np.abs(want))) + 1e-5, err
    assert (np.argmax(got, -1) == np.argmax(want, -1)).all()
