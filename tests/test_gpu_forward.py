"""GPU parity of the layer forward (K1 decode attention, K2 prefill attention,
K3 RoPE + KV append, norms, GEMMs, lm_head) against the CPU oracle, through
the C-ABI. Tolerances (bf16 engine vs fp32 oracle with bf16 storage points):
attention output rel-L2 <= 1e-2; logits max-abs <= min(2e-2, 0.06 x std of
the oracle logits); argmax agreement >= 99% on rows whose oracle top-2 gap
exceeds twice that bound (helpers.logit_bound / decisive_rows)."""
import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from helpers import DECISIVE_AGREE, Driver, decisive_rows, logit_bound, rel_l2

pytestmark = pytest.mark.gpu

ATTN_TOL = 1e-2
LOGIT_TOL = 2e-2


def _check(drv, info, logits, ref, attn_rows=None):
    assert ref is not None
    assert logits.shape == ref.shape
    err = float(np.max(np.abs(logits - ref)))
    bound = logit_bound(ref)
    assert err <= bound, (err, bound)
    ok, dec = decisive_rows(logits, ref, bound)
    assert ok >= DECISIVE_AGREE * dec, (ok, dec)
    if attn_rows is not None:
        c = drv.cfg
        got = drv.eng.read_activation(0, attn_rows, c.n_heads * c.head_dim)
        from oracle import numeric as N
        got = N.from_bf16_bits(got)
        want = drv.orc.last_attn
        assert rel_l2(got, want) <= ATTN_TOL, rel_l2(got, want)


def test_tiny_mixed_prefill_decode():
    drv = Driver(cs.model_config("tiny"))
    drv.add(0, 40, online=False)
    drv.add(1, 20, online=True)
    drv.add(2, 33, online=False)
    info, lg, ref = drv.step([(1, None), (0, None), (2, 17)])
    _check(drv, info, lg, ref, attn_rows=20 + 40 + 17)
    info, lg, ref = drv.step([(1, None), (0, None), (2, None)])
    _check(drv, info, lg, ref, attn_rows=1 + 1 + 16)
    for _ in range(3):
        info, lg, ref = drv.step([(1, None), (0, None), (2, None)])
        _check(drv, info, lg, ref, attn_rows=3)
    drv.eng.audit()
    drv.close()


@pytest.mark.parametrize("heads,kv_heads", [(32, 8), (40, 8), (64, 8), (16, 16)])
def test_gqa_shapes_d128(heads, kv_heads):
    cfg = cs.model_config("tiny", num_layers=2, hidden=512, n_heads=heads, n_kv_heads=kv_heads, head_dim=128,
                          ffn=512, vocab=512, max_batched_tokens=2048, gpu_kv_capacity=4096 * 16 * 2 * 2 * 2 * kv_heads * 128,
                          rope_theta=500000.0)
    drv = Driver(cfg)
    for r in range(6):
        drv.add(r, 100 + 37 * r, online=r < 2)
    info, lg, ref = drv.step([(0, None), (1, None), (2, None), (3, None), (4, 64), (5, 200)])
    _check(drv, info, lg, ref)
    for _ in range(2):
        info, lg, ref = drv.step([(0, None), (1, None), (2, None), (3, None), (4, None), (5, None)])
        _check(drv, info, lg, ref)
    drv.close()


def test_long_context_split_decode():
    """Decode over ~3K tokens of context with few sequences -> split-K path."""
    cfg = cs.model_config("tiny", num_layers=2, hidden=256, n_heads=32, n_kv_heads=8, head_dim=128, ffn=256,
                          vocab=256, max_batched_tokens=1024, gpu_kv_capacity=8192 * 2 * 2 * 2 * 8 * 128,
                          rope_theta=500000.0)
    drv = Driver(cfg)
    drv.add(0, 2900, online=False)
    drv.add(1, 700, online=True)
    for _ in range(3):
        drv.step([(0, 1000)], want_logits=False)
    drv.step([(1, None)], want_logits=False)
    for _ in range(3):
        info, lg, ref = drv.step([(1, None), (0, None)])
        _check(drv, info, lg, ref, attn_rows=2)
    drv.close()
