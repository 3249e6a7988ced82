"""KV-head-group sharding on the device: each rank's
weights, generated in place from the same seeded hashes, must be exactly the
rank's slice of the unsharded model -- Wqkv rows of its q/k/v heads, Wo
columns of its q heads, W_gate|up rows and W_down columns of its FFN slice --
and its KV block holds 1/g of a block. (The all-reduce itself needs >1 GPU;
the host allocator's rank agreement is covered by test_multirank.py.)"""
import numpy as np
import pytest

import paper_2410_01228_b200 as cs

pytestmark = pytest.mark.gpu

SHAPE = dict(num_layers=2, hidden=256, n_heads=8, n_kv_heads=4, head_dim=64, ffn=512, vocab=512)


def _weights(tp, rank):
    cfg = cs.model_config("tiny", tp_size=tp, tp_rank=rank, **SHAPE)
    eng = cs.Engine(cfg)
    try:
        return {k: eng.read_weight(1, k) for k in (1, 2, 4, 5)}, eng.block_bytes()
    finally:
        eng.close()


@pytest.mark.parametrize("tp", [2, 4])
def test_rank_weights_are_slices_of_the_full_model(tp):
    full, full_block = _weights(1, 0)
    H, Hq, Hkv, D, F = SHAPE["hidden"], SHAPE["n_heads"], SHAPE["n_kv_heads"], SHAPE["head_dim"], SHAPE["ffn"]
    wqkv = full[1].reshape((Hq + 2 * Hkv) * D, H)
    wo = full[2].reshape(H, Hq * D)
    wgu = full[4].reshape(2 * F, H)
    wd = full[5].reshape(H, F)
    hq, hkv, f = Hq // tp, Hkv // tp, F // tp
    for r in range(tp):
        w, blk = _weights(tp, r)
        q = wqkv[r * hq * D:(r + 1) * hq * D]
        k = wqkv[Hq * D + r * hkv * D:Hq * D + (r + 1) * hkv * D]
        v = wqkv[(Hq + Hkv) * D + r * hkv * D:(Hq + Hkv) * D + (r + 1) * hkv * D]
        assert np.array_equal(w[1].reshape(-1, H), np.concatenate([q, k, v]))
        assert np.array_equal(w[2].reshape(H, hq * D), wo[:, r * hq * D:(r + 1) * hq * D])
        assert np.array_equal(w[4].reshape(2 * f, H), np.concatenate([wgu[r * f:(r + 1) * f], wgu[F + r * f:F + (r + 1) * f]]))
        assert np.array_equal(w[5].reshape(H, f), wd[:, r * f:(r + 1) * f])
        assert blk * tp == full_block
