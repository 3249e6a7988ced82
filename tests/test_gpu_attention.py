"""Kernel-level parity of K1 (decode) and K2 (tcgen05 prefill) paged
attention at Llama-3.1-8B head shapes (32 q heads, 8 KV heads, d=128),
against an fp32 numpy reference computed from the device's own bf16 inputs:
q from the post-RoPE qkv activation, K/V read back from the HBM blocks the
block table names. Covers multi-tile causal chunks over a cached context,
partial pages, GQA grouping, several entries in one launch and the lazy
O-rescale path (a late, large score). Tolerance: rel-L2 <= 1e-2 per row
block (bf16 P/V products, fp32 accumulation)."""
import os

import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from oracle import numeric as N

pytestmark = pytest.mark.gpu

HQ, HKV, D = 32, 8, 128
G = HQ // HKV


def _engine(hq=HQ):
    # These checks recompute attention from the q in the qkv activation, so
    # they run the unfused path (rope_append rotates q in place); in a
    # decode-only graph the fused path rotates q inside K1 instead -- that
    # path is pinned bit for bit against this one by test_gpu_fusion.py.
    os.environ["CS_NO_FUSE"] = "1"
    try:
        return _engine_cfg(hq)
    finally:
        os.environ.pop("CS_NO_FUSE", None)


def _engine_cfg(hq):
    cfg = cs.model_config("tiny", num_layers=1, hidden=512, n_heads=hq, n_kv_heads=HKV, head_dim=D, ffn=512,
                          vocab=512, max_batched_tokens=4096, gpu_kv_capacity=(1 << 14) * 16 * 2 * HKV * D * 2,
                          rope_theta=500000.0, instrumented=0)
    return cs.Engine(cfg)


def _kv_of(eng, rid, n_pos):
    blocks, _ = eng.block_table(rid)
    K = np.zeros((n_pos, HKV, D), np.float32)
    V = np.zeros((n_pos, HKV, D), np.float32)
    for pg in range((n_pos + 15) // 16):
        blk = N.from_bf16_bits(eng.read_block(blocks[pg])).reshape(1, 2, HKV, 16, D)[0]
        n = min(16, n_pos - pg * 16)
        K[pg * 16:pg * 16 + n] = blk[0, :, :n].transpose(1, 0, 2)
        V[pg * 16:pg * 16 + n] = blk[1, :, :n].transpose(1, 0, 2)
    return K, V


def _ref_rows(q, K, V, positions):
    """q [T, hq, D] fp32; K/V [n, HKV, D]; row t attends keys [0, positions[t]]."""
    out = np.zeros_like(q)
    scale = 1.0 / np.sqrt(D)
    hq = q.shape[1]
    g = hq // HKV
    for t, pos in enumerate(positions):
        for h in range(hq):
            s = K[:pos + 1, h // g] @ q[t, h] * scale
            s = np.exp(s - s.max())
            out[t, h] = (s / s.sum()) @ V[:pos + 1, h // g]
    return out


def _run(eng, entries, allocs):
    for e, n in zip(entries, allocs):
        assert eng.allocate(e.request_id, n).ok
    eng.forward_launch(entries, 1)
    eng.iter_wait()
    for e in entries:
        eng.commit_allocations(e.request_id)


def _check_rows(eng, entries, row_pos, T, hq=HQ):
    qkv = N.from_bf16_bits(eng.read_activation(2, T, (hq + 2 * HKV) * D))
    got = N.from_bf16_bits(eng.read_activation(0, T, hq * D)).reshape(T, hq, D)
    row = 0
    for e, positions in zip(entries, row_pos):
        n = len(positions)
        K, V = _kv_of(eng, e.request_id, max(positions) + 1)
        q = qkv[row:row + n, :hq * D].reshape(n, hq, D)
        want = _ref_rows(q, K, V, positions)
        err = np.linalg.norm(got[row:row + n] - want) / np.linalg.norm(want)
        assert err <= 1e-2, (e, err)
        row += n


def test_k2_prefill_chunks_over_cached_context():
    eng = _engine()
    try:
        eng.register_request(0, False)
        eng.register_request(1, True)
        # chunk 1: 700 fresh tokens of request 0 (single-tile and multi-tile CTAs)
        e0 = cs.BatchEntry(0, 700, 0, cs.CS_PREFILL, False)
        _run(eng, [e0], [700])
        # chunk 2 of request 0 (C=700, P=1100: crosses 128-key tiles and partial
        # pages) next to a fresh 333-token online prefill
        e1 = cs.BatchEntry(1, 333, 0, cs.CS_PREFILL, True)
        e2 = cs.BatchEntry(0, 1100, 700, cs.CS_PREFILL, False)
        _run(eng, [e1, e2], [334, 1101])
        _check_rows(eng, [e1, e2], [list(range(333)), list(range(700, 1800))], 333 + 1100)
    finally:
        eng.close()


def test_k1_decode_and_k2_in_one_launch():
    eng = _engine()
    try:
        for r in range(5):
            eng.register_request(r, r == 0)
        ctx = [1, 17, 300, 2049, 4000]
        for r, c in enumerate(ctx):  # write context KV with a prefill of c tokens
            _run(eng, [cs.BatchEntry(r, c, 0, cs.CS_PREFILL, r == 0)], [c + 1])
        dec = [cs.BatchEntry(r, 1, c + 1, cs.CS_DECODE, r == 0) for r, c in enumerate(ctx)]
        eng.register_request(9, False)
        pre = cs.BatchEntry(9, 257, 0, cs.CS_PREFILL, False)
        _run(eng, dec + [pre], [1] * 5 + [257])
        _check_rows(eng, dec + [pre], [[c] for c in ctx] + [list(range(257))], 5 + 257)
    finally:
        eng.close()


@pytest.mark.parametrize("ctx", [
    [5, 1, 4000, 33, 2100, 16, 17, 900, 3999, 64] * 4,   # 40 rows: pairs cut by CTA ranges, CTAs over many pairs
    [7999],                                             # one long row: 8 pairs spread over many CTAs
    [300, 17, 2000, 1] * 15,                            # 60 rows = 480 pairs: the per-pair split-K kernel
])
def test_k1_stream_k_mixed_lengths(ctx):
    """K1 with fewer (entry, KV head) pairs than resident CTAs: the stream-K
    kernel splits the flattened pages of all pairs into equal ranges over one
    wave of CTAs; a pair cut by range boundaries is folded from its covering
    CTAs' partials. With more pairs: the per-pair split-K kernel. Decode-only
    plan = the CUDA-graph path; rows of 1..7999 context (partial pages,
    single-page pairs)."""
    eng = _engine()
    try:
        for r, c in enumerate(ctx):
            eng.register_request(r, r == 0)
            done = 0
            while done < c:  # write context KV with prefill chunks of <= 4000 tokens
                n = min(4000, c - done)
                _run(eng, [cs.BatchEntry(r, n, done, cs.CS_PREFILL, r == 0)], [n + (1 if done + n == c else 0)])
                done += n
        dec = [cs.BatchEntry(r, 1, c + 1, cs.CS_DECODE, r == 0) for r, c in enumerate(ctx)]
        for rep in range(2):  # the second step replays the captured graph
            _run(eng, dec, [1] * len(ctx))
            _check_rows(eng, dec, [[c + rep] for c in ctx], len(ctx))
            dec = [cs.BatchEntry(r, 1, c + 2, cs.CS_DECODE, r == 0) for r, c in enumerate(ctx)]
    finally:
        eng.close()


@pytest.mark.parametrize("hq", [40, 64])
def test_k1_k2_other_group_sizes(hq):
    """The Qwen-2.5-14B (40/8: G = 5) and Llama-3.1-70B (64/8: G = 8) head
    groupings, whose K1 / K2 template instances the 8B tests never launch:
    decode rows (stream-K K1) and a multi-tile prefill chunk in one plan."""
    eng = _engine(hq)
    try:
        for r in range(4):
            eng.register_request(r, r == 0)
        ctx = [1, 300, 2049, 4000]
        for r, c in enumerate(ctx):
            _run(eng, [cs.BatchEntry(r, c, 0, cs.CS_PREFILL, r == 0)], [c + 1])
        dec = [cs.BatchEntry(r, 1, c + 1, cs.CS_DECODE, r == 0) for r, c in enumerate(ctx)]
        eng.register_request(9, False)
        pre = cs.BatchEntry(9, 700, 0, cs.CS_PREFILL, False)
        _run(eng, dec + [pre], [1] * 4 + [700])
        _check_rows(eng, dec + [pre], [[c] for c in ctx] + [list(range(700))], 4 + 700, hq)
        # and the per-pair split-K K1 kernel: 60 decode rows x 8 heads > resident stream-K CTAs
        dec2 = []
        for r in range(60):
            eng.register_request(100 + r, False)
            _run(eng, [cs.BatchEntry(100 + r, 200 + r, 0, cs.CS_PREFILL, False)], [201 + r])
            dec2.append(cs.BatchEntry(100 + r, 1, 201 + r, cs.CS_DECODE, False))
        _run(eng, dec2, [1] * 60)
        _check_rows(eng, dec2, [[200 + r] for r in range(60)], 60, hq)
    finally:
        eng.close()


def test_k2_lazy_rescale_path():
    """A key late in the sequence with a much larger score than everything
    before forces the O-in-TMEM correction (max grows by > 2^8 in log2 units)."""
    eng = _engine()
    try:
        eng.register_request(0, False)
        _run(eng, [cs.BatchEntry(0, 600, 0, cs.CS_PREFILL, False)], [600])
        # blow up K at position 500 for every head: huge positive dot with q
        blocks, _ = eng.block_table(0)
        blk = N.from_bf16_bits(eng.read_block(blocks[500 // 16])).reshape(2, HKV, 16, D)
        qkv = N.from_bf16_bits(eng.read_activation(2, 600, (HQ + 2 * HKV) * D))
        for h in range(HKV):
            qv = qkv[550, h * G * D:(h * G + 1) * D]
            blk[0, h, 500 % 16] = 40.0 * np.sign(qv)
        eng.write_block(blocks[500 // 16], N.bf16_bits(blk.reshape(-1)))
        # a second chunk attends over the modified cache
        e = cs.BatchEntry(0, 300, 600, cs.CS_PREFILL, False)
        _run(eng, [e], [300])
        _check_rows(eng, [e], [list(range(600, 900))], 300)
    finally:
        eng.close()


def test_k2_split_k_small_chunks_over_long_context():
    """Few prefill rows over a long context launch fewer CTAs than SMs: K2
    splits the key range (split-K + merge), including splits that hold no
    visible key for a short entry (empty partials)."""
    eng = _engine()
    try:
        eng.register_request(0, False)
        eng.register_request(1, False)
        eng.register_request(2, True)
        _run(eng, [cs.BatchEntry(0, 4000, 0, cs.CS_PREFILL, False)], [4000])
        e_on = cs.BatchEntry(2, 30, 0, cs.CS_PREFILL, True)        # short: 1 key tile
        e_long = cs.BatchEntry(0, 20, 4000, cs.CS_PREFILL, False)  # 20 rows over 4020 keys
        _run(eng, [e_on, e_long], [30, 20])
        _check_rows(eng, [e_on, e_long], [list(range(30)), list(range(4000, 4020))], 50)
        e3 = cs.BatchEntry(1, 700, 0, cs.CS_PREFILL, False)
        _run(eng, [e3], [700])
        e4 = cs.BatchEntry(0, 40, 4020, cs.CS_PREFILL, False)
        _run(eng, [e4], [40])
        _check_rows(eng, [e4], [list(range(4020, 4060))], 40)
    finally:
        eng.close()


def test_k2_recompute_of_discarded_pages():
    """Recompute entries (kv_cache.cpp:76-107, scheduler.cpp:286): every page of
    an offline request is discarded, then re-materialised head-first in two
    whole-page chunks (recompute_chunk, the last page partial); each chunk's
    rows sit at the positions of its pages and attend causally over the
    already re-materialised prefix. A decode after the recompute reads the
    rebuilt KV."""
    eng = _engine()
    try:
        eng.register_request(0, False)
        _run(eng, [cs.BatchEntry(0, 700, 0, cs.CS_PREFILL, False)], [700])
        st = eng.discard_request(0)
        assert st.discarded_tokens == 700
        done = 0
        for cap in (320, 4096):
            n = eng.recompute_chunk(0, 700 - done, cap)
            assert n > 0 and (n % 16 == 0 or done + n == 700)
            e = cs.BatchEntry(0, n, 700, cs.CS_RECOMPUTE, False)
            _run(eng, [e], [n])
            _check_rows(eng, [e], [list(range(done, done + n))], n)
            done += n
        assert done == 700 and eng.recompute_chunk(0, 1, 4096) == 0
        dec = cs.BatchEntry(0, 1, 700, cs.CS_DECODE, False)
        _run(eng, [dec], [1])
        _check_rows(eng, [dec], [[699]], 1)
        eng.audit()
    finally:
        eng.close()
