"""K4/K5 checkpoint gather + restore scatter: bit-exact host copies of every
written KV position and bit-exact restore into fresh blocks (SURVEY.md 8a
A8/A10), with the reference's byte accounting intact."""
import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from helpers import Driver

pytestmark = pytest.mark.gpu


def _positions_view(eng, block_u16):
    c = eng.cfg
    hkv = c.n_kv_heads // c.tp_size
    return block_u16.reshape(c.num_layers, 2, hkv, 16, c.head_dim)


def test_checkpoint_then_restore_is_bit_exact():
    drv = Driver(cs.model_config("tiny"), oracle=False)
    drv.add(0, 45, online=False)
    drv.step([(0, None)], want_logits=False)          # prefill 45 (+1 first-token slot)
    eng = drv.eng
    eng.stage_checkpoint(0, 0, 46)                     # reference stages known tokens [0, 46)
    job = eng.flush_checkpoints(1000)
    assert job is not None and job.bytes == 46 * 2048  # reference bytes (known tokens)
    assert job.moved_bytes == 45 * 2048                # only written KV crosses the link
    eng.on_transfer_done(job.id, job.done_time)
    blocks, slots = eng.block_table(0)
    before = {b: eng.read_block(b) for b in blocks}
    for pg, (b, s) in enumerate(zip(blocks, slots)):
        dev = _positions_view(eng, before[b])
        host = _positions_view(eng, eng.read_host_slot(s))
        n = min(16, 45 - pg * 16)
        assert np.array_equal(dev[:, :, :, :n], host[:, :, :, :n]), pg
    # decode 3 tokens; each stage maps known [C, C+1) onto written C-1
    for _ in range(3):
        c0 = drv.known[0]
        drv.step([(0, None)], want_logits=False)
        eng.stage_checkpoint(0, c0, c0 + 1)
        j = eng.flush_checkpoints(2000)
        assert j is not None and j.moved_bytes == 2048
        eng.on_transfer_done(j.id, j.done_time)
    blocks, slots = eng.block_table(0)
    written = 45 + 3
    snap = [eng.read_block(b) for b in blocks]
    # pause + evict: everything except the last partial page is host-complete
    eng.on_request_paused(0, 1)
    ev = eng.evict_request_gpu(0)
    assert ev.freed_pages >= 1
    cost = eng.resume_cost(0)
    assert cost.host_only_pages == ev.freed_pages
    eng.fill_pool(1234)                                 # clobber every block
    pf = eng.start_prefetch(0, 5000)
    assert pf is not None
    eng.on_transfer_done(pf.id, pf.done_time)
    assert eng.fully_resident(0)
    nb, _ = eng.block_table(0)
    for pg in range(len(nb)):
        n = min(16, written - pg * 16)
        if n <= 0:
            continue
        got = _positions_view(eng, eng.read_block(nb[pg]))
        want = _positions_view(eng, snap[pg])
        if pg < ev.freed_pages:  # restored pages
            assert np.array_equal(got[:, :, :, :n], want[:, :, :, :n]), pg
    eng.audit()
    s = eng.stats()
    assert s.moved_d2h_ms > 0 and s.moved_h2d_ms > 0
    drv.close()
