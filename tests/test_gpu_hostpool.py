"""Host-memory-limited regime on the device: the
reference's own config-1 runs with a 40- / 48-page host pool
(tests/golden/config1_host40, config1_host48) replayed through the engine
with the real gather / restore kernels. flush_checkpoints runs out of host
slots, so the host LRU drops older host copies and the recompute fallback
tags pages (kv_cache.cpp:326-362, 379-384); evicted requests restore from
what is left. Checks, after the run:
  * bookkeeping bit-exact with the reference (0 mismatches, page-table
    digests at every build) and the same final audit verdict;
  * the LRU and the recompute tagging really fired;
  * every page the reference holds on both sides ("both") has a host slot
    whose bytes equal the device block over the page's written positions
    (the copy a restore would bring back is the KV the forward wrote)."""
import json
import os

import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from paper_2410_01228_b200 import replay as R

from conftest import ROOT

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name", ["config1_host40", "config1_host48"])
def test_host_limited_replay_bit_exact(name):
    import torch
    g = os.path.join(GOLDEN, name)
    tr = R.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))
    eng = cs.Engine(R.engine_config_for(tr, "tiny", max_entries=256))
    try:
        res = R.run(eng, tr, 0, tr.n_iter, check_page_tables=True)
        assert res.mismatches == 0 and res.iterations == tr.n_iter
        torch.cuda.synchronize()
        st = eng.stats()
        assert st.host_lru_evicted_pages > 0 and st.recompute_tagged_tokens > 0
        m = json.load(open(os.path.join(g, "metrics.json")))
        assert st.total_d2h_bytes == m["transferred_bytes"]["d2h"]
        assert st.total_h2d_bytes == m["transferred_bytes"]["h2d"]
        verdict = "ok"
        try:
            eng.audit()
        except cs.CsLogicError as ex:
            verdict = str(ex)
        assert verdict == tr.audit
        checked = 0
        for rid, rq in tr.requests.items():
            try:
                pt = json.loads(eng.page_table_json(rid))
            except cs.CsError:
                continue  # released
            blocks, slots = eng.block_table(rid)
            done = rq["prefill_done"] + rq["decode_done"]
            # KV exists for processed positions only: the newest known token
            # of a decoding request is written by its next step
            written = done - (1 if rq["decode_done"] >= 1 else 0)
            for pg, page in enumerate(pt["pages"]):
                if page["location"] != "both" or slots[pg] < 0:
                    continue
                a, b = page["range"]
                n = min(b, written) - a
                if n <= 0:
                    continue
                L, H, D = 2, eng.cfg.n_kv_heads, eng.cfg.head_dim
                dev = eng.read_block(blocks[pg]).reshape(L, 2, H, 16, D)[:, :, :, :n]
                host = eng.read_host_slot(slots[pg]).reshape(L, 2, H, 16, D)[:, :, :, :n]
                assert np.array_equal(dev, host), (rid, pg)
                checked += 1
        assert checked > 0
    finally:
        eng.close()
