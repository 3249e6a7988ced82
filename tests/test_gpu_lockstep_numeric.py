"""Numeric parity on the reference's own co-serving runs (GPU).

Every iteration of a recorded reference run (tests/golden/config1*, the
tiny config-1 decoder of SURVEY.md 8d) is replayed op by op through the
engine -- the same KvCacheManager calls, dispatches, preemption signals,
checkpoints, evictions, restores and recomputes the reference issued -- and
the logits of every surviving entry are compared with the fp32 CPU oracle run
on the same plan (teacher-forced ids). The KV that attention reads has been
through the device's checkpoint gather, eviction and restore scatter, so this
checks those paths numerically end to end. Tolerance (bf16 engine vs fp32
oracle with bf16 storage points): logits max-abs <= 2e-2 per iteration,
argmax agreement >= 99% over the run's decisive rows (oracle top-2 gap above
twice the logit bound, helpers.logit_bound)."""
import os

import numpy as np
import pytest

import paper_2410_01228_b200 as cs
from oracle import numeric as N
from paper_2410_01228_b200 import replay as R

from conftest import ROOT
from helpers import DECISIVE_AGREE, decisive_rows, logit_bound

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(ROOT, "tests", "golden")
OPC = R.OPC


def _replay_with_oracle(name):
    g = os.path.join(GOLDEN, name)
    tr = R.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))
    cfg = R.engine_config_for(tr, "tiny", max_entries=256)
    eng = cs.Engine(cfg)
    orc = N.Oracle(N.ModelShape.from_cfg(cfg))
    plans = tr.plans
    epoch = 5000
    inflight = None   # (entries, signal_armed)
    worst, agree, rows, iters, drops = 0.0, 0, 0, 0, 0
    try:
        for o in tr.ops:
            c = int(o[0])
            if c == OPC["register"]:
                eng.register_request(int(o[1]), bool(o[2]))
            elif c == OPC["allocate"]:
                r = eng.allocate(int(o[1]), int(o[2]), int(o[3]))
                assert (r.ok, r.shortfall_pages) == (bool(o[4]), int(o[5]))
            elif c == OPC["commit"]:
                eng.commit_allocations(int(o[1]))
            elif c == OPC["rollback"]:
                eng.rollback_allocations(int(o[1]))
            elif c == OPC["evict"]:
                eng.evict_request_gpu(int(o[1]), int(o[2]), int(o[3]))
            elif c == OPC["discard"]:
                eng.discard_request(int(o[1]), int(o[2]))
            elif c == OPC["release_on_demand"]:
                eng.release_offline_pages_on_demand(int(o[1]), int(o[2]))
            elif c == OPC["stage"]:
                eng.stage_checkpoint(int(o[1]), int(o[2]), int(o[3]))
            elif c == OPC["flush"]:
                eng.flush_checkpoints(int(o[1]))
            elif c == OPC["prefetch"]:
                eng.start_prefetch(int(o[7]), int(o[1]))
            elif c == OPC["done"]:
                eng.on_transfer_done(int(o[1]), int(o[2]))
            elif c == OPC["paused"]:
                eng.on_request_paused(int(o[1]), int(o[2]))
            elif c == OPC["active"]:
                eng.on_request_active(int(o[1]))
            elif c == OPC["release"]:
                eng.release_request(int(o[1]))
            elif c == OPC["dispatch"]:
                off, n = int(o[1]), int(o[2])
                entries = [cs.BatchEntry(int(p[0]), int(p[1]), int(p[2]), int(p[3]), bool(p[4]))
                           for p in plans[off:off + n]]
                epoch += 1
                eng.forward_launch(entries, epoch)
                inflight = (entries, bool(o[3]))
            elif c == OPC["signal"]:
                if inflight and inflight[1]:
                    eng.preempt_signal(epoch)
                    inflight = (inflight[0], False)
            elif c == OPC["iter_end"] and inflight:
                entries = inflight[0]
                info, logits = eng.iter_wait(want_logits=True)
                inflight = None
                dropped = info.preempted_at_layer is not None
                drops += dropped
                alive = [e for e in entries if e.online or not dropped]
                keep = [i for i, e in enumerate(alive) if e.kind != cs.CS_RECOMPUTE]
                ref = orc.forward([N.Entry(e.request_id, e.compute_tokens, e.context_tokens, e.kind, e.online)
                                   for e in (alive[i] for i in keep)])
                got = logits[keep]
                bound = logit_bound(ref)
                worst = max(worst, float(np.max(np.abs(got - ref))) / bound)
                ok, dec = decisive_rows(got, ref, bound)
                agree += ok
                rows += dec
                iters += 1
        if inflight:
            eng.iter_wait()
        eng.audit() if tr.audit == "ok" else None
        return iters, worst, agree / max(rows, 1), drops, eng.stats()
    finally:
        eng.close()


@pytest.mark.parametrize("name", ["config1", "config1_pool48", "config1_pool80", "config1_nolayerwise",
                                  "config1_noincr", "config1_nonpreemptive", "config1_onlineonly", "config1_sarathi",
                                  "config1_host40", "config1_host48"])
def test_reference_run_logits_match_oracle(name):
    iters, worst, agree, drops, st = _replay_with_oracle(name)
    assert iters >= 15
    assert worst <= 1.0, worst             # max-abs / bound, worst iteration
    assert agree >= DECISIVE_AGREE, agree
    if name in ("config1", "config1_pool48", "config1_nolayerwise"):
        assert st.moved_d2h_bytes > 0  # KV went through checkpoint (and restore) on the device
