"""Lockstep parity against the UNMODIFIED reference (control plane).

Each golden call log (tests/golden/<scenario>/calls.jsonl.gz, recorded by
oracle/lockstep/recorder.cpp around the reference SimEngine -- script:
oracle/lockstep/make_traces.py) is replayed through the C-ABI
(cs_replay_run, csrc/replay.cpp). Every KvCacheManager result (allocate
ok/shortfall, evict/discard/release stats, checkpoint and prefetch jobs with
their id, bytes and modelled done time, transfer-done frees) must equal the
reference's, and at every scheduler build the logical page table of every
live request (page_table_json + request_gpu_pages + covered_tokens,
kv_cache.cpp:622-634) must hash to the reference's digest. The final audit()
verdict (kv_cache.cpp:566-620) must match too -- including the reference's own
D3 failure on the llama8b run.

CPU tests run the engine bookkeeping-only (CS_FLAG_HOST_ONLY); the GPU tests
replay the tiny scenarios with the real forward, checkpoint gather and restore
kernels on the device.
"""
import os

import pytest

import paper_2410_01228_b200 as cs
from paper_2410_01228_b200 import _ffi as F
from paper_2410_01228_b200 import replay as R

from conftest import ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden")
PRESET = {"config1": "tiny", "llama8b": "llama8b", "llama70b": "llama70b", "qwen14b": "qwen14b", "fuzz": "qwen14b"}
SCENARIOS = sorted(d for d in os.listdir(GOLDEN) if os.path.exists(os.path.join(GOLDEN, d, "calls.jsonl.gz")))


def _preset(name):
    for k, v in PRESET.items():
        if name.startswith(k):
            return v
    raise KeyError(name)


def _load(name):
    g = os.path.join(GOLDEN, name)
    return R.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))


def _replay(name, flags, check_page_tables=True):
    tr = _load(name)
    cfg = R.engine_config_for(tr, _preset(name), flags=flags, max_entries=256)
    eng = cs.Engine(cfg)
    try:
        res = R.run(eng, tr, 0, tr.n_iter, check_page_tables=check_page_tables)
        assert res.iterations == tr.n_iter
        assert res.mismatches == 0, f"first mismatch at op {res.first_mismatch_op}: {tr.ops[res.first_mismatch_op]}"
        verdict = "ok"
        try:
            eng.audit()
        except cs.CsLogicError as ex:
            verdict = str(ex)
        assert verdict == tr.audit
        return tr, res, eng.stats()
    finally:
        eng.close()


def test_scenarios_present():
    assert {"config1", "llama8b", "fuzz2", "config1_sarathi", "config1_noincr"} <= set(SCENARIOS)


@pytest.mark.parametrize("name", SCENARIOS)
def test_lockstep_bookkeeping_bit_exact(name):
    tr, res, st = _replay(name, F.CS_FLAG_HOST_ONLY)
    n_pt = int((tr.ops[:, 0] == R.OPC["pt"]).sum())
    assert n_pt >= tr.n_iter  # one page-table digest per build (+ the final state)
    # the reference's byte totals (metrics.json d2h/h2d) are reproduced
    import json
    m = json.load(open(os.path.join(GOLDEN, name, "metrics.json")))
    assert st.total_d2h_bytes == m["transferred_bytes"]["d2h"]
    assert st.total_h2d_bytes == m["transferred_bytes"]["h2d"]


def test_config1_golden_run_matches_survey():
    """SURVEY.md 8c config-1 golden run: 18 iterations, a drop at layer 1 of
    offline [7, 3, 2, 8], D2H 7,372,800 B and H2D 1,341,440 B."""
    tr, res, st = _replay("config1", F.CS_FLAG_HOST_ONLY)
    assert tr.n_iter == 18
    k = [i for i, l in enumerate(tr.dropped) if l >= 0]
    assert len(k) == 1 and tr.dropped[k[0]] == 1
    dropped = {int(e[0]) for e in tr.plan_of[k[0]] if not e[4]}
    assert dropped == {7, 3, 2, 8}
    assert st.total_d2h_bytes == 7372800 and st.total_h2d_bytes == 1341440


def test_llama8b_self_eviction_reads_are_counted():
    """D3: the reference dispatches entries whose context pages it marks
    HostOnly; the engine counts those block-table reads (and serves them from
    quarantined, intact blocks)."""
    _, _, st = _replay("llama8b", F.CS_FLAG_HOST_ONLY, check_page_tables=False)
    assert st.nonresident_reads > 0


@pytest.mark.gpu
@pytest.mark.parametrize("name", [s for s in SCENARIOS if s.startswith("config1")])
def test_lockstep_on_device(name):
    """The same replay with the real forward, gather and restore kernels."""
    tr, res, st = _replay(name, 0)
    assert (res.gpu_ms > 0).all()
    if st.total_d2h_bytes:
        assert st.moved_d2h_bytes > 0 and st.moved_d2h_ms > 0
