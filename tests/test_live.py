"""Live mode (oracle/lockstep/live.cpp): the UNMODIFIED reference SimEngine
driving the engine through the drop-in KvCacheManager, with the forward seam
(oracle_latency, sim_engine.cpp:256), the drop seam (apply_drop) and the
iteration-end seam wrapped onto the C-ABI.

CPU (here): with --dry the engine is bookkeeping-only and the wrapped forward
returns the reference's own latency, so the tool must reproduce the
reference's run byte for byte -- metrics.json (MetricsReport::to_json_text,
metrics.cpp:114-191) and events.jsonl (SimEngine::log_event,
sim_engine.cpp:44-48) -- and write the reference's timeseries.csv. That pins
the wiring (forward launch per dispatch, retro drop at the reference's layer,
cs_iter_wait at iteration end) on every golden scenario, drops included.
GPU: the same tool on the B200 (measured latency), in test_gpu_live.py."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "oracle", "_ref")
GOLDEN = os.path.join(ROOT, "tests", "golden")
PRESET = {"config1": "tiny", "llama8b": "llama8b", "qwen14b": "qwen14b", "llama70b": "llama70b"}

pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference sources not present on this machine")


@pytest.fixture(scope="module")
def built():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-j8", "all", "run-engines", "live"],
                   check=True, capture_output=True)
    return True


def _preset(name):
    for k, v in PRESET.items():
        if name.startswith(k):
            return v
    return None


@pytest.mark.parametrize("name", ["config1", "config1_pool48", "config1_sarathi", "config1_noincr",
                                  "llama8b_b200_spike", "llama70b_b200"])
def test_live_dry_reproduces_the_reference_run(built, name, tmp_path):
    g = os.path.join(GOLDEN, name)
    ref = subprocess.run([os.path.join(OUT, "run_engine_ref"), "run_config.json"], cwd=g, capture_output=True,
                         text=True, timeout=600)
    assert ref.returncode == 0, ref.stdout[-500:]
    r = subprocess.run([os.path.join(OUT, "adapter", "live"), "run_config.json", str(tmp_path), _preset(name), "--dry"],
                       cwd=g, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    summary = json.loads(r.stdout.strip().splitlines()[-1])
    metrics = (tmp_path / "metrics.json").read_text()
    events = (tmp_path / "events.jsonl").read_text()
    assert ref.stdout == metrics + "\n" + events
    m = json.loads(metrics)
    assert summary["drops"] == m["preemptions"] and summary["iterations"] > 0
    ts = (tmp_path / "timeseries.csv").read_text().splitlines()
    assert ts[0] == "t,p99_ttft_5s,p99_tbt_5s,offline_tput_5s" and len(ts) >= 2
