"""Live mode on the B200 (oracle/lockstep/live.cpp): the reference SimEngine's
clock advances by the MEASURED device time of each real forward; its KV calls
run on the HBM block pool. The run must complete with the reference's
invariants intact and write the reference's wire formats (metrics.json,
events.jsonl with measured latency_ms per dispatch, timeseries.csv)."""
import json
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
LIVE = os.path.join(ROOT, "oracle", "_ref", "adapter", "live")
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name", ["config1", "config1_pool48"])
def test_live_tiny_on_device(name, tmp_path):
    if not os.path.exists(LIVE):
        pytest.fail("oracle/_ref/adapter/live not built (make -C oracle live)")
    g = os.path.join(GOLDEN, name)
    r = subprocess.run([LIVE, "run_config.json", str(tmp_path), "tiny"], cwd=g, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    s = json.loads(r.stdout.strip().splitlines()[-1])
    assert not s["dry"] and s["iterations"] > 0 and s["measured_ms"] > 0
    m = json.loads((tmp_path / "metrics.json").read_text())
    assert m["online_finished"] == 4
    disp = [json.loads(ln) for ln in (tmp_path / "events.jsonl").read_text().splitlines() if '"dispatch"' in ln]
    assert len(disp) == s["iterations"]
    # the clock is the device's: every dispatch carries its measured time
    assert abs(sum(d["latency_ms"] for d in disp) - s["measured_ms"]) < 1e-3 * s["measured_ms"] + 1e-3
    assert (tmp_path / "timeseries.csv").read_text().startswith("t,p99_ttft_5s")
