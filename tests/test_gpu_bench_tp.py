"""The sharded bench path end to end (the driver's `--gpus N` launch:
torchrun, one process per rank, KV-head-group sharding, exchange regions
attached over IPC, max-over-ranks timing, per-rank checkpoint GB/s) on a
ONE-GPU box: CS_BENCH_ONE_DEVICE=1 puts both ranks on GPU 0 (gloo process
group; the two contexts time-slice the device), over the reference's tiny
config-1 co-serving trace. Plumbing, not a measurement."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_two_rank_sharded_bench_runs_and_prints_one_line():
    env = dict(os.environ, CS_BENCH_ONE_DEVICE="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--workload", "config1", "--steps", "2", "--warmup", "1", "--no-probes", "--no-cpu", "--legs", ""]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["parallelism"].startswith("tp2")
    ck = d["kv_ckpt"]
    assert len(ck["per_rank"]) == 2
