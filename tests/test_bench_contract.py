"""bench.py's JSON-line contract, checked on the CPU through the reference arm
(`--impl reference`: the CPU port of the path on one bounded sample of the
headline workload) and its helpers. The GPU arm prints the same keys plus
roofline / clocks / gpu_launches; it runs on the B200 (driver, gpurun)."""
import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_prints_one_contract_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "vs_baseline",
              "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["unit"] == "tok/s" and d["e2e"]["unit"] == "tok/s"
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "workload" in d["config"] and cb["sample"]


def test_reference_arm_never_loads_the_product():
    """The reference arm times the CPU port and the reference's own control
    plane only: the product package (and its .so) must stay unloaded."""
    code = ("import sys, bench, argparse; "
            "bench.run_reference(argparse.Namespace(workload='llama8b', warmup=0, steps=1, gpus=1, replicas=False)); "
            "bad = [m for m in sys.modules if m.startswith('paper_2410_01228_b200')]; "
            "maps = open('/proc/self/maps').read(); "
            "assert not bad and 'libconserve_b200' not in maps, (bad,)")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]


def test_step_slices_cover_the_run():
    sys.path.insert(0, ROOT)
    import bench
    W, sl = bench.slices(1375, 5, 20)
    assert W == 5 and len(sl) == 20 and sl[0][0] == 5 and sl[-1][1] == 1375
    assert all(a < b for a, b in sl) and all(sl[i][1] == sl[i + 1][0] for i in range(19))
    W, sl = bench.slices(10, 3, 50)
    assert W == 3 and len(sl) == 7 and sl[-1][1] == 10


def test_percentile_is_nearest_rank():
    sys.path.insert(0, ROOT)
    import bench
    xs = [5.0, 1.0, 4.0, 2.0, 3.0]
    assert bench.percentile(xs, 0.99) == 5.0
    assert bench.percentile(xs, 0.5) == 3.0
    assert bench.percentile(xs, 0.2) == 1.0
    assert bench.percentile([], 0.99) == 0.0


def test_ckpt_ranks_aggregate_is_bytes_over_slowest_rank():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.ckpt_ranks(None) == {}
    rows = [[4e9, 100.0, 2e9, 50.0, 0], [4e9, 80.0, 2e9, 40.0, 1]]
    d = bench.ckpt_ranks(rows)
    assert [r["rank"] for r in d["per_rank"]] == [0, 1]
    assert abs(d["per_rank"][1]["d2h_gbs"] - 50.0) < 1e-9
    assert abs(d["aggregate_d2h_gbs"] - 80.0) < 1e-9   # 8 GB over the slower rank's 100 ms
    assert abs(d["aggregate_h2d_gbs"] - 80.0) < 1e-9
    assert d["per_rank"][1]["host_numa_node"] == 1
