"""Shadow-mode fuzz: the reference coserve::KvCacheManager (compiled from
/root/reference by oracle/Makefile -- the checker) and the B200 block pool
(csrc/block_pool.cpp -- the product's allocator) receive the same random call
sequences; return values, exception kinds and messages, byte counters, every
live request's page_table_json (kv_cache.cpp:622-634) and both audits must
agree after every call (tests/cpp/shadow_fuzz.cpp). CPU only."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "shadow_fuzz")


def _build():
    if not os.path.isdir("/root/reference/proj"):
        if not os.path.exists(BIN):
            pytest.skip("reference sources not present on this machine")
        return
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "shadow_fuzz"], check=True,
                   capture_output=True)


@pytest.mark.parametrize("seed", [1, 2])
@pytest.mark.parametrize("incremental,host_pages,gpu_pages", [(1, 256, 64), (0, 64, 48), (1, 32, 40)])
def test_block_pool_shadows_reference(seed, incremental, host_pages, gpu_pages):
    _build()
    r = subprocess.run([BIN, str(seed), "5000", str(incremental), str(host_pages), str(gpu_pages)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    m = re.search(r"failures=(\d+)", r.stdout)
    assert m and int(m.group(1)) == 0, r.stdout + r.stderr[-3000:]
    # the sequence must actually exercise the checkpoint/restore paths
    assert "flush=" in r.stdout and "prefetch=" in r.stdout


def test_directed_advice_sequences():
    """(high) a late partial checkpoint landing on a page that was
    discarded and recomputed while the copy was in flight must leave the
    page's host slot holding [0, host_tokens) -- the pool re-gathers it; and
    (medium) blocks released by one request are reusable while an unrelated
    checkpoint is still copying. Checked through the content model."""
    _build()
    r = subprocess.run([BIN, "0", "1"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr[-3000:]
    assert "failures=0 fixups=1" in r.stdout


@pytest.mark.parametrize("seed", [3, 4])
def test_block_pool_content_long(seed):
    """20k random calls on a small host pool (host LRU + recompute fallback)
    with the physical content model checked after every call."""
    _build()
    r = subprocess.run([BIN, str(seed), "20000", "1", "16", "24"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr[-3000:]
    assert "failures=0" in r.stdout
