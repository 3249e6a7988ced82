"""N>1 host logic on CPU (gloo, world_size 2): KV-head-group sharding
 needs no block-table exchange because every rank's allocator
is deterministic and fed the same call sequence. Two ranks replay the same
reference call log with tp_size=2 and must hold identical physical block
tables and host-slot ids for every live request, identical reference byte
accounting, and each move exactly half of the checkpoint bytes (its heads)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, preset, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        import paper_2410_01228_b200 as cs
        from paper_2410_01228_b200 import _ffi as F
        from paper_2410_01228_b200 import replay as R
        g = os.path.join(ROOT, "tests", "golden", name)
        tr = R.load(os.path.join(g, "calls.jsonl.gz"), os.path.join(g, "requests.jsonl.gz"))
        cfg = R.engine_config_for(tr, preset, flags=F.CS_FLAG_HOST_ONLY, max_entries=256, tp_rank=rank,
                                  tp_size=world)
        eng = cs.Engine(cfg)
        digests = []
        # replay iteration by iteration; after each, digest the physical tables
        live = set()
        for k in range(tr.n_iter):
            ops = tr.ops[tr.bounds[k]:tr.bounds[k + 1]]
            live |= {int(o[1]) for o in ops if o[0] == R.OPC["register"]}
            live -= {int(o[1]) for o in ops if o[0] == R.OPC["release"]}
            res = R.run(eng, tr, k, k + 1)
            assert res.mismatches == 0
            h = []
            for rid in sorted(live):
                b, s = eng.block_table(rid)
                h.append((rid, tuple(b), tuple(s)))
            digests.append(hash(tuple(h)))
        st = eng.stats()
        local = torch.tensor([float(x % (1 << 52)) for x in digests] +
                             [float(st.total_d2h_bytes), float(st.moved_d2h_bytes)], dtype=torch.float64)
        gathered = [torch.zeros_like(local) for _ in range(world)]
        dist.all_gather(gathered, local)
        if rank == 0:
            q.put([g.numpy() for g in gathered])
        eng.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,preset", [("config1", "tiny"), ("fuzz4", "qwen14b")])
def test_two_ranks_agree_on_physical_block_tables(name, preset):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, preset, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = out
    assert np.array_equal(a[:-2], b[:-2])          # identical block/slot tables every iteration
    assert a[-2] == b[-2] > 0                       # reference D2H bytes (whole token)
    assert a[-1] == b[-1]
    assert a[-1] <= a[-2] / world                   # each rank moves its heads' share only
