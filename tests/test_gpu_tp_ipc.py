"""The multi-process form of KV-head-group sharding, on one device: two
processes (one rank engine each, tp_size=2), exchange-region IPC handles
all-gathered over torch.distributed (gloo), peers mapped with
cs_tp_attach_ipc -- exactly what one-process-per-GPU ranks do over NVLink,
here with both processes time-sliced on GPU 0. Both ranks must produce the
same logits, within bf16 tolerance of the fp32 oracle, for prefill and
decode (CUDA-graph) steps."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_dir):
    import ctypes as C

    import numpy as np
    import torch.distributed as dist

    sys.path.insert(0, ROOT)
    import paper_2410_01228_b200 as cs
    from oracle import numeric as N

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = dict(num_layers=3, hidden=256, n_heads=8, n_kv_heads=4, head_dim=64, ffn=512, vocab=512,
                 max_batched_tokens=1024, gpu_kv_capacity=2048 * 16 * 2 * 3 * 64 * 2 * 4, instrumented=0)
    eng = cs.Engine(cs.model_config("tiny", tp_size=world, tp_rank=rank, **shape))
    h = (C.c_uint8 * 64)()
    cs.engine._check(cs.lib().cs_tp_exchange_ipc_handle(eng._h, h))
    handles = [None] * world
    dist.all_gather_object(handles, bytes(h))
    allh = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(handles))
    cs.engine._check(cs.lib().cs_tp_attach_ipc(eng._h, allh, world))
    orc = N.Oracle(N.ModelShape.from_cfg(cs.model_config("tiny", **shape)))
    known = {0: 0, 1: 0}
    prompts = {0: 50, 1: 90}
    for r in prompts:
        eng.register_request(r, r == 0)
    worst = 0.0
    logits_all = []
    for it in range(4):
        plan, allocs = [], []
        for r in prompts:
            c = known[r]
            if c < prompts[r]:
                plan.append(cs.BatchEntry(r, prompts[r] - c, c, cs.CS_PREFILL, r == 0))
                allocs.append(prompts[r] - c + 1)
            else:
                plan.append(cs.BatchEntry(r, 1, c, cs.CS_DECODE, r == 0))
                allocs.append(1)
        for b, n in zip(plan, allocs):
            assert eng.allocate(b.request_id, n).ok
        dist.barrier()
        eng.forward_launch(plan, 50 + it)
        info, lg = eng.iter_wait(want_logits=True)
        ref = orc.forward([N.Entry(b.request_id, b.compute_tokens, b.context_tokens, b.kind, b.online) for b in plan])
        worst = max(worst, float(np.max(np.abs(lg - ref))))
        logits_all.append(lg)
        for b, n in zip(plan, allocs):
            eng.commit_allocations(b.request_id)
            known[b.request_id] += n
    np.save(os.path.join(out_dir, f"logits{rank}.npy"), np.concatenate(logits_all))
    with open(os.path.join(out_dir, f"worst{rank}.txt"), "w") as f:
        f.write(str(worst))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


def test_two_processes_exchange_partials_over_ipc(tmp_path):
    import numpy as np
    port = _free_port()
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import test_gpu_tp_ipc as t; "
            "t._rank_main(int(sys.argv[1]), 2, %d, %r)" % (ROOT, os.path.join(ROOT, "tests"), port, str(tmp_path)))
    env = dict(os.environ, CUDA_MODULE_LOADING="EAGER")
    procs = [subprocess.Popen([sys.executable, "-c", code, str(r)], env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=400)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    l0 = np.load(tmp_path / "logits0.npy")
    l1 = np.load(tmp_path / "logits1.npy")
    assert np.array_equal(l0, l1)
    for r in range(2):
        assert float((tmp_path / f"worst{r}.txt").read_text()) <= 2e-2
