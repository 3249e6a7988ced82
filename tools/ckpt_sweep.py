"""KV checkpoint / restore sweep (BASELINE.json configs[4]).

N dirty blocks of the Llama-3.1-8B shape (2 MiB per block over 32 layers x
8 KV heads x 16 tokens x d=128, bf16; 1/g of that per GPU at KV-head-group
sharding g), in two shapes:
  * block  -- whole 16-token blocks (a prefill chunk's checkpoint)
  * token  -- 1 new token in each of N blocks (a decode step's checkpoint over
              N sequences): N x L x 2 x H_kv runs of 256 B
D2H is one flush_checkpoints job (K4 gather straight into mapped pinned host
slots); H2D is one start_prefetch job per request (K5 scatter into fresh
blocks). Times are the kernels' CUDA-event durations (cs_kv_stats
moved_*_ms), bytes are the bytes that crossed the host link. Every point is
checked bit-exact (host slot == device block; restored block == original).

  python tools/ckpt_sweep.py [--max-blocks 16384] [--tp 1] [--out gpurun_out/ckpt_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2410_01228_b200 as cs  # noqa: E402
from paper_2410_01228_b200 import _ffi as F  # noqa: E402


def _engine(n_blocks: int, tp: int):
    page = 16 * 131072
    cfg = cs.model_config("llama8b", flags=F.CS_FLAG_NO_MODEL | F.CS_FLAG_NO_FWD_QUARANTINE, gpu_kv_capacity=(n_blocks + 8) * page,
                          host_kv_capacity=(n_blocks + 8) * page, max_entries=64, extra_blocks=64,
                          extra_host_slots=64, tp_size=tp, tp_rank=0)
    return cs.Engine(cfg)


def _check_some(eng, rids, rng, shape, k=4):
    """Bit-exact host copy of k random blocks (written positions)."""
    for rid in rng.choice(rids, size=min(k, len(rids)), replace=False):
        blocks, slots = eng.block_table(int(rid))
        pick = rng.choice(len(blocks), size=min(8, len(blocks)), replace=False)
        for b, s in ((blocks[i], slots[i]) for i in pick):
            dev = eng.read_block(b)
            host = eng.read_host_slot(s)
            c = eng.cfg
            n_tok = 16 if shape == "block" else 1
            dv = dev.reshape(c.num_layers, 2, -1, 16, c.head_dim)[:, :, :, :n_tok]
            hv = host.reshape(c.num_layers, 2, -1, 16, c.head_dim)[:, :, :, :n_tok]
            assert np.array_equal(dv, hv), (rid, b, s)


def point(n: int, shape: str, tp: int, rng) -> dict:
    eng = _engine(n, tp)
    try:
        eng.fill_pool(1234 + n)
        if shape == "block":
            rids = [0]
            eng.register_request(0, False)
            assert eng.allocate(0, 16 * n).ok
            eng.commit_allocations(0)
            eng.note_written(0, 0, 16 * n)
            eng.stage_checkpoint(0, 0, 16 * n)
        else:
            rids = list(range(n))
            for r in rids:
                eng.register_request(r, False)
                assert eng.allocate(r, 1).ok
                eng.commit_allocations(r)
                eng.note_written(r, 0, 1)
                eng.stage_checkpoint(r, 0, 1)
        s0 = eng.stats()
        t0 = time.perf_counter()
        job = eng.flush_checkpoints(0)
        eng.on_transfer_done(job.id, job.done_time)
        wall_d2h = time.perf_counter() - t0
        s1 = eng.stats()
        _check_some(eng, rids, rng, shape)
        d2h_b = s1.moved_d2h_bytes - s0.moved_d2h_bytes
        d2h_ms = s1.moved_d2h_ms - s0.moved_d2h_ms
        # restore: snapshot, pause + evict every request, clobber, prefetch back
        probe = [int(r) for r in rng.choice(rids, size=min(4, len(rids)), replace=False)]
        snap = {r: [eng.read_block(b) for b in eng.block_table(r)[0][:8]] for r in probe}
        for k, r in enumerate(rids):
            eng.on_request_paused(r, k + 1)
            eng.evict_request_gpu(r)
        eng.fill_pool(99)
        s2 = eng.stats()
        t0 = time.perf_counter()
        jobs = [eng.start_prefetch(r, 0) for r in rids]
        for j in jobs:
            eng.on_transfer_done(j.id, j.done_time)
        wall_h2d = time.perf_counter() - t0
        s3 = eng.stats()
        for r, blocks in snap.items():
            nb = eng.block_table(int(r))[0]
            c = eng.cfg
            n_tok = 16 if shape == "block" else 1
            for old, b in zip(blocks, nb):
                got = eng.read_block(b).reshape(c.num_layers, 2, -1, 16, c.head_dim)[:, :, :, :n_tok]
                want = old.reshape(c.num_layers, 2, -1, 16, c.head_dim)[:, :, :, :n_tok]
                assert np.array_equal(got, want), (r, b)
        h2d_b = s3.moved_h2d_bytes - s2.moved_h2d_bytes
        h2d_ms = s3.moved_h2d_ms - s2.moved_h2d_ms
        return {"blocks": n, "shape": shape, "tp": tp,
                "d2h_bytes": d2h_b, "d2h_ms": d2h_ms, "d2h_gbs": d2h_b / d2h_ms / 1e6 if d2h_ms else None,
                "d2h_wall_ms": wall_d2h * 1e3,
                "h2d_bytes": h2d_b, "h2d_ms": h2d_ms, "h2d_gbs": h2d_b / h2d_ms / 1e6 if h2d_ms else None,
                "h2d_jobs": len(jobs), "h2d_wall_ms": wall_h2d * 1e3, "bit_exact": True}
    finally:
        eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-blocks", type=int, default=65536)
    ap.add_argument("--max-host-gib", type=float, default=40.0, help="pinned host pool cap per point")
    ap.add_argument("--tp", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ckpt_sweep.json"))
    args = ap.parse_args()
    rng = np.random.default_rng(1)
    res = []
    block_bytes = 32 * 2 * 8 * 16 * 128 * 2  # Llama-3.1-8B, all layers
    for tp in args.tp:
        sizes = [n for n in (1, 4, 16, 64, 256, 1024, 4096, 16384, 65536)
                 if n <= args.max_blocks and n * block_bytes / tp <= args.max_host_gib * (1 << 30)]
        for shape in ("block", "token"):
            for n in sizes:
                r = point(n, shape, tp, rng)
                print(json.dumps(r), flush=True)
                res.append(r)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
