"""Shared test drivers: run the same plans through the engine (C-ABI) and the
CPU oracle, allocating KV the way the reference scheduler does
(scheduler.cpp:138-158, 183-195: the final prefill chunk also claims the first
generated token's slot; a decode entry claims one more slot)."""
from __future__ import annotations

from typing import Dict, List, Sequence

import numpy as np

import paper_2410_01228_b200 as cs
from oracle import numeric as N


class Driver:
    def __init__(self, cfg, oracle: bool = True):
        self.cfg = cfg
        self.eng = cs.Engine(cfg)
        self.orc = N.Oracle(N.ModelShape.from_cfg(cfg)) if oracle else None
        self.known: Dict[int, int] = {}     # context_len (prefill_done + decode_done)
        self.prompt: Dict[int, int] = {}
        self.online: Dict[int, bool] = {}
        self.epoch = 0

    def add(self, rid: int, prompt: int, online: bool = False):
        self.eng.register_request(rid, online)
        self.known[rid] = 0
        self.prompt[rid] = prompt
        self.online[rid] = online

    def entry_for(self, rid: int, P: int = None):
        """(BatchEntry, tokens to allocate) as build_conserve would make it."""
        C = self.known[rid]
        if C < self.prompt[rid]:
            P = min(P or self.prompt[rid] - C, self.prompt[rid] - C)
            final = C + P == self.prompt[rid]
            return cs.BatchEntry(rid, P, C, cs.CS_PREFILL, self.online[rid]), P + (1 if final else 0)
        return cs.BatchEntry(rid, 1, C, cs.CS_DECODE, self.online[rid]), 1

    def step(self, plan: Sequence[tuple], want_logits=True, preempt_after_launch=False):
        """plan: [(rid, P or None)], online first. Returns (info, logits, oracle logits)."""
        entries, allocs = [], []
        for rid, P in plan:
            e, n = self.entry_for(rid, P)
            r = self.eng.allocate(rid, n)
            assert r.ok, (rid, n, r)
            entries.append(e)
            allocs.append(n)
        self.epoch += 1
        self.eng.forward_launch(entries, self.epoch)
        if preempt_after_launch:
            self.eng.preempt_signal(self.epoch)
        out = self.eng.iter_wait(want_logits=want_logits)
        info, logits = out if want_logits else (out, None)
        dropped = info.preempted_at_layer is not None
        ref = None
        survivors = [e for e in entries if (e.online or not dropped)]
        if self.orc is not None and survivors:
            ref = self.orc.forward([N.Entry(e.request_id, e.compute_tokens, e.context_tokens, e.kind, e.online)
                                    for e in survivors])
        for e, n in zip(entries, allocs):
            if e.online or not dropped:
                self.eng.commit_allocations(e.request_id)
                self.known[e.request_id] += n
            else:
                self.eng.rollback_allocations(e.request_id)
        return info, logits, ref

    def close(self):
        self.eng.close()


def rel_l2(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


# Logit parity bounds shared by the GPU numeric tests (bf16 engine vs the fp32
# oracle with bf16 storage points): max-abs within LOGIT_ABS and within
# LOGIT_REL x std(oracle logits), and argmax agreement >= DECISIVE_AGREE on
# the rows whose oracle top-2 gap exceeds twice that bound (near-ties may
# legitimately flip; decisive rows may not).
LOGIT_ABS = 2e-2
LOGIT_REL = 0.06
DECISIVE_AGREE = 0.99


def logit_bound(ref: np.ndarray) -> float:
    return min(LOGIT_ABS, LOGIT_REL * float(np.std(ref)))


def decisive_rows(got: np.ndarray, ref: np.ndarray, bound: float):
    """(agreeing, decisive) row counts: rows whose oracle top-2 gap > 2*bound."""
    top2 = np.sort(ref, axis=-1)[..., -2:]
    dec = (top2[..., 1] - top2[..., 0]) > 2 * bound
    same = np.argmax(got, -1) == np.argmax(ref, -1)
    return int(np.sum(same & dec)), int(np.sum(dec))
