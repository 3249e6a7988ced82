"""Minimal reader of a recorded reference call log (tests/golden/<scenario>/
calls.jsonl.gz, written by oracle/lockstep/recorder.cpp) -- TEST / BENCH
INFRASTRUCTURE ONLY. bench.py's reference arm uses it to pick and account
the iterations it runs on the CPU port without importing the product package
(paper_2410_01228_b200 loads libconserve_b200.so).

Token accounting follows SimEngine::handle_iteration_end
(/root/reference/proj/src/sim_engine.cpp:190-199): per entry of the plan at
iteration end, a prefill chunk adds P tokens (+1 first output token when the
chunk completes the prompt), a decode adds 1, a recompute adds 0; offline
throughput counts offline entries only (proj/src/metrics.cpp:30-39).
"""
from __future__ import annotations

import gzip
import json
from dataclasses import dataclass, field
from typing import Dict, List

import numpy as np


@dataclass
class CallLog:
    config: dict
    plan_of: List[np.ndarray]       # dispatched plan per iteration: [n, 5] (id, P, C, kind, online)
    end_plan_of: List[np.ndarray]   # plan at iteration end (the residual after a drop)
    dropped: List[int]              # reference drop layer per iteration (-1)
    requests: Dict[int, dict] = field(default_factory=dict)

    @property
    def n_iter(self) -> int:
        return len(self.plan_of)

    def offline_tokens(self, k: int) -> int:
        off = 0
        for rid, P, Cc, kind, online in self.end_plan_of[k]:
            if online or kind == 2:
                continue
            off += int(P) if kind == 0 else 1
            rq = self.requests.get(int(rid))
            if kind == 0 and rq is not None and Cc + P >= rq["in"]:
                off += 1
        return off


def load(calls_path: str, requests_path: str) -> CallLog:
    plan_of, end_plan_of, dropped = [], [], []
    config = {}
    with gzip.open(calls_path, "rt") as f:
        for line in f:
            d = json.loads(line)
            if "config" in d:
                config = d["config"]
                continue
            op = d.get("op")
            if op == "dispatch":
                plan_of.append(np.array(d["plan"], dtype=np.int64).reshape(-1, 5))
                end_plan_of.append(np.zeros((0, 5), np.int64))
                dropped.append(-1)
            elif op == "iter_end":
                end_plan_of[-1] = np.array(d["plan"], dtype=np.int64).reshape(-1, 5)
            elif op == "drop":
                dropped[-1] = int(d["layer"])
    log = CallLog(config, plan_of, end_plan_of, dropped)
    with gzip.open(requests_path, "rt") as f:
        for line in f:
            r = json.loads(line)
            log.requests[r["id"]] = r
    return log
