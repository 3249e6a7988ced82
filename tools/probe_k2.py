"""Debug probe: repeated single-entry prefill forwards over a cached context."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_2410_01228_b200 as cs

C = int(sys.argv[1])
Ps = [int(x) for x in sys.argv[2:]]
cfg = cs.model_config("llama8b", gpu_kv_capacity=12 << 30, host_kv_capacity=1 << 30, max_batched_tokens=8192,
                      instrumented=0, max_entries=64)
eng = cs.Engine(cfg)
eng.register_request(0, False)
assert eng.allocate(0, C).ok
eng.commit_allocations(0)
for P in Ps:
    for rep in range(3):
        assert eng.allocate(0, P).ok
        print("launch", P, C, rep, flush=True)
        t = time.time()
        info = eng.forward([cs.BatchEntry(0, P, C, cs.CS_PREFILL, False)], epoch=1)
        print(P, C, rep, round(info.gpu_ms, 3), round(time.time() - t, 3), flush=True)
        eng.rollback_allocations(0)
