"""Probe a GPU box: host cores, GPU info, pinned host-link bandwidth (D2H/H2D)."""
import json, os, subprocess, time
import torch

out = {"nproc": os.cpu_count()}
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:2000]
except Exception as e:
    out["lscpu"] = str(e)
out["smi"] = subprocess.run(["nvidia-smi", "-q", "-d", "CLOCK,MEMORY"], capture_output=True, text=True).stdout[:3000]
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:3000]
dev = torch.device("cuda:0")
res = {}
for mib in [1, 16, 256, 1024]:
    n = mib << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for direction in ["d2h", "h2d"]:
        best = 1e9
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                if direction == "d2h":
                    h.copy_(d, non_blocking=True)
                else:
                    d.copy_(h, non_blocking=True)
                e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[f"{direction}_{mib}MiB_GBps"] = n / (best * 1e-3) / 1e9
# bidirectional
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device=dev); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
with torch.cuda.stream(s1):
    h1.copy_(d1, non_blocking=True)
with torch.cuda.stream(s2):
    d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize()
res["bidir_1GiB_each_GBps_total"] = 2 * n / (time.perf_counter() - t0) / 1e9
out["link"] = res
print(json.dumps(res, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
