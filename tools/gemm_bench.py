import torch, time
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
shapes = {"qkv": (6144, 4096), "o": (4096, 4096), "gu": (28672, 4096), "down": (4096, 14336), "lm": (128256, 4096)}
for name, (N, K) in shapes.items():
    W = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for M in (1, 8, 16, 32, 64, 128, 256):
        X = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        for _ in range(3): Y = X @ W.t()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(20): Y = X @ W.t()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"{name:5s} M={M:4d} {ms*1e3:8.1f} us  {N*K*2/ms/1e6:7.0f} GB/s")
