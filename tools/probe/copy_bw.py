import torch, time
n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8).pin_memory()
for ns in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        ch = n // ns
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                h[i*ch:(i+1)*ch].copy_(d[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"D2H streams={ns}: {n/dt/1e9:.1f} GB/s")
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"H2D streams={ns}: {n/dt/1e9:.1f} GB/s")
