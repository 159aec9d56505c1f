import torch, time
n = 4 << 30
d = torch.empty(n // 4, dtype=torch.float32, device='cuda')
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = n // 4 // ns
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter()
        for i, st in enumerate(streams):
            with torch.cuda.stream(st):
                h[i*parts:(i+1)*parts].copy_(d[i*parts:(i+1)*parts], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{ns} streams: {n/dt/1e9:.1f} GB/s D2H")
    t0 = time.perf_counter()
    for i, st in enumerate(streams):
        with torch.cuda.stream(st):
            d[i*parts:(i+1)*parts].copy_(h[i*parts:(i+1)*parts], non_blocking=True)
    torch.cuda.synchronize()
    print(f"{ns} streams: {n/(time.perf_counter()-t0)/1e9:.1f} GB/s H2D")
