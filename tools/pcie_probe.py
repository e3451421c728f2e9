import torch, time
n = 24883200  # one 1080p fp32 RGB frame
dev = torch.device("cuda")
src = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(8)]
dst = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(8)]
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for k in range(64):
            s = streams[k % ns]
            with torch.cuda.stream(s):
                dst[k % 8].copy_(src[k % 8], non_blocking=True)
        torch.cuda.synchronize(); el = time.perf_counter() - t0
    print(ns, "streams:", round(64 * n / el / 1e9, 1), "GB/s D2H")
h2d = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
torch.cuda.synchronize(); t0 = time.perf_counter()
for k in range(32):
    src[k % 8].copy_(h2d[k % 2], non_blocking=True)
torch.cuda.synchronize(); print("H2D", round(32 * n / (time.perf_counter() - t0) / 1e9, 1), "GB/s")
