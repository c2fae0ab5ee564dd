import torch, time
n = 1 << 30
h = [torch.empty(n // 4, dtype=torch.uint8).pin_memory() for _ in range(4)]
d = [torch.empty(n // 4, dtype=torch.uint8, device="cuda") for _ in range(4)]
ss = [torch.cuda.Stream() for _ in range(4)]
for ns in (1, 2, 4):
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i in range(4):
            with torch.cuda.stream(ss[i % ns]):
                d[i].copy_(h[i], non_blocking=True)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print(ns, "streams:", round(n / (t1 - t0) / 1e9, 1), "GB/s")
