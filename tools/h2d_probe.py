import torch, time
n = 256 * 1024 * 1024 // 8
h = torch.empty(8 * n, dtype=torch.float64).pin_memory()
d = torch.empty(8 * n, dtype=torch.float64, device="cuda")
for chunk in (n, 8 * n):
    for _ in range(2):
        torch.cuda.synchronize(); t = time.perf_counter()
        for c in range(0, 8 * n, chunk):
            d[c:c + chunk].copy_(h[c:c + chunk], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("chunk MB", chunk * 8 >> 20, "GB/s", 8 * n * 8 / dt / 1e9)
