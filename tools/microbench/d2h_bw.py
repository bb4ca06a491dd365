"""Pinned D2H / H2D bandwidth on this box: 1 vs 2 vs 4 concurrent streams."""
import time
import torch

n = 4 << 30  # bytes per copy
dev = torch.empty(n // 8, dtype=torch.float64, device="cuda")
host = [torch.empty(n // 8 // 4, dtype=torch.float64).pin_memory() for _ in range(4)]
for nstream in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstream)]
    part = n // 8 // 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rep in range(3):
        for i in range(4):
            s = streams[i % nstream]
            with torch.cuda.stream(s):
                host[i].copy_(dev[i * part:(i + 1) * part], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"D2H {nstream} stream(s): {3 * n / dt / 1e9:.1f} GB/s", flush=True)
