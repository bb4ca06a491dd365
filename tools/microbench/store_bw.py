"""Streaming store / copy bandwidth of one B200 (torch fill_ / zero_ / copy_, CUDA events):
the practical ceiling for the store-bound p = 1 kernels.  python tools/microbench/store_bw.py"""
import torch
x = torch.empty(int(16e9 // 8), dtype=torch.float64, device="cuda")
y = torch.empty(int(8e9 // 8), dtype=torch.float64, device="cuda")
z = torch.empty(int(8e9 // 8), dtype=torch.float64, device="cuda")
for name, fn, by in [("fill 16GB", lambda: x.fill_(1.0), 16e9), ("memset 16GB", lambda: x.zero_(), 16e9),
                     ("copy 8GB", lambda: y.copy_(z), 16e9)]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); 
    for _ in range(5): fn()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(name, f"{by / ms / 1e6:.0f} GB/s")
