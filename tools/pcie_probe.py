"""Pinned host<->device copy bandwidth and the SINR e2e call breakdown (C2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
for mb in (1, 4, 13, 64):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e1.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e2.record(); e2.synchronize()
    print(f"{mb} MB: H2D {n*10/e0.elapsed_time(e1)/1e6:.1f} GB/s  D2H {n*10/e1.elapsed_time(e2)/1e6:.1f} GB/s", flush=True)
# concurrent both directions on two streams
n = 64 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"duplex 64 MB each way x10: {2*n*10/(t1-t0)/1e9:.1f} GB/s aggregate", flush=True)
