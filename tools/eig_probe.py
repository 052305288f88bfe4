"""Time the batched eigensolver alone on Tucker-like shapes (C2: 1024 x 32^2 top-12, 128 x 64^2 top-24)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
ctx = gw.Context(0)
ctx.use_torch_stream()
rng = np.random.default_rng(0)
for (b, n, c) in [(1024, 32, 12), (128, 64, 24), (512, 4, 4), (64, 256, 64)]:
    A = rng.standard_normal((b, n, 3 * n)) + 1j * rng.standard_normal((b, n, 3 * n))
    H = torch.from_numpy((A @ np.conj(np.swapaxes(A, 1, 2))).astype(np.complex64)).cuda()
    for _ in range(2):
        ctx.leading_eigenvectors(H, c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.leading_eigenvectors(H, c)
    e1.record(); e1.synchronize()
    print(f"batch {b} n {n} count {c}: {e0.elapsed_time(e1)/5:.3f} ms", flush=True)
