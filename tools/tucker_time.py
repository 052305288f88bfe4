"""Time groupwise_solve (20 fixed sweeps) at a BASELINE shape: tools/tucker_time.py C4 [groups]"""
import os, sys, dataclasses, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
name = sys.argv[1]
cfg = gw.CONFIGS[name]
ng = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.groups
X, _ = gw.generate_channels(cfg.topology(), ng, seed=0, dtype=np.complex64 if cfg.dtype == "c64" else np.complex128, nthreads=16)
Xd = torch.from_numpy(X).cuda()
ctx = gw.Context(0)
ctx.use_torch_stream()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), cfg.sweeps, early_stop=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    nm = res.trace.cpu().numpy()[:, -1] / res.energy.cpu().numpy()
    print(f"{name} groups {ng}: {dt*1e3:.1f} ms  {ng*cfg.G/dt:.1f} channels/s  nmse[0] {nm[0]:.9f}", flush=True)
