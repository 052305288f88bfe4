"""Time groupwise_solve (fixed sweeps) at BASELINE shapes with a reduced group count; prints ms/solve,
channels/s and algorithmic TFLOP/s (canonical contraction order, bench.tucker_flops)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from bench import tucker_flops
import dataclasses
ctx = gw.Context(0)
ctx.use_torch_stream()
for name, groups, sweeps in [("C2", 64, 20), ("C3", 16, 5), ("C4", 4, 3), ("C5", 32, 5)]:
    cfg = dataclasses.replace(gw.CONFIGS[name], groups=groups, sweeps=sweeps)
    X, _ = gw.generate_channels(cfg.topology(), groups, seed=0, dtype=np.complex64, nthreads=16)
    Xd = torch.from_numpy(X).cuda()
    ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), sweeps, early_stop=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), sweeps, early_stop=False); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    st = ctx.stage_ms()
    fl = tucker_flops(cfg)
    print(f"{name}: groups {groups} sweeps {sweeps}: {ms:.2f} ms, {cfg.links/(ms*1e-3):.0f} ch/s, "
          f"{fl/(ms*1e-3)/1e12:.2f} TFLOP/s, init {st[1]:.2f} ms, sweeps {st[2]:.2f} ms", flush=True)
