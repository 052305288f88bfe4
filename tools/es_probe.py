"""Time groupwise_solve in fixed-sweep and reference-stop-rule modes (C2, device-resident)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
cfg = gw.CONFIGS["C2"]
ctx = gw.Context(0)
ctx.use_torch_stream()
X, _ = gw.generate_channels(cfg.topology(), cfg.groups, seed=0, dtype=np.complex64, nthreads=16)
Xd = torch.from_numpy(X).cuda()
for es in (False, True, False, True):
    ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), 20, early_stop=es)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); f = ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), 20, early_stop=es); e1.record(); e1.synchronize()
    it = f.iterations_run
    it = np.asarray(it.cpu() if hasattr(it, "cpu") else it)
    print(f"early_stop={es}: {e0.elapsed_time(e1):.2f} ms (wall {1e3*(time.perf_counter()-t0):.2f}) iters mean {it.mean():.2f} max {it.max()} stages {ctx.stage_ms()[:3]}", flush=True)
