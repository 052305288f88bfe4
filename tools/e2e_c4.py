"""Host-buffer (e2e) vs device-resident SINR timing at a BASELINE shape on random factors:
tools/e2e_c4.py C4 [groups]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
cfg = gw.CONFIGS[sys.argv[1]]
ng = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.groups
g = torch.Generator().manual_seed(0)
C = torch.randn(ng, cfg.G, cfg.p, cfg.P, dtype=torch.complex64, generator=g)
G = torch.randn(ng, cfg.G, cfg.p, cfg.n, cfg.m, dtype=torch.complex64, generator=g)
tau = torch.rand(ng, cfg.G, cfg.P, dtype=torch.float64, generator=g) * 1e-6
freqs = torch.from_numpy(cfg.freqs())
ctx = gw.Context(0)
for name, fac, ta, fr in (("device", gw.GroupwiseFactorSet(None, None, C.cuda(), G.cuda()), tau.cuda(), freqs.cuda()),
                          ("host", gw.GroupwiseFactorSet(None, None, C.pin_memory(), G.pin_memory()), tau.pin_memory(), freqs.pin_memory())):
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=ta, freqs=fr)
        torch.cuda.synchronize(); t1 = time.perf_counter()
        print(f"{name}: {(t1-t0)*1e3:.1f} ms  stages {[round(x,2) for x in ctx.stage_ms()]}", flush=True)
