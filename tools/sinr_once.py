"""One compressed-SINR pipeline call at a BASELINE shape on device-resident inputs (for ncu):
tools/sinr_once.py C2 [groups]"""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
name = sys.argv[1]
cfg = gw.CONFIGS[name]
if len(sys.argv) > 2:
    cfg = dataclasses.replace(cfg, groups=int(sys.argv[2]))
ctx = gw.Context(0)
ctx.use_torch_stream()
dt = torch.complex64 if cfg.dtype == "c64" else torch.complex128
g = torch.Generator().manual_seed(0)
L = cfg.links
C = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.P, dtype=dt, generator=g).cuda()
G = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.n, cfg.m, dtype=dt, generator=g).cuda()
tau = (torch.rand(cfg.groups, cfg.G, cfg.P, dtype=torch.float64, generator=g) * 1e-6).cuda()
freqs = torch.from_numpy(cfg.freqs()).cuda()
rep = ctx.run_compressed_pipeline(cfg.topology(), gw.GroupwiseFactorSet(None, None, C, G), cfg.ranks(), tau=tau, freqs=freqs)
torch.cuda.synchronize()
print("ok", ctx.stage_ms())
