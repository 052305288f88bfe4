"""Replicate bench.py's e2e loop (pinned inputs, new factor-set per call, optional L2 flush) to
separate the flush/sync effect from the call itself."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
cfg = gw.CONFIGS["C2"]
g = torch.Generator().manual_seed(0)
Ch = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.P, dtype=torch.complex64, generator=g).pin_memory()
Gh = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.n, cfg.m, dtype=torch.complex64, generator=g).pin_memory()
tauh = (torch.rand(cfg.groups, cfg.G, cfg.P, dtype=torch.float64, generator=g) * 1e-6).pin_memory()
fh = torch.from_numpy(cfg.freqs()).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ctx = gw.Context(0)
topo, ranks = cfg.topology(), cfg.ranks()
import itertools
for (ch, ln), mode in itertools.product([("4", "4"), ("5", "5"), ("8", "8"), ("2", "2"), ("1", "1")], ("flush", "flush")):
    os.environ["GWT_SINR_PIPELINE"] = ch
    os.environ["GWT_SINR_LANES"] = ln
    ts = []
    for it in range(25):
        if mode == "flush":
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.run_compressed_pipeline(topo, gw.GroupwiseFactorSet(None, None, Ch, Gh), ranks, tau=tauh, freqs=fh)
        t1 = time.perf_counter()
        if it >= 5:
            ts.append((t1 - t0) * 1e3)
    print(f"chunks {ch} lanes {ln} {mode}: mean {np.mean(ts):.3f} ms  median {np.median(ts):.3f}  min {np.min(ts):.3f} max {np.max(ts):.3f}", flush=True)
