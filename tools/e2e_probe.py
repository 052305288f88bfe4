"""Break down the SINR e2e call (pinned host buffers, C2): wall time of the public API call vs the
C-ABI call alone vs device-resident compute."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import api
cfg = gw.CONFIGS["C2"]
dt = torch.complex64
g = torch.Generator().manual_seed(0)
Ch = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.P, dtype=dt, generator=g).pin_memory()
Gh = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.n, cfg.m, dtype=dt, generator=g).pin_memory()
tauh = (torch.rand(cfg.groups, cfg.G, cfg.P, dtype=torch.float64, generator=g) * 1e-6).pin_memory()
fh = torch.from_numpy(cfg.freqs()).pin_memory()
ctx = gw.Context(0)
topo, ranks = cfg.topology(), cfg.ranks()
fac = gw.GroupwiseFactorSet(None, None, Ch, Gh)
users = topo.num_users
F = fh.shape[0]
so = torch.empty((cfg.groups, F, users, topo.num_streams), dtype=torch.float64).pin_memory()
sg = torch.empty_like(so).pin_memory()
stt = torch.empty((cfg.groups, F, users), dtype=torch.int32).pin_memory()
led = api.L.Ledger() if hasattr(api, "L") else None
for chunks, lanes in (("4", "2"), ("5", "2"), ("6", "2"), ("3", "2"), ("4", "2")):
    os.environ["GWT_SINR_PIPELINE"] = chunks
    os.environ["GWT_SINR_LANES"] = lanes
    for _ in range(3):
        ctx.run_compressed_pipeline(topo, fac, ranks, tau=tauh, freqs=fh)
    t = []
    for _ in range(20):
        t0 = time.perf_counter(); ctx.run_compressed_pipeline(topo, fac, ranks, tau=tauh, freqs=fh); t.append(time.perf_counter() - t0)
    tc = []
    for _ in range(20):
        t0 = time.perf_counter()
        rc = ctx.lib.gwt_sinr_compressed(ctx.h, C.byref(topo.c()), C.byref(ranks.c()), cfg.groups, 0, 0,
                                         C.c_void_p(Ch.data_ptr()), C.c_void_p(Gh.data_ptr()), C.c_void_p(tauh.data_ptr()),
                                         C.c_void_p(fh.data_ptr()), F, 1, C.c_void_p(so.data_ptr()),
                                         C.c_void_p(sg.data_ptr()), C.c_void_p(stt.data_ptr()), None)
        tc.append(time.perf_counter() - t0)
        assert rc == 0, ctx.lib.gwt_last_error(ctx.h)
    print(f"chunks {chunks} lanes {lanes}: API {np.median(t)*1e3:.3f} ms  C-ABI {np.median(tc)*1e3:.3f} ms  stage_ms {ctx.stage_ms()[0]:.3f}", flush=True)
