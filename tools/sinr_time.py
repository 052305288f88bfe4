"""Time run_compressed_pipeline on device-resident C2 inputs: per-step events with/without an L2 flush,
plus the ctx stage split (tools/sinr_time.py C2 [steps])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
cfg = gw.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
ctx = gw.Context(0)
ctx.use_torch_stream()
dt = torch.complex64 if cfg.dtype == "c64" else torch.complex128
g = torch.Generator().manual_seed(0)
C = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.P, dtype=dt, generator=g).cuda()
G = torch.randn(cfg.groups, cfg.G, cfg.p, cfg.n, cfg.m, dtype=dt, generator=g).cuda()
tau = (torch.rand(cfg.groups, cfg.G, cfg.P, dtype=torch.float64, generator=g) * 1e-6).cuda()
freqs = torch.from_numpy(cfg.freqs()).cuda()
fac = gw.GroupwiseFactorSet(None, None, C, G)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for flushing in (False, True):
    ts, st = [], []
    for it in range(steps + 3):
        if flushing:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=tau, freqs=freqs)
        e1.record()
        e1.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
            st.append(ctx.stage_ms())
    st = np.mean(np.array(st), 0)
    print(f"flush={flushing}: {np.mean(ts):.4f} ms/step  stages rebuild {st[4]:.4f} pair {st[5]:.4f} small {st[6]:.4f}")
