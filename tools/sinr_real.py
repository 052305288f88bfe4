"""SINR step timing on REAL (Tucker-compressed) factors of a BASELINE config subset, single device lane:
tools/sinr_real.py C4 [groups] [sweeps] [steps] -> step ms and the ctx stage split (prep / R+Gram / solve)."""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
name = sys.argv[1]
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 32
sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = gw.CONFIGS[name]
X, tau = gw.generate_channels(cfg.topology(), ng, seed=0, dtype=np.complex64 if cfg.dtype == "c64" else np.complex128, nthreads=16)
ctx = gw.Context(0)
ctx.use_torch_stream()
fac = ctx.groupwise_solve(cfg.topology(), torch.from_numpy(X).cuda(), cfg.ranks(), sweeps, early_stop=False)
taud = torch.from_numpy(tau).cuda()
freqs = torch.from_numpy(cfg.freqs()).cuda()
ts, st = [], []
for it in range(steps + 1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=taud, freqs=freqs)
    e1.record()
    e1.synchronize()
    if it:
        ts.append(e0.elapsed_time(e1))
        st.append(ctx.stage_ms())
st = np.mean(np.array(st), 0)
full = cfg.groups / ng
print(f"{name} {ng} groups: {np.mean(ts):.3f} ms/step (x{full:.0f} = {np.mean(ts)*full:.1f} ms full) "
      f"stages prep {st[4]:.3f} rgram {st[5]:.3f} solve {st[6]:.3f}  status!=0: {int(rep.status.ne(0).sum())}")
