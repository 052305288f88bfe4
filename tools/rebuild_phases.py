import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import _lib
cfg = gw.CONFIGS["C2"]
ctx = gw.Context(0); ctx.use_torch_stream()
X, tau = gw.generate_channels(cfg.topology(), 64, seed=0, dtype=np.complex64)
fac = ctx.groupwise_solve(cfg.topology(), torch.from_numpy(X).cuda(), cfg.ranks(), 2, early_stop=False)
for _ in range(3):
    rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=torch.from_numpy(tau).cuda(), freqs=torch.from_numpy(cfg.freqs()).cuda())
out = (C.c_longlong * 4)(); _lib.load().gwt_debug_rebuild_phases(out)
print("rebuild phases (cycles): phasor", out[0], "E", out[1], "H+store", out[2])
