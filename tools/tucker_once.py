"""One groupwise_solve at a BASELINE shape (for ncu launch lists): tools/tucker_once.py C4 4 1"""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
name, groups, sweeps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = dataclasses.replace(gw.CONFIGS[name], groups=groups, sweeps=sweeps)
ctx = gw.Context(0)
ctx.use_torch_stream()
X, _ = gw.generate_channels(cfg.topology(), groups, seed=0, dtype=np.complex64, nthreads=16)
Xd = torch.from_numpy(X).cuda()
ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), sweeps, early_stop=False)
torch.cuda.synchronize()
print("ok")
