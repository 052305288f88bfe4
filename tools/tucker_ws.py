"""groupwise_solve time against the Tucker workspace budget (group chunk size): tools/tucker_ws.py C4 512 16 48 96"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
name, ng = sys.argv[1], int(sys.argv[2])
cfg = gw.CONFIGS[name]
X, _ = gw.generate_channels(cfg.topology(), ng, seed=0, dtype=np.complex64, nthreads=16)
Xd = torch.from_numpy(X).cuda()
del X
for gib in [int(a) for a in sys.argv[3:]]:
    os.environ["GWT_WS_BYTES"] = str(gib << 30)
    ctx = gw.Context(0)
    ctx.use_torch_stream()
    for it in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), cfg.sweeps, early_stop=False)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"{name} groups {ng} ws {gib} GiB: {dt*1e3:.1f} ms  {ng*cfg.G/dt:.1f} channels/s  mem {torch.cuda.mem_get_info()[0]/2**30:.0f} GiB free", flush=True)
    del ctx, res
