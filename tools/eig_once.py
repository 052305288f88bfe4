"""One leading_eigenvectors call (for ncu): tools/eig_once.py batch n count [c64|c128]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
b, n, c = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = np.complex128 if len(sys.argv) > 4 and sys.argv[4] == "c128" else np.complex64
ctx = gw.Context(0)
ctx.use_torch_stream()
rng = np.random.default_rng(0)
A = rng.standard_normal((b, n, 3 * n)) + 1j * rng.standard_normal((b, n, 3 * n))
H = torch.from_numpy((A @ np.conj(np.swapaxes(A, 1, 2))).astype(dt)).cuda()
ctx.leading_eigenvectors(H, c)
torch.cuda.synchronize()
print("ok")
