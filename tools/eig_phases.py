import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import _lib
ctx = gw.Context(0)
lib = _lib.load()
rng = np.random.default_rng(0)
for (b, n, c) in [(2048, 32, 12), (256, 64, 24), (64, 128, 40), (16, 256, 64)]:
    A = rng.standard_normal((b, n, 3 * n)) + 1j * rng.standard_normal((b, n, 3 * n))
    H = torch.from_numpy((A @ np.conj(np.swapaxes(A, 1, 2))).astype(np.complex64)).cuda()
    ctx.leading_eigenvectors(H, c)
    out = (C.c_longlong * 4)()
    lib.gwt_debug_eig_phases(out)
    print(n, c, "householder", out[0], "bisection", out[1], "inverse-iter", out[2], "backtransform", out[3], flush=True)
