"""Eigensolver phase cycles on Tucker-realistic Grams (C2 init Grams: tx N x N per base, delay P x P per
link) in the phase-timer build: GWT_LIB_PATH=.../phase/libgwt_b200.so python tools/eig_real_phases.py"""
import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import _lib
cfg = gw.CONFIGS["C2"]
X, _ = gw.generate_channels(cfg.topology(), 16, seed=0, dtype=np.complex128, nthreads=16)
g, L, P, N, M = X.shape
J, K = cfg.J, cfg.K
Xl = X.reshape(g, J, J * K, P, N, M)  # [g][k][(i,j)][P][N][M] (link = (k*J+i)*K+j)
tx = np.einsum("gklpnm,gklpqm->gknq", Xl, np.conj(Xl)).reshape(-1, N, N)   # per base k
dl = np.einsum("glpnm,glqnm->glpq", X, np.conj(X)).reshape(-1, P, P)       # per link
ctx = gw.Context(0)
lib = _lib.load()
for name, H, c in (("tx", tx, cfg.n), ("delay", dl, cfg.p)):
    Hd = torch.from_numpy(H.astype(np.complex64)).cuda()
    ctx.leading_eigenvectors(Hd, c)
    out = (C.c_longlong * 4)()
    lib.gwt_debug_eig_phases(out)
    w = np.linalg.eigvalsh(H[0])[::-1]
    rel = w[:c] / w[0]
    clusters = int(np.sum(np.abs(np.diff(w[:c])) <= 1e-3 * w[0]))
    print(f"{name}: batch {H.shape[0]} D {H.shape[1]} count {c}: householder {out[0]} bisection {out[1]} "
          f"inverse-iter {out[2]} backtransform {out[3]}; lambda_c/lambda_1 {rel[-1]:.2e}, close pairs {clusters}", flush=True)
