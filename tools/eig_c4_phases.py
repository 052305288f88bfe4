"""Eigensolver phase cycles on C4 Grams (tx N x N per base in c64, delay P x P per link in c128, as the
Tucker solve runs them) in the phase-timer build:
GWT_LIB_PATH=.../phase/libgwt_b200.so python tools/eig_c4_phases.py [groups]"""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from paper_2401_09792_b200 import _lib
cfg = gw.CONFIGS["C4"]
groups = int(sys.argv[1]) if len(sys.argv) > 1 else 2
X, _ = gw.generate_channels(cfg.topology(), groups, seed=0, dtype=np.complex128, nthreads=16)
g, L, P, N, M = X.shape
J, K = cfg.J, cfg.K
Xl = X.reshape(g, J, J * K, P, N, M)
tx = np.einsum("gklpnm,gklpqm->gknq", Xl, np.conj(Xl)).reshape(-1, N, N)
dl = np.einsum("glpnm,glqnm->glpq", X, np.conj(X)).reshape(-1, P, P)
ctx = gw.Context(0)
lib = _lib.load()
for name, H, c, dt in (("tx", tx, cfg.n, np.complex64), ("delay", dl, cfg.p, np.complex128)):
    Hd = torch.from_numpy(H.astype(dt)).cuda()
    ctx.leading_eigenvectors(Hd, c)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.leading_eigenvectors(Hd, c)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    out = (C.c_longlong * 8)()
    if hasattr(lib, "gwt_debug_eig_phases"): lib.gwt_debug_eig_phases(out)
    print(f"{name}: batch {H.shape[0]} D {H.shape[1]} count {c}: {ms:.2f} ms; householder {out[0]} bisection {out[1]} "
          f"inverse-iter {out[2]} backtransform {out[3]} | hh: col+refl {out[4]} dots {out[5]} matvec {out[6]} tail {out[7]}", flush=True)
