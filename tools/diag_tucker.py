"""Tucker accuracy diagnostic (tools/diag_tucker.py C4 4 5): GPU vs oracle NMSE trace, the oracle
objective (explicit reconstruction) on the GPU factors, and the factors' orthonormality in binary64."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_09792_b200 as gw
from oracle import oracle as O
from tests.helpers import baseline_inputs, dims_of
name, ng, sw = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = gw.CONFIGS[name]
X, X128, _ = baseline_inputs(cfg, ng)
ctx = gw.Context(0)
res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), sw, early_stop=False)
nm_g = np.asarray(res.trace) / np.asarray(res.energy)[:, None]
fo = O.alternating_solve(dims_of(cfg), X128, sw, early_stop=False, nthreads=16)
nm_o = fo["trace"] / fo["energy"][:, None]
np.set_printoptions(precision=9, linewidth=200)
print("gpu  ", nm_g[0]); print("oracle", nm_o[0]); print("diff max", np.abs(nm_g - nm_o).max(axis=0))
def orth(F):  # F [..., cols, rows] column-major per item
    F = np.asarray(F).astype(np.complex128)
    Fm = np.swapaxes(F, -1, -2)  # rows x cols
    I = np.eye(Fm.shape[-1])
    return np.abs(np.conj(np.swapaxes(Fm, -1, -2)) @ Fm - I).max()
print("orth rx", orth(res.rx), "tx", orth(res.tx), "delay", orth(res.delay))
for g in range(ng):
    f_o, _ = O.objective(dims_of(cfg), X128[g], res.rx[g].astype(np.complex128), res.tx[g].astype(np.complex128),
                         res.delay[g].astype(np.complex128))
    print("group", g, "oracle objective on gpu factors", f_o / fo["energy"][g], "gpu reported", nm_g[g, -1],
          "oracle own", nm_o[g, -1])
