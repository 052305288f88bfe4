"""Accuracy diagnostic at C4 (8 groups, 1-sweep GPU factors): rebuild error of H~ on the device vs a
binary64 rebuild of the same factors, and the SINR error it causes (oracle on each H~) vs the error of
the device solve on its own H~ (tools/diag_c4.py [name] [groups])."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09792_b200 as gw
from oracle import oracle as O
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
ng = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = gw.CONFIGS[name]
X, tau = gw.generate_channels(cfg.topology(), ng, seed=0, dtype=np.complex64)
ctx = gw.Context(0)
fac = ctx.groupwise_solve(cfg.topology(), torch.from_numpy(X).cuda(), cfg.ranks(), 1, early_stop=False)
fidx = np.unique(np.r_[np.linspace(0, cfg.F - 1, 48).astype(np.int64), cfg.F - 1])
freqs = cfg.freqs()[fidx]
Cd = fac.delay.cpu().numpy(); G = fac.cores.cpu().numpy()
Hg = ctx.assemble_compressed(cfg.topology(), cfg.ranks(), Cd, G, tau=tau, freqs=freqs)  # [g,F,links,n,m]
co = O.coeffs_from_tau(tau, freqs)  # [g,F,links,P]
J, K, m, n, p, P, L = cfg.J, cfg.K, cfg.m, cfg.n, cfg.p, cfg.P, cfg.L
links = J * J * K
C128 = Cd.astype(np.complex128).reshape(ng, links, p, P)
G128 = G.astype(np.complex128).reshape(ng, links, p, n, m)
d = np.einsum("glqP,gflP->gflq", C128, np.conj(co))
Hr = np.einsum("glqnm,gflq->gflnm", G128, d)
err = np.linalg.norm((Hg - Hr).reshape(ng, len(fidx), links, -1), axis=-1) / np.linalg.norm(Hr.reshape(ng, len(fidx), links, -1), axis=-1)
print("H~ rel Frobenius error: max", err.max(), "median", np.median(err))
E32 = np.einsum("glqP,gflP->gflq", C128, np.conj(co.astype(np.complex64)).astype(np.complex128))
print("E phasor-rounding check (c in c64):", np.abs(E32 - d).max() / np.abs(d).max())
dims = dict(J=J, K=K, M=cfg.M, N=cfg.N, P=P, m=m, n=n, p=p)
want, _ = O.sinr_compressed(dims, C128, G128, co, cfg.sigma, L, O.SCOPE_PAPER, nthreads=16)
rep = ctx.run_compressed_pipeline(cfg.topology(), gw.GroupwiseFactorSet(None, None, Cd, G), cfg.ranks(), tau=tau, freqs=freqs)
got = np.asarray(rep.sinr)
print("device pipeline vs oracle: max rel", (np.abs(got - want) / np.abs(want)).max())
worst = np.unravel_index(np.argmax(np.abs(got - want) / np.abs(want)), got.shape)
print("worst item", worst, got[worst], want[worst])
g0, f0 = worst[0], worst[1]
# oracle on the device's H~ and on the binary64 H~ at the worst slice
for tag, HH in (("device H~", Hg[g0, f0].astype(np.complex128)), ("fp64 H~", Hr[g0, f0])):
    s, _ = O.evaluate_assembled(J, K, L, cfg.sigma, HH)
    print(tag, "-> oracle SINR at worst user:", s[worst[2]], "rel vs want", np.abs(s[worst[2]] - want[worst][..., None] if False else s[worst[2]] - want[g0, f0, worst[2]]) / np.abs(want[g0, f0, worst[2]]))
sv = np.linalg.svd(Hr[g0, f0, (worst[2] // K * J + worst[2] // K) * K + worst[2] % K], compute_uv=False)
print("serving singular values at worst", sv)
