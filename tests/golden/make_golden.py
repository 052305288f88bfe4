"""Generate tests/golden/*.npz — independent numpy/LAPACK restatement of the
reference hot path used to PIN the C++ oracle (tests/test_oracle.py).

The reference (gwtucker, Eigen) cannot be built in this container (SURVEY.md
§8(c)); this script re-derives the same quantities through numpy.linalg
(LAPACK zheevd / zgesdd / zpotrf) — a code path that shares nothing with
oracle/gwt_oracle.cpp — following the reference's algorithm:
  groupwise alternating solve   proj/src/decompose.cpp:248-381
  compressed SINR pipeline      proj/src/sinr.cpp:147-254, 296-326
  full SINR pipeline            proj/src/sinr.cpp:67-142, 259-294
Inputs come from the repo's seeded BASELINE generator (C1) and from the oracle's
restatement of the reference generator (desk topology of proj/tests/test_sinr.cpp);
their checksums are stored so the fixture also pins input generation.

Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)


# ---------------------------------------------------------------- numpy restatement
def phase_normalize(u):
    u = u.copy()
    for c in range(u.shape[1]):
        mags = np.abs(u[:, c])
        b = int(np.argmax(mags))  # first maximum on ties
        if mags[b] > 0:
            u[:, c] *= np.conj(u[b, c]) / mags[b]
    return u


def leading(h, count):
    w, v = np.linalg.eigh(h)
    return phase_normalize(v[:, ::-1][:, :count])


def unfold(x, mode):  # x[i1,i2,i3]; columns with the lower remaining mode fastest (tensor.hpp:60-63)
    if mode == 1:
        return x.reshape(x.shape[0], -1, order="F")
    if mode == 2:
        return np.transpose(x, (1, 0, 2)).reshape(x.shape[1], -1, order="F")
    return np.transpose(x, (2, 0, 1)).reshape(x.shape[2], -1, order="F")


def mprod(x, u, mode):
    return np.moveaxis(np.tensordot(u, x, axes=([1], [mode - 1])), 0, mode - 1)


def core_of(x, a, b, c):
    return mprod(mprod(mprod(x, a.conj().T, 1), b.conj().T, 2), c.conj().T, 3)


def recon(g, a, b, c):
    return mprod(mprod(mprod(g, a, 1), b, 2), c, 3)


def groupwise(xs, J, K, m, n, p, sweeps):
    """xs[l] natural [M,N,P] arrays, link l = (k*J+i)*K+j."""
    link = lambda k, i, j: (k * J + i) * K + j
    A = [leading(sum(unfold(xs[link(k, i, j)], 1) @ unfold(xs[link(k, i, j)], 1).conj().T for k in range(J)), m)
         for i in range(J) for j in range(K)]
    B = [leading(sum(unfold(xs[link(k, i, j)], 2) @ unfold(xs[link(k, i, j)], 2).conj().T
                     for i in range(J) for j in range(K)), n) for k in range(J)]
    C = [leading(unfold(x, 3) @ unfold(x, 3).conj().T, p) for x in xs]

    def objective():
        f = 0.0
        for k in range(J):
            for i in range(J):
                for j in range(K):
                    l = link(k, i, j)
                    g = core_of(xs[l], A[i * K + j], B[k], C[l])
                    f += np.sum(np.abs(xs[l] - recon(g, A[i * K + j], B[k], C[l])) ** 2)
        return f

    trace = [objective()]
    for _ in range(sweeps):
        newA = []
        for i in range(J):
            for j in range(K):
                gm = 0
                for k in range(J):
                    w = unfold(mprod(mprod(xs[link(k, i, j)], B[k].conj().T, 2), C[link(k, i, j)].conj().T, 3), 1)
                    gm = gm + w @ w.conj().T
                newA.append(leading(gm, m))
        A = newA
        newB = []
        for k in range(J):
            gm = 0
            for i in range(J):
                for j in range(K):
                    w = unfold(mprod(mprod(xs[link(k, i, j)], A[i * K + j].conj().T, 1), C[link(k, i, j)].conj().T, 3), 2)
                    gm = gm + w @ w.conj().T
            newB.append(leading(gm, n))
        B = newB
        for k in range(J):
            for i in range(J):
                for j in range(K):
                    l = link(k, i, j)
                    w = unfold(mprod(mprod(xs[l], A[i * K + j].conj().T, 1), B[k].conj().T, 2), 3)
                    C[l] = leading(w @ w.conj().T, p)
        trace.append(objective())
    G = [core_of(xs[link(k, i, j)], A[i * K + j], B[k], C[link(k, i, j)])
         for k in range(J) for i in range(J) for j in range(K)]
    return A, B, C, G, np.array(trace)


def scope_pairs(J, K, scope, i, j):
    if scope == "full":
        return [(k, l) for k in range(J) for l in range(K)]
    return [(i, j)] + [(k, 0) for k in range(J) if k != i]


def evaluate(h, J, K, L, sigma, scope):
    """Full-path stages on assembled channels h[l] (sinr.cpp:259-285); returns sinr [users, L]."""
    link = lambda k, i, j: (k * J + i) * K + j
    V = []
    for i in range(J):
        for j in range(K):
            u, s, vh = np.linalg.svd(h[link(i, i, j)], full_matrices=False)
            V.append(vh.conj().T[:, :L])
    out = np.zeros((J * K, L))
    for i in range(J):
        for j in range(K):
            hs = h[link(i, i, j)]
            q = sigma ** 2 * np.eye(hs.shape[0], dtype=complex)
            for k, l in scope_pairs(J, K, scope, i, j):
                t = h[link(k, i, j)] @ V[k * K + l]
                q = q + t @ t.conj().T
            hv = hs @ V[i * K + j]
            w = np.linalg.solve(q, hv)
            for r in range(L):
                amp = np.vdot(w[:, r], hv[:, r])
                s = abs(amp) ** 2
                den = np.real(np.vdot(w[:, r], q @ w[:, r])) - s
                out[i * K + j, r] = s / max(den, np.finfo(float).tiny)
    return out


def compressed_channels(G, C, coeffs):
    return [np.einsum("abq,q->ab", g, np.conj(c.conj().T @ co)) for g, c, co in zip(G, C, coeffs)]


# ---------------------------------------------------------------- fixtures
def main():
    import paper_2401_09792_b200 as gw
    from oracle import oracle as O

    out = {}
    # (1) dense kernels: Hermitian eig / SVD / Cholesky from LAPACK
    rng = np.random.default_rng(2024)
    for n in (3, 8, 24):
        a = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
        h = a @ a.conj().T
        out[f"eig{n}_h"] = h
        out[f"eig{n}_w"] = np.linalg.eigvalsh(h)
        out[f"eig{n}_lead"] = leading(h, max(1, n // 2))
    a = rng.standard_normal((4, 24)) + 1j * rng.standard_normal((4, 24))
    out["svd_a"] = a
    out["svd_s"] = np.linalg.svd(a, compute_uv=False)

    # (2) BASELINE C1, group 0: generator checksum + groupwise solve + compressed SINR
    cfg = gw.CONFIGS["C1"]
    X, tau = gw.generate_channels(cfg.topology(), 1, seed=0, dtype=np.complex128)
    out["c1_x_sum"] = np.array([X.sum(), np.abs(X).sum()])
    out["c1_x_probe"] = X.reshape(-1)[::997][:64]
    out["c1_tau_probe"] = tau.reshape(-1)[::7][:32]
    xs = [np.transpose(X[0, l], (2, 1, 0)) for l in range(cfg.G)]
    A, B, Cf, G, tr = groupwise(xs, cfg.J, cfg.K, cfg.m, cfg.n, cfg.p, 6)
    out["c1_trace6"] = tr
    out["c1_energy"] = np.array(sum(np.sum(np.abs(x) ** 2) for x in xs))
    freqs = cfg.freqs()[:5]
    co = O.coeffs_from_tau(tau, freqs)[0]  # [F, links, P]
    sinr = []
    for f in range(len(freqs)):
        hs = compressed_channels(G, Cf, co[f])
        sinr.append(evaluate(hs, cfg.J, cfg.K, cfg.L, cfg.sigma, "paper_experiment"))
    out["c1_sinr6"] = np.array(sinr)

    # (3) reference desk topology (test_sinr.cpp desk_topology, seed 14, ranks (4,5,3), 6 sweeps)
    Xr, cr = O.generate_reference(2, 2, 6, 8, 5, 14)
    out["desk_x_sum"] = np.array([Xr.sum(), np.abs(Xr).sum()])
    xs = [np.transpose(Xr[l], (2, 1, 0)) for l in range(8)]
    A, B, Cf, G, tr = groupwise(xs, 2, 2, 4, 5, 3, 6)
    out["desk_trace6"] = tr
    hs = compressed_channels(G, Cf, cr)
    for scope in ("paper_experiment", "full"):
        out[f"desk_sinr_{scope}"] = evaluate(hs, 2, 2, 2, 0.1, scope)
    # full pipeline on the raw channels (sinr.cpp:287-294)
    hf = [np.einsum("abq,q->ab", x, np.conj(c)) for x, c in zip(xs, cr)]
    out["desk_full_sinr"] = evaluate(hf, 2, 2, 2, 0.1, "paper_experiment")
    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_v1.npz"), {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
