"""Pin the oracle restatement to the REFERENCE ITSELF (oracle/_ref: the reference's own
proj/src/{tensor,linalg,channel,decompose,sinr,archive,metrics}.cpp compiled unchanged
against the in-repo Eigen-subset shim, oracle/Makefile `ref`).

Parity of the oracle against the reference: solver traces (relative to the channel
energy) within 1e-12 with equal iteration counts (the reference's own stop rule,
decompose.cpp:363-368), factor subspaces within 1e-8, per-stream SINR of the
compressed and full pipelines within 1e-12, ledgers equal, reference generator
identical, archive bytes identical. The eigen/SVD/Cholesky arithmetic differs by
construction (the shim is an independent Jacobi/Cholesky implementation of Eigen's
documented contract), so agreement is to rounding, not bitwise.
"""
import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built and /root/reference absent")

DESK = [  # (J, K, M, N, P, m, n, p, seed, L)
    (2, 2, 6, 8, 5, 3, 4, 3, 12, 2),
    (2, 2, 6, 8, 5, 6, 8, 5, 3, 2),   # lossless ranks
    (3, 2, 4, 6, 4, 2, 3, 2, 7, 1),
    (1, 1, 4, 6, 5, 2, 3, 2, 1, 2),   # J = K = 1 (single link)
]


def _angle(U1, U2):
    Q1, _ = np.linalg.qr(U1)
    Q2, _ = np.linalg.qr(U2)
    R = Q2 - Q1 @ (Q1.conj().T @ Q2)
    return np.linalg.svd(R, compute_uv=False)[0] if R.size else 0.0


def _compare_solve(dims, X, sweeps):
    r = O.ref_groupwise_solve(dims, X, sweeps)
    o = O.alternating_solve(dims, X, sweeps, early_stop=True)
    np.testing.assert_array_equal(r["iters"], o["iters"])
    for g in range(X.shape[0]):
        it = int(r["iters"][g])
        e = o["energy"][g]
        assert np.max(np.abs(r["trace"][g, :it + 1] - o["trace"][g, :it + 1])) <= 1e-12 * e
        for key in ("A", "B", "C"):
            for a, b in zip(r[key][g], o[key][g]):
                assert _angle(a.T, b.T) <= 1e-8
    return r, o


@pytest.mark.parametrize("case", DESK)
def test_groupwise_solve_matches_reference(case):
    J, K, M, N, P, m, n, p, seed, L = case
    X, c = O.ref_generate_channel_set(J, K, M, N, P, seed)
    X2, c2 = O.generate_reference(J, K, M, N, P, seed)
    assert np.abs(X - X2).max() <= 1e-14 * np.abs(X).max() and np.abs(c - c2).max() <= 1e-14 * np.abs(c).max()
    dims = dict(J=J, K=K, M=M, N=N, P=P, m=m, n=n, p=p)
    r, o = _compare_solve(dims, X[None], 12)
    for scope in (O.SCOPE_PAPER, O.SCOPE_FULL):
        want, wsig, wled = O.ref_sinr_compressed(dims, r["C"], r["G"], c[None, None], 0.1, L, scope)
        got, gsig, gled = O.sinr_compressed(dims, r["C"], r["G"], c[None, None], 0.1, L, scope, with_ledger=True)
        assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-12
        assert np.max(np.abs(gsig - wsig) / np.abs(wsig)) <= 1e-10  # |w^H H v|^2 carries the factorisations' rounding
        np.testing.assert_array_equal(gled, wled)
        fw, _ = O.ref_sinr_full(dims, X[None], c[None, None], 0.1, L, scope)
        fg, _ = O.sinr_full(dims, X[None], c[None, None], 0.1, L, scope)
        assert np.max(np.abs(fg - fw) / np.abs(fw)) <= 1e-10  # s / (w^H Q w - s) cancels at high SINR


def test_c1_baseline_solve_and_sinr_match_reference():
    """BASELINE C1 (4 groups, complex128): the reference's groupwise_solve and compressed pipeline."""
    cfg = gw.CONFIGS["C1"]
    X, tau = O.generate_baseline(cfg.J, cfg.K, cfg.M, cfg.N, cfg.P, cfg.groups)
    dims = dict(J=cfg.J, K=cfg.K, M=cfg.M, N=cfg.N, P=cfg.P, m=cfg.m, n=cfg.n, p=cfg.p)
    r, _ = _compare_solve(dims, X, cfg.sweeps)
    co = O.coeffs_from_tau(tau, cfg.freqs()[::8])
    want, _, _ = O.ref_sinr_compressed(dims, r["C"], r["G"], co, cfg.sigma, cfg.L)
    got, _ = O.sinr_compressed(dims, r["C"], r["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=4)
    assert np.max(np.abs(got - want) / np.abs(want)) <= 1e-12


def test_shared_solve_matches_reference():
    X, _ = O.ref_generate_channel_set(2, 2, 6, 8, 5, 21)
    dims = dict(J=2, K=2, M=6, N=8, P=5, m=3, n=4, p=3)
    r = O.ref_groupwise_solve(dims, X[None], 8, pooled=True)
    o = O.alternating_solve(dims, X[None], 8, early_stop=True, pooled=True)
    it = int(r["iters"][0])
    assert it == int(o["iters"][0])
    assert np.max(np.abs(r["trace"][0, :it + 1] - o["trace"][0, :it + 1])) <= 1e-12 * o["energy"][0]


def test_archive_bytes_match_reference(tmp_path):
    """archive.py writes the same bytes as the reference's gwt::save_archive (archive.cpp:178-229)."""
    from paper_2401_09792_b200 import archive as ar
    J, K, M, N, P, m, n, p = 2, 2, 6, 8, 5, 3, 4, 3
    X, c = O.ref_generate_channel_set(J, K, M, N, P, 12)
    dims = dict(J=J, K=K, M=M, N=N, P=P, m=m, n=n, p=p)
    r = O.ref_groupwise_solve(dims, X[None], 4)
    O.ref_save_archive(tmp_path / "ref.gwtk", 2, dims, r["A"][0], r["B"][0], r["C"][0], r["G"][0], c)
    fac = gw.GroupwiseFactorSet(r["A"], r["B"], r["C"], r["G"])
    ar.save_archive(tmp_path / "ours.gwtk", "groupwise", fac, c, J, K)
    assert (tmp_path / "ours.gwtk").read_bytes() == (tmp_path / "ref.gwtk").read_bytes()


def test_model_names_match_reference():
    from paper_2401_09792_b200 import api
    for k, name in ((0, "individual"), (1, "shared"), (2, "groupwise")):
        assert O.ref_model_name(k) == name == api.model_name(api.ModelKind(k))
        assert O.ref_model_from_name(name) == k == int(api.model_from_name(name))
    with pytest.raises(O.OracleError) as e:
        O.ref_model_from_name("tucker")
    with pytest.raises(gw.InvalidArgument) as e2:
        api.model_from_name("tucker")
    assert str(e.value) == str(e2.value)
