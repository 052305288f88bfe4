"""CPU tests pinning the oracle (oracle/gwt_oracle.cpp).

(1) against golden fixtures from the independent numpy/LAPACK restatement
    (tests/golden/make_golden.py), and
(2) against the reference's own known-answer tests and identities, restated
    (proj/tests/test_{tensor,decompose,sinr,channel,acceptance}.cpp).
"""
import os

import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from oracle import oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.npz"))
DESK = dict(J=2, K=2, M=6, N=8, P=5)


def nat(X):
    """[links,P,N,M] product layout -> list of natural [M,N,P] tensors."""
    return [np.transpose(x, (2, 1, 0)) for x in X]


# ------------------------------------------------------------------ golden pins
@pytest.mark.parametrize("n", [3, 8, 24])
def test_eig_matches_lapack_golden(n):
    h = GOLD[f"eig{n}_h"]
    w, v = O.heev(h)
    assert np.max(np.abs(w - GOLD[f"eig{n}_w"])) <= 1e-12 * np.abs(GOLD[f"eig{n}_w"]).max()
    lead = O.leading_eigenvectors(h, max(1, n // 2))
    assert np.max(np.abs(lead - GOLD[f"eig{n}_lead"])) <= 1e-10


def test_svd_matches_lapack_golden():
    a = GOLD["svd_a"]
    u, s, v = O.truncated_svd(a, 4)
    assert np.max(np.abs(s - GOLD["svd_s"])) <= 1e-12 * s[0]
    assert np.linalg.norm(u * s @ v.conj().T - a) <= 1e-12 * np.linalg.norm(a)


def test_generator_pinned():
    cfg = gw.CONFIGS["C1"]
    X, tau = gw.generate_channels(cfg.topology(), 1, seed=0, dtype=np.complex128)
    np.testing.assert_allclose([X.sum(), np.abs(X).sum()], GOLD["c1_x_sum"], rtol=1e-13)
    np.testing.assert_array_equal(X.reshape(-1)[::997][:64], GOLD["c1_x_probe"])
    np.testing.assert_array_equal(tau.reshape(-1)[::7][:32], GOLD["c1_tau_probe"])
    Xr, _ = O.generate_reference(2, 2, 6, 8, 5, 14)
    np.testing.assert_allclose([Xr.sum(), np.abs(Xr).sum()], GOLD["desk_x_sum"], rtol=1e-13)


def test_groupwise_and_sinr_match_golden_c1():
    cfg = gw.CONFIGS["C1"]
    X, tau = gw.generate_channels(cfg.topology(), 1, seed=0, dtype=np.complex128)
    d = dict(J=cfg.J, K=cfg.K, M=cfg.M, N=cfg.N, P=cfg.P, m=cfg.m, n=cfg.n, p=cfg.p)
    fo = O.alternating_solve(d, X, 6, early_stop=False)
    np.testing.assert_allclose(fo["trace"][0], GOLD["c1_trace6"], rtol=1e-9)
    np.testing.assert_allclose(fo["energy"][0], GOLD["c1_energy"], rtol=1e-13)
    co = O.coeffs_from_tau(tau, cfg.freqs()[:5])
    sinr, _ = O.sinr_compressed(d, fo["C"], fo["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER)
    np.testing.assert_allclose(sinr[0], GOLD["c1_sinr6"], rtol=1e-9)


def test_desk_system_matches_golden():
    Xr, cr = O.generate_reference(2, 2, 6, 8, 5, 14)
    d = dict(DESK, m=4, n=5, p=3)
    fo = O.alternating_solve(d, Xr[None], 6, early_stop=False)
    np.testing.assert_allclose(fo["trace"][0], GOLD["desk_trace6"], rtol=1e-9)
    for scope, code in (("paper_experiment", O.SCOPE_PAPER), ("full", O.SCOPE_FULL)):
        s, _ = O.sinr_compressed(d, fo["C"], fo["G"], cr[None, None], 0.1, 2, code)
        np.testing.assert_allclose(s[0, 0], GOLD[f"desk_sinr_{scope}"], rtol=1e-9)
    s, _ = O.sinr_full(d, Xr[None], cr[None, None], 0.1, 2, O.SCOPE_PAPER)
    np.testing.assert_allclose(s[0, 0], GOLD["desk_full_sinr"], rtol=1e-9)


# ------------------------------------------------------------------ restated reference tests
def test_mode_product_identity_commute_and_errors():  # test_tensor.cpp:61-119
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 4, 5)) + 1j * rng.standard_normal((3, 4, 5))
    for mode, d in ((1, 3), (2, 4), (3, 5)):
        np.testing.assert_allclose(O.mode_product(x, np.eye(d), mode), x, atol=0)
    u1 = rng.standard_normal((2, 3)) + 0j
    u3 = rng.standard_normal((6, 5)) + 0j
    a = O.mode_product(O.mode_product(x, u1, 1), u3, 3)
    b = O.mode_product(O.mode_product(x, u3, 3), u1, 1)
    np.testing.assert_allclose(a, b, rtol=1e-13)
    np.testing.assert_allclose(a, np.einsum("ai,ijk,ck->ajc", u1, x, u3), rtol=1e-12)
    with pytest.raises(O.OracleError, match="mode 3"):
        O.mode_product(x, np.eye(4), 3)


def test_contract_mode3_selects_slice():  # test_tensor.cpp:134-160
    rng = np.random.default_rng(2)
    x = rng.standard_normal((3, 4, 5)) + 1j * rng.standard_normal((3, 4, 5))
    e = np.zeros(5, complex)
    e[2] = 1
    np.testing.assert_array_equal(O.contract_mode3(x, e), x[:, :, 2])
    c = rng.standard_normal(5) + 1j * rng.standard_normal(5)
    np.testing.assert_allclose(O.contract_mode3(x, c), np.einsum("abq,q->ab", x, np.conj(c)), rtol=1e-13)
    with pytest.raises(O.OracleError, match="coefficient length 4 does not match mode-3 size 5"):
        O.contract_mode3(x, c[:4])


def test_hosvd_exact_rank_and_energy_identity():  # test_decompose.cpp:55-79
    rng = np.random.default_rng(3)
    core = rng.standard_normal((2, 3, 2)) + 1j * rng.standard_normal((2, 3, 2))
    q1 = np.linalg.qr(rng.standard_normal((5, 2)) + 1j * rng.standard_normal((5, 2)))[0]
    q2 = np.linalg.qr(rng.standard_normal((6, 3)) + 1j * rng.standard_normal((6, 3)))[0]
    q3 = np.linalg.qr(rng.standard_normal((4, 2)) + 1j * rng.standard_normal((4, 2)))[0]
    x = np.einsum("ai,bj,ck,ijk->abc", q1, q2, q3, core)
    A, B, Cc, G = O.hosvd(x, 2, 3, 2)
    xr = O.reconstruct(A, B, Cc, G)
    assert np.linalg.norm(xr - x) <= 1e-12 * np.linalg.norm(x)
    # truncation: residual == ||X||^2 - ||G||^2
    y = rng.standard_normal((5, 6, 4)) + 1j * rng.standard_normal((5, 6, 4))
    A, B, Cc, G = O.hosvd(y, 2, 3, 2)
    res = np.sum(np.abs(y - O.reconstruct(A, B, Cc, G)) ** 2)
    assert abs(res - (np.sum(np.abs(y) ** 2) - np.sum(np.abs(G) ** 2))) <= 1e-10 * np.sum(np.abs(y) ** 2)
    with pytest.raises(O.OracleError, match="rank m = 6 out of range for mode-1 size 5"):
        O.hosvd(y, 6, 1, 1)


def test_hooi_exact_rank_one_sweep():  # test_decompose.cpp:105-114
    rng = np.random.default_rng(4)
    core = rng.standard_normal((2, 2, 2)) + 1j * rng.standard_normal((2, 2, 2))
    qs = [np.linalg.qr(rng.standard_normal((d, 2)) + 1j * rng.standard_normal((d, 2)))[0] for d in (4, 5, 3)]
    x = np.einsum("ai,bj,ck,ijk->abc", *qs, core)
    *_, tr, it = O.hooi(x, 2, 2, 2, 3)
    assert tr[-1] <= 1e-20 * np.sum(np.abs(x) ** 2)


def test_groupwise_contracts():  # test_decompose.cpp:152-160, test_acceptance.cpp:178-218
    Xr, _ = O.generate_reference(2, 2, 6, 8, 5, 21)
    d = dict(DESK, m=3, n=4, p=3)
    fo = O.alternating_solve(d, Xr[None], 8, early_stop=False)
    tr = fo["trace"][0]
    assert (np.diff(tr) <= 1e-12 * fo["energy"][0]).all()  # monotone
    for u in range(4):
        a = fo["A"][0, u].T
        assert np.linalg.norm(a.conj().T @ a - np.eye(3)) < 1e-12
    # f + g = sum ||X||^2
    f, g = O.objective(d, Xr, fo["A"][0], fo["B"][0], fo["C"][0])
    assert abs(f + g - fo["energy"][0]) <= 1e-10 * fo["energy"][0]
    assert abs(f - tr[-1]) <= 1e-10 * fo["energy"][0]


def test_groupwise_1x1_matches_hooi():  # test_decompose.cpp:134-140
    Xr, _ = O.generate_reference(1, 1, 6, 8, 5, 33)
    d = dict(J=1, K=1, M=6, N=8, P=5, m=3, n=4, p=2)
    fo = O.alternating_solve(d, Xr[None], 4, early_stop=False)
    *_, tr, it = O.hooi(nat(Xr)[0], 3, 4, 2, 4)
    np.testing.assert_allclose(fo["trace"][0][: it + 1], tr[: it + 1], rtol=1e-10)


def test_lossless_compressed_equals_full():  # test_sinr.cpp:337-365, test_acceptance.cpp:143-176
    Xr, cr = O.generate_reference(2, 2, 6, 8, 5, 12)
    d = dict(DESK, m=6, n=8, p=5)
    fo = O.alternating_solve(d, Xr[None], 2)
    comp, _ = O.sinr_compressed(d, fo["C"], fo["G"], cr[None, None], 0.1, 2, O.SCOPE_PAPER)
    full, _ = O.sinr_full(d, Xr[None], cr[None, None], 0.1, 2, O.SCOPE_PAPER)
    np.testing.assert_allclose(comp, full, rtol=1e-8)


def test_truncated_compressed_equals_full_on_rebuilt():  # test_sinr.cpp:413-425
    Xr, cr = O.generate_reference(2, 2, 6, 8, 5, 14)
    d = dict(DESK, m=4, n=5, p=3)
    fo = O.alternating_solve(d, Xr[None], 6)
    comp, _ = O.sinr_compressed(d, fo["C"], fo["G"], cr[None, None], 0.1, 2, O.SCOPE_PAPER)
    hs = []
    for l in range(8):
        k, i, j = l // 4, (l // 2) % 2, l % 2
        a, b, c = fo["A"][0, i * 2 + j].T, fo["B"][0, k].T, fo["C"][0, l].T
        g = np.transpose(fo["G"][0, l], (2, 1, 0))
        h_small = np.einsum("abq,q->ab", g, np.conj(c.conj().T @ cr[l]))
        hs.append((a @ h_small @ b.T).T)  # transposed tx factor (sinr.cpp:342-344)
    ref, _ = O.evaluate_assembled(2, 2, 2, 0.1, np.array(hs), O.SCOPE_PAPER)
    np.testing.assert_allclose(comp[0, 0], ref, rtol=1e-8)


def test_single_link_closed_form():  # test_sinr.cpp:161-174
    for seed in (11, 22, 33):
        Xr, cr = O.generate_reference(1, 1, 6, 8, 5, seed)
        s, _ = O.sinr_full(dict(J=1, K=1, M=6, N=8, P=5), Xr[None], cr[None, None], 0.3, 1, O.SCOPE_FULL)
        h = O.contract_mode3(nat(Xr)[0], cr[0])
        s1 = np.linalg.svd(h, compute_uv=False)[0]
        assert abs(s[0, 0, 0, 0] - s1 ** 2 / 0.09) <= 1e-10 * s1 ** 2 / 0.09


def test_noise_dominated_sinr_vanishes():  # test_sinr.cpp:235-245
    Xr, cr = O.generate_reference(1, 1, 6, 8, 5, 9)
    s, _ = O.sinr_full(dict(J=1, K=1, M=6, N=8, P=5), Xr[None], cr[None, None], 1e6, 2, O.SCOPE_FULL)
    assert (s < 1e-6).all()


def test_precoder_stream_count_error():  # test_sinr.cpp:379-389
    d = dict(J=2, K=1, M=3, N=4, P=2, m=3, n=4, p=2)
    z = np.zeros((1, 2, 2, 2), complex)
    G = np.ones((1, 2, 2, 4, 3), complex)
    with pytest.raises(O.OracleError, match="stream count"):
        O.sinr_compressed(d, z, G, np.ones((1, 1, 2, 2), complex), 0.1, 4, O.SCOPE_PAPER)


def test_flop_ledger_spot_values():  # test_sinr.cpp:427-470
    topo = gw.SystemTopology(21, 5, 64, 512, 401, 4, 0.1)
    r = gw.CompressionRanks(60, 230, 150)
    full, comp = gw.flop_estimate(topo, r, "full"), gw.flop_estimate(topo, r, "compressed")
    links = 21 * 21 * 5
    assert full.reconstruct // links == 13139968
    assert comp.reconstruct // links == 2130150
    assert full.total() > comp.total()
    # the oracle pipeline charges exactly the closed form
    Xr, cr = O.generate_reference(2, 2, 6, 8, 5, 15)
    d = dict(DESK, m=4, n=5, p=3)
    fo = O.alternating_solve(d, Xr[None], 2)
    _, _, led = O.sinr_compressed(d, fo["C"], fo["G"], cr[None, None], 0.1, 2, O.SCOPE_PAPER, with_ledger=True)
    want = gw.flop_estimate(gw.SystemTopology(2, 2, 6, 8, 5, 2, 0.1), gw.CompressionRanks(4, 5, 3))
    assert list(led) == [want.reconstruct, want.precoder, want.covariance, want.inverse, want.filter, want.sinr]


def test_reference_generator_rank_one_and_determinism():  # test_channel.cpp:28-56
    a, ca = O.generate_reference(2, 2, 6, 8, 5, 7, rays=1)
    b, cb = O.generate_reference(2, 2, 6, 8, 5, 7, rays=1)
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(ca, cb)
    s = np.linalg.svd(a[0, 3].T, compute_uv=False)
    assert s[1] <= 1e-12 * s[0]
    with pytest.raises(O.OracleError, match="rays_per_slice"):
        O.generate_reference(1, 1, 2, 2, 2, 0, rays=0)


@pytest.mark.parametrize("name,ngroups,group0", [("C1", 4, 0), ("C2", 2, 5), ("C4", 1, 300)])
def test_baseline_generator_bit_identical(name, ngroups, group0):
    """The oracle's generator (used by bench.py's reference arm, which loads no product code) and the
    product's gwt_generate_channels produce bit-identical X and tau, in both precisions."""
    cfg = gw.CONFIGS[name]
    t = cfg.topology()
    for dt in (np.complex128, np.complex64):
        Xp, tp = gw.generate_channels(t, ngroups, seed=0, dtype=dt, group0=group0)
        Xo, to = O.generate_baseline(cfg.J, cfg.K, cfg.M, cfg.N, cfg.P, ngroups, seed=0, group0=group0, dtype=dt)
        assert Xp.tobytes() == Xo.tobytes()
        assert tp.tobytes() == to.tobytes()
