"""GPU parity: the B200 kernels (through the C ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star): per-stream SINR 1e-9 relative for
complex128, 1e-4 relative for complex64 (c64-rounded inputs, oracle in fp64);
reconstruction NMSE within 1e-6 absolute. Factors are compared only through
NMSE/SINR and subspace angles (unique up to phase/rotation).
"""
import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from oracle import oracle as O
from tests.helpers import baseline_inputs, dims_of, rel_err

pytestmark = pytest.mark.gpu

SINR_TOL = {"c128": 1e-9, "c64": 1e-4}


def _np_dtype(cfg):
    return np.complex64 if cfg.dtype == "c64" else np.complex128


def _oracle_factors(cfg, X128, sweeps=None, early=False):
    return O.alternating_solve(dims_of(cfg), X128, cfg.sweeps if sweeps is None else sweeps, early_stop=early)


def _max_angle(U1, U2):
    """sin of the largest principal angle between column spaces (oracles.hpp:113-118)."""
    Q1, _ = np.linalg.qr(U1)
    Q2, _ = np.linalg.qr(U2)
    R = Q2 - Q1 @ (Q1.conj().T @ Q2)
    return np.linalg.svd(R, compute_uv=False)[0] if R.size else 0.0


# ---------------------------------------------------------------------------
# linalg

@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 12, 17, 24, 32, 64, 128, 256])
def test_leading_eigenvectors_match_oracle_and_lapack(ctx, n):
    rng = np.random.default_rng(n)
    b = 3
    A = rng.standard_normal((b, n, n)) + 1j * rng.standard_normal((b, n, n))
    H = A @ np.conj(np.swapaxes(A, 1, 2))
    count = max(1, n // 2)
    vec, ev = ctx.leading_eigenvectors(H, count, with_values=True)
    for k in range(b):
        w = np.linalg.eigvalsh(H[k])[::-1][:count]
        assert np.max(np.abs(ev[k] - w)) <= 1e-10 * np.abs(w).max()
        ref = O.leading_eigenvectors(H[k], count)
        # same phase convention (linalg.cpp:11-25) => equal vectors for distinct eigenvalues
        assert np.max(np.abs(vec[k] - ref)) < 1e-8
        assert np.linalg.norm(vec[k].conj().T @ vec[k] - np.eye(count)) < 1e-10


@pytest.mark.parametrize("n,count", [(12, 5), (24, 12), (32, 12), (64, 8), (64, 24), (128, 40), (128, 64), (130, 40), (200, 48),
                                     (256, 64), (256, 128)])
def test_leading_eigenvectors_c64(ctx, n, count):
    """c64 Grams are decomposed in fp32 (warp kernel for n <= 32): subspace angle and eigenvalues vs fp64."""
    rng = np.random.default_rng(5 + n)
    A = rng.standard_normal((4, n, n)) + 1j * rng.standard_normal((4, n, n))
    H = (A @ np.conj(np.swapaxes(A, 1, 2))).astype(np.complex64)
    vec, ev = ctx.leading_eigenvectors(H, count, with_values=True)
    for k in range(4):
        ref = O.leading_eigenvectors(H[k].astype(np.complex128), count)
        assert _max_angle(vec[k].astype(np.complex128), ref) < 1e-3
        w = np.linalg.eigvalsh(H[k].astype(np.complex128))[::-1][:count]
        assert np.max(np.abs(ev[k] - w)) <= 1e-5 * np.abs(w).max()
        assert np.linalg.norm(vec[k].astype(np.complex128).conj().T @ vec[k] - np.eye(count)) < 1e-4


@pytest.mark.parametrize("n,count,batch", [(17, 6, 8), (31, 16, 40), (33, 10, 8), (47, 16, 96), (64, 16, 8), (64, 16, 96),
                                               (137, 40, 8), (256, 64, 16), (256, 96, 4)])
def test_leading_eigenvectors_c64_paths_decaying_spectrum(ctx, n, count, batch):
    """fp32 eigensolver code paths (register-resident warp Householder for 16 < n <= 32, the CTA kernel's
    register (batch <= 64) and shared-memory (batch > 64) Householder for 32 < n <= 64, division-free
    Sturm counts) on Gram-like spectra with exponential decay (clustered small eigenvalues, as the
    channel Grams have): eigenvalues and the top-count subspace vs fp64 LAPACK."""
    rng = np.random.default_rng(100 + n + batch)
    Z = rng.standard_normal((batch, n, n)) + 1j * rng.standard_normal((batch, n, n))
    Qm, _ = np.linalg.qr(Z)
    # decay e^-0.2 per index (at most e^-4 down to the count-th value for the large n, so the kept
    # subspace stays resolvable in fp32)
    lam = np.exp(-min(0.2, 4.0 / count) * np.arange(n)) * (1.0 + 0.05 * rng.random((batch, n)))
    H = ((Qm * lam[:, None, :]) @ np.conj(np.swapaxes(Qm, 1, 2))).astype(np.complex64)
    vec, ev = ctx.leading_eigenvectors(H, count, with_values=True)
    for k in range(0, batch, max(1, batch // 8)):
        Hk = H[k].astype(np.complex128)
        w, U = np.linalg.eigh(Hk)
        w, U = w[::-1][:count], U[:, ::-1][:, :count]
        assert np.max(np.abs(ev[k] - w)) <= 1e-5 * w[0]
        assert _max_angle(vec[k].astype(np.complex128), U) < 1e-3
        assert np.linalg.norm(vec[k].astype(np.complex128).conj().T @ vec[k] - np.eye(count)) < 1e-4


def test_woodbury_inverse_apply_matches_dense_inverse(ctx):
    """woodbury_inverse_apply on the device (sinr.cpp:205-227): T = Q^-1 (Q - s^2 I) vs a dense inverse, the
    lift Q (1/s^2)(I - T) = I (test_sinr.cpp:269-314), and the reference's error texts."""
    rng = np.random.default_rng(11)
    for m, b in ((4, 7), (8, 3), (24, 2)):
        A = rng.standard_normal((b, m, 2 * m)) + 1j * rng.standard_normal((b, m, 2 * m))
        sigma = 0.3
        Q = A @ np.conj(np.swapaxes(A, 1, 2)) + sigma ** 2 * np.eye(m)
        T, iss = ctx.woodbury_inverse_apply(Q, sigma)
        want = np.linalg.solve(Q, Q - sigma ** 2 * np.eye(m))
        assert np.max(np.abs(T - want)) <= 1e-10 * max(1.0, np.abs(want).max())
        lift = Q @ (iss * (np.eye(m) - T)) - np.eye(m)
        assert np.max(np.abs(lift)) <= 1e-8
    with pytest.raises(gw.InvalidArgument, match="sigma must be > 0"):
        ctx.woodbury_inverse_apply(np.eye(3, dtype=np.complex128)[None], 0.0)
    with pytest.raises(gw.NumericalError, match="covariance is numerically singular"):
        ctx.woodbury_inverse_apply(np.zeros((1, 3, 3), np.complex128), 0.1)
    ill = np.diag([1.0, 1e-15, 1.0]).astype(np.complex128)[None]
    with pytest.raises(gw.NumericalError, match="condition estimate above 1e14"):
        ctx.woodbury_inverse_apply(ill, 0.1)
    bad = np.eye(3, dtype=np.complex128)[None].copy()
    bad[0, 1, 1] = np.nan
    with pytest.raises(gw.InvalidArgument, match="non-finite input"):
        ctx.woodbury_inverse_apply(bad, 0.1)


def test_leading_eigenvectors_errors(ctx):
    H = np.eye(4, dtype=np.complex128)[None]
    with pytest.raises(gw.InvalidArgument, match="count 5 out of range for size 4"):
        ctx.leading_eigenvectors(H, 5)


# ---------------------------------------------------------------------------
# compressed assembly

@pytest.mark.parametrize("dt", [np.complex128, np.complex64])
def test_assemble_compressed_matches_definition(ctx, dt):
    rng = np.random.default_rng(7)
    topo = gw.SystemTopology(2, 2, 6, 8, 5, 2, 0.1)
    ranks = gw.CompressionRanks(4, 5, 3)
    g, F, links = 2, 3, topo.num_links
    Cd = (rng.standard_normal((g, links, 3, 5)) + 1j * rng.standard_normal((g, links, 3, 5))).astype(dt)
    G = (rng.standard_normal((g, links, 3, 5, 4)) + 1j * rng.standard_normal((g, links, 3, 5, 4))).astype(dt)
    co = (rng.standard_normal((g, F, links, 5)) + 1j * rng.standard_normal((g, F, links, 5))).astype(dt)
    H = ctx.assemble_compressed(topo, ranks, Cd, G, coeffs=co)
    # channel.cpp:189-208: d = C^H c, H~ = sum_q G(:,:,q) conj(d_q)
    d = np.einsum("glqr,gflr->gflq", np.conj(Cd.astype(np.complex128)), co.astype(np.complex128))
    want = np.einsum("glqba,gflq->gflba", G.astype(np.complex128), np.conj(d))
    tol = 1e-12 if dt == np.complex128 else 1e-5
    assert np.max(np.abs(H - want)) <= tol * np.abs(want).max()
    # oracle cross-check of one item through contract_mode3
    h_or = O.contract_mode3(np.transpose(G[1, 2].astype(np.complex128), (2, 1, 0)), d[1, 2, 2])
    assert np.max(np.abs(H[1, 2, 2].T - h_or)) <= tol * np.abs(h_or).max()


def test_assemble_from_delays(ctx):
    cfg = gw.CONFIGS["C1"]
    rng = np.random.default_rng(3)
    g, links = 2, cfg.G
    Cd = rng.standard_normal((g, links, cfg.p, cfg.P)) + 1j * rng.standard_normal((g, links, cfg.p, cfg.P))
    G = rng.standard_normal((g, links, cfg.p, cfg.n, cfg.m)) + 1j * rng.standard_normal((g, links, cfg.p, cfg.n, cfg.m))
    tau = rng.uniform(0, 1e-6, (g, links, cfg.P))
    freqs = cfg.freqs()[:7]
    H = ctx.assemble_compressed(cfg.topology(), cfg.ranks(), Cd, G, tau=tau, freqs=freqs)
    co = O.coeffs_from_tau(tau, freqs)
    d = np.einsum("glqr,gflr->gflq", np.conj(Cd), co)
    want = np.einsum("glqba,gflq->gflba", G, np.conj(d))
    assert np.max(np.abs(H - want)) <= 1e-12 * np.abs(want).max()


# ---------------------------------------------------------------------------
# SINR stage parity on identical factors

@pytest.mark.parametrize("name,ngroups,scope", [("C1", None, "paper_experiment"), ("C1", None, "full"),
                                                ("C2", 2, "paper_experiment"), ("C2d", 2, "paper_experiment")])
def test_sinr_stage_parity(ctx, name, ngroups, scope):
    cfg = gw.CONFIGS[name]
    X, X128, tau = baseline_inputs(cfg, ngroups)
    fo = _oracle_factors(cfg, X128, sweeps=4)
    dt = _np_dtype(cfg)
    Cd, G = fo["C"].astype(dt), fo["G"].astype(dt)
    freqs = cfg.freqs()
    oscope = O.SCOPE_FULL if scope == "full" else O.SCOPE_PAPER
    want, wsig = O.sinr_compressed(dims_of(cfg), Cd.astype(np.complex128), G.astype(np.complex128),
                                   O.coeffs_from_tau(tau, freqs), cfg.sigma, cfg.L, oscope, nthreads=8)
    fac = gw.GroupwiseFactorSet(None, None, Cd, G)
    rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), scope, tau=tau, freqs=freqs)
    assert (np.asarray(rep.status) == 0).all()
    tol = SINR_TOL[cfg.dtype]
    assert rel_err(rep.sinr, want).max() <= tol
    assert rel_err(rep.signal_power, wsig).max() <= tol
    led = gw.flop_estimate(cfg.topology(), cfg.ranks())
    assert rep.ledger.total() == led.total() * X.shape[0] * cfg.F


def test_sinr_explicit_coefficients_reference_generator(ctx):
    """Reference-style system (test_sinr.cpp desk_topology, seed 14): coefficient path, ranks (4,5,3)."""
    topo = gw.SystemTopology(2, 2, 6, 8, 5, 2, 0.1)
    X, c = O.generate_reference(2, 2, 6, 8, 5, 14)
    dims = dict(J=2, K=2, M=6, N=8, P=5, m=4, n=5, p=3)
    fo = O.alternating_solve(dims, X[None], 6)
    co = c[None, None]
    for scope, osc in (("paper_experiment", O.SCOPE_PAPER), ("full", O.SCOPE_FULL)):
        want, _ = O.sinr_compressed(dims, fo["C"], fo["G"], co, 0.1, 2, osc)
        rep = ctx.run_compressed_pipeline(topo, gw.GroupwiseFactorSet(None, None, fo["C"], fo["G"]),
                                          gw.CompressionRanks(4, 5, 3), scope, coeffs=co)
        assert rel_err(rep.sinr, want).max() <= 1e-9
        # and the reference's strongest pin: compressed == full pipeline on rebuilt channels (test_sinr.cpp:413-425)
        Hs = []
        for l, (k, i, j) in enumerate((k, i, j) for k in range(2) for i in range(2) for j in range(2)):
            u = i * 2 + j
            A = fo["A"][0, u].T
            B = fo["B"][0, k].T
            Cm = fo["C"][0, l].T
            core = np.transpose(fo["G"][0, l], (2, 1, 0))
            d = Cm.conj().T @ c[l]
            hs = np.einsum("abq,q->ab", core, np.conj(d))
            Hs.append((A @ hs @ B.T).T)
        ref_full, _ = O.evaluate_assembled(2, 2, 2, 0.1, np.array(Hs), osc)
        assert rel_err(rep.sinr[0, 0], ref_full).max() <= 1e-8


def test_sinr_closed_form_single_link(ctx):
    """SINR = sigma1^2 / sigma^2 for J=K=1, one stream (test_sinr.cpp:161-174, 391-399)."""
    topo = gw.SystemTopology(1, 1, 6, 8, 5, 1, 0.3)
    X, c = O.generate_reference(1, 1, 6, 8, 5, 13)
    dims = dict(J=1, K=1, M=6, N=8, P=5, m=6, n=8, p=5)
    fo = O.alternating_solve(dims, X[None], 1)
    rep = ctx.run_compressed_pipeline(topo, gw.GroupwiseFactorSet(None, None, fo["C"], fo["G"]),
                                      gw.CompressionRanks(6, 8, 5), "full", coeffs=c[None, None])
    h = O.contract_mode3(np.transpose(X[0], (2, 1, 0)), c[0])
    s1 = np.linalg.svd(h, compute_uv=False)[0]
    assert abs(rep.sinr[0, 0, 0, 0] - s1 * s1 / 0.09) <= 1e-8 * s1 * s1 / 0.09


def test_sinr_errors(ctx):
    topo = gw.SystemTopology(2, 1, 4, 8, 5, 4, 0.1)
    z = np.zeros((1, 2, 3, 5), np.complex128)
    G = np.zeros((1, 2, 3, 3, 4), np.complex128)
    with pytest.raises(gw.InvalidArgument, match="stream count"):
        ctx.run_compressed_pipeline(topo, gw.GroupwiseFactorSet(None, None, z, G), gw.CompressionRanks(4, 3, 3),
                                    coeffs=np.zeros((1, 1, 2, 5), np.complex128))


# ---------------------------------------------------------------------------
# Tucker compression parity

@pytest.mark.parametrize("name,ngroups", [("C1", None), ("C2d", 2), ("C2", 2)])
def test_groupwise_solve_nmse_parity(ctx, name, ngroups):
    cfg = gw.CONFIGS[name]
    X, X128, tau = baseline_inputs(cfg, ngroups)
    fo = _oracle_factors(cfg, X128)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), cfg.sweeps, early_stop=False)
    nmse_gpu = res.trace[:, -1] / res.energy
    nmse_orc = fo["trace"][:, -1] / fo["energy"]
    assert np.max(np.abs(nmse_gpu - nmse_orc)) <= 1e-6
    assert np.max(rel_err(res.energy, fo["energy"])) <= (1e-6 if cfg.dtype == "c64" else 1e-12)
    # every trace entry (init + each sweep) tracks the oracle
    assert np.max(np.abs(res.trace / res.energy[:, None] - fo["trace"] / fo["energy"][:, None])) <= 1e-6
    assert (np.asarray(res.iterations_run) == cfg.sweeps).all()
    # factors orthonormal, and their subspaces match the oracle's (fp64)
    if cfg.dtype == "c128":
        for g in range(X.shape[0]):
            for k in range(cfg.J):
                assert _max_angle(res.tx[g, k].T, fo["B"][g, k].T) < 1e-6
            for u in range(cfg.J * cfg.K):
                assert _max_angle(res.rx[g, u].T, fo["A"][g, u].T) < 1e-6


def test_groupwise_solve_early_stop_and_trace(ctx):
    cfg = gw.CONFIGS["C1"]
    X, X128, _ = baseline_inputs(cfg)
    fo = _oracle_factors(cfg, X128, sweeps=60, early=True)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), 60, early_stop=True)
    assert np.array_equal(np.asarray(res.iterations_run), fo["iters"])
    tr = np.asarray(res.trace)
    assert (np.diff(tr, axis=1) <= 1e-9 * res.energy[:, None]).all()  # monotone (decompose.hpp:33-41)
    assert np.max(np.abs(tr[:, -1] / res.energy - fo["trace"][:, -1] / fo["energy"])) <= 1e-6


def test_shared_solve_parity(ctx):
    cfg = gw.CONFIGS["C1"]
    X, X128, _ = baseline_inputs(cfg, 2)
    fo = O.alternating_solve(dims_of(cfg), X128, 5, early_stop=False, pooled=True)
    res = ctx.shared_solve(cfg.topology(), X, cfg.ranks(), 5, early_stop=False)
    assert np.max(np.abs(res.trace / res.energy[:, None] - fo["trace"] / fo["energy"][:, None])) <= 1e-9
    # every user carries the same receive factor
    assert np.allclose(res.rx[:, :1], res.rx)


def test_warm_start_and_zero_sweeps(ctx):
    cfg = gw.CONFIGS["C1"]
    X, X128, _ = baseline_inputs(cfg, 2)
    fo = _oracle_factors(cfg, X128, sweeps=3)
    init = gw.GroupwiseFactorSet(fo["A"], fo["B"], fo["C"], None)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), 0, init=init)
    assert rel_err(res.trace[:, 0], fo["trace"][:, -1]).max() <= 1e-10
    assert np.max(np.abs(res.cores - fo["G"])) <= 1e-10 * np.abs(fo["G"]).max()


def test_reconstruct_parity(ctx):
    cfg = gw.CONFIGS["C1"]
    X, X128, _ = baseline_inputs(cfg, 1)
    fo = _oracle_factors(cfg, X128, sweeps=2)
    fac = gw.GroupwiseFactorSet(fo["A"], fo["B"], fo["C"], fo["G"])
    Xh = ctx.reconstruct(cfg.topology(), cfg.ranks(), fac)
    for l in range(cfg.G):
        k, u = l // (cfg.J * cfg.K), l % (cfg.J * cfg.K)
        want = O.reconstruct(fo["A"][0, u].T, fo["B"][0, k].T, fo["C"][0, l].T, np.transpose(fo["G"][0, l], (2, 1, 0)))
        got = np.transpose(Xh[0, l], (2, 1, 0))
        assert np.max(np.abs(got - want)) <= 1e-12 * np.abs(want).max()


def test_solver_errors(ctx):
    cfg = gw.CONFIGS["C1"]
    X, _, _ = baseline_inputs(cfg, 1)
    with pytest.raises(gw.InvalidArgument, match="rank m = 5 out of range for mode-1 size 4"):
        ctx.groupwise_solve(cfg.topology(), X, gw.CompressionRanks(5, 4, 4), 1)
    with pytest.raises(gw.InvalidArgument, match="sweeps must be >= 0"):
        ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), -1)


def test_end_to_end_compress_then_sinr(ctx):
    """GPU compress -> GPU SINR against oracle compress -> oracle SINR (C1, fp64)."""
    cfg = gw.CONFIGS["C1"]
    X, X128, tau = baseline_inputs(cfg)
    fo = _oracle_factors(cfg, X128)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), cfg.sweeps, early_stop=False)
    rep = ctx.run_compressed_pipeline(cfg.topology(), res, cfg.ranks(), tau=tau, freqs=cfg.freqs())
    want, _ = O.sinr_compressed(dims_of(cfg), fo["C"], fo["G"], O.coeffs_from_tau(tau, cfg.freqs()), cfg.sigma,
                                cfg.L, O.SCOPE_PAPER, nthreads=8)
    assert rel_err(rep.sinr, want).max() <= 1e-6


def test_device_resident_torch_path(ctx):
    torch = pytest.importorskip("torch")
    cfg = gw.CONFIGS["C1"]
    X, X128, tau = baseline_inputs(cfg)
    Xd = torch.from_numpy(X).cuda()
    before = ctx.launches
    res = ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), 3, early_stop=False)
    rep = ctx.run_compressed_pipeline(cfg.topology(), res, cfg.ranks(), tau=torch.from_numpy(tau).cuda(),
                                      freqs=torch.from_numpy(cfg.freqs()).cuda())
    torch.cuda.synchronize()
    assert ctx.launches > before
    host = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), 3, early_stop=False)
    assert np.allclose(res.trace.cpu().numpy(), host.trace, rtol=1e-12, atol=0)
    assert rep.sinr.is_cuda


def test_cpp_dropin_api_on_gpu():
    """The gwt:: C++ drop-in library (host/) runs the reference's test idioms on the B200."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_09792_b200", "_build",
                       "test_dropin")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASSED" in r.stdout


@pytest.mark.parametrize("mode", [1, 2, 3])
def test_mode_product_matches_oracle(ctx, mode):
    rng = np.random.default_rng(mode)
    X = rng.standard_normal((3, 5, 4, 3)) + 1j * rng.standard_normal((3, 5, 4, 3))  # [b, d3, d2, d1]
    d = (3, 4, 5)[mode - 1]
    U = rng.standard_normal((2, d)) + 1j * rng.standard_normal((2, d))
    Y = ctx.mode_product(X, U, mode)
    for b in range(3):
        want = O.mode_product(np.transpose(X[b], (2, 1, 0)), U, mode)
        assert np.max(np.abs(np.transpose(Y[b], (2, 1, 0)) - want)) <= 1e-12 * np.abs(want).max()
    with pytest.raises(gw.InvalidArgument, match="mode 3 has size 5"):
        ctx.mode_product(X, np.eye(4, dtype=complex), 3)


@pytest.mark.parametrize("name,ngroups,sweeps,F", [("C3", 1, 2, 12), ("C4", 1, 1, 8), ("C5", 1, 2, 12)])
def test_large_configs_parity(ctx, name, ngroups, sweeps, F):
    """BASELINE C3/C4/C5 shapes (m=8, L=8, N up to 256, P up to 64) on a few groups: NMSE and SINR vs oracle."""
    cfg = gw.CONFIGS[name]
    X, X128, tau = baseline_inputs(cfg, ngroups)
    fo = O.alternating_solve(dims_of(cfg), X128, sweeps, early_stop=False, nthreads=8)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), sweeps, early_stop=False)
    assert np.max(np.abs(res.trace / res.energy[:, None] - fo["trace"] / fo["energy"][:, None])) <= 1e-6
    freqs = cfg.freqs()[:F]
    Cd, G = fo["C"].astype(np.complex64), fo["G"].astype(np.complex64)
    want, _ = O.sinr_compressed(dims_of(cfg), Cd.astype(np.complex128), G.astype(np.complex128),
                                O.coeffs_from_tau(tau, freqs), cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=8)
    rep = ctx.run_compressed_pipeline(cfg.topology(), gw.GroupwiseFactorSet(None, None, Cd, G), cfg.ranks(),
                                      tau=tau, freqs=freqs)
    assert (np.asarray(rep.status) == 0).all()
    assert rel_err(rep.sinr, want).max() <= 1e-4


@pytest.mark.parametrize("n,p", [(16, 8), (96, 32)])
def test_c5_rank_sweep_corners(ctx, n, p):
    """BASELINE C5 rank sweep corners (Nt-mode n in {16..96}, K-mode p in {8..32}) on the C5 shape:
    NMSE trace vs the oracle (exercises the count > 64 eigensolver route for n = 96)."""
    import dataclasses
    cfg = dataclasses.replace(gw.CONFIGS["C5"], n=n, p=p)
    X, X128, tau = baseline_inputs(cfg, 1)
    fo = O.alternating_solve(dims_of(cfg), X128, 2, early_stop=False, nthreads=8)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), 2, early_stop=False)
    assert np.max(np.abs(res.trace / res.energy[:, None] - fo["trace"] / fo["energy"][:, None])) <= 1e-6


@pytest.mark.parametrize("name,ngroups", [("C1", None), ("C2", 2), ("C2d", 2)])
def test_full_pipeline_parity(ctx, name, ngroups):
    """run_full_pipeline (the e_c / R_t comparator) on the uncompressed channels vs the oracle."""
    cfg = gw.CONFIGS[name]
    X, X128, tau = baseline_inputs(cfg, ngroups)
    freqs = cfg.freqs()[:32]
    want, wsig = O.sinr_full(dims_of(cfg), X128, O.coeffs_from_tau(tau, freqs), cfg.sigma, cfg.L, O.SCOPE_PAPER,
                             nthreads=8)
    rep = ctx.run_full_pipeline(cfg.topology(), X, tau=tau, freqs=freqs)
    assert (np.asarray(rep.status) == 0).all()
    assert rel_err(rep.sinr, want).max() <= SINR_TOL[cfg.dtype]
    led = gw.flop_estimate(cfg.topology(), cfg.ranks(), "full")
    assert rep.ledger.total() == led.total() * X.shape[0] * len(freqs)


def test_full_pipeline_reference_generator_and_lossless_identity(ctx):
    """Reference desk system: full path vs oracle, and lossless compressed == full (test_sinr.cpp:337-365)."""
    from paper_2401_09792_b200 import metrics
    topo = gw.SystemTopology(2, 2, 6, 8, 5, 2, 0.1)
    X, c = O.generate_reference(2, 2, 6, 8, 5, 12)
    co = c[None, None]
    for scope, osc in (("paper_experiment", O.SCOPE_PAPER), ("full", O.SCOPE_FULL)):
        want, _ = O.sinr_full(dict(J=2, K=2, M=6, N=8, P=5), X[None], co, 0.1, 2, osc)
        full = ctx.run_full_pipeline(topo, X[None], scope, coeffs=co)
        assert rel_err(full.sinr, want).max() <= 1e-9
    fac = ctx.groupwise_solve(topo, X[None], gw.CompressionRanks(6, 8, 5), 2)
    comp = ctx.run_compressed_pipeline(topo, fac, gw.CompressionRanks(6, 8, 5), coeffs=co)
    full = ctx.run_full_pipeline(topo, X[None], coeffs=co)
    assert rel_err(comp.sinr, full.sinr).max() <= 1e-8
    assert metrics.sinr_error(full.sinr, comp.sinr) <= 1e-8


def test_individual_solve_matches_per_link_hooi(ctx):
    """individual_solve == single-tensor HOOI per link (test_decompose.cpp:326-335), warm start supported."""
    cfg = gw.CONFIGS["C1"]
    X, X128, _ = baseline_inputs(cfg, 1)
    res = ctx.individual_solve(cfg.topology(), X, cfg.ranks(), 4)
    for l in (0, 5):
        *_, tr, it = O.hooi(np.transpose(X128[0, l], (2, 1, 0)), cfg.m, cfg.n, cfg.p, 4)
        np.testing.assert_allclose(res["link_trace"][0, l], tr, rtol=1e-9, atol=1e-12 * tr[0])
    fo = O.alternating_solve(dims_of(cfg), X128, 3)
    warm = ctx.individual_solve(cfg.topology(), X, cfg.ranks(), 0,
                                init=gw.GroupwiseFactorSet(fo["A"], fo["B"], fo["C"], None))
    # warm start at the groupwise factors: link objectives sum to the groupwise objective
    assert abs(warm["trace"][0, 0] - fo["trace"][0, -1]) <= 1e-9 * fo["energy"][0]


def test_archive_round_trip_of_gpu_factors(ctx, tmp_path):
    from paper_2401_09792_b200 import archive as ar
    cfg = gw.CONFIGS["C1"]
    X, _, tau = baseline_inputs(cfg, 1)
    fac = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), 3)
    co = O.coeffs_from_tau(tau, cfg.freqs()[:1])[0, 0]
    ar.save_archive(tmp_path / "c.gwtk", "groupwise", fac, co, cfg.J, cfg.K)
    out = ar.load_archive(tmp_path / "c.gwtk")
    a = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), coeffs=co[None, None])
    b = ctx.run_compressed_pipeline(cfg.topology(), out["factors"], cfg.ranks(), coeffs=out["coeffs"][None, None])
    np.testing.assert_array_equal(a.sinr, b.sinr)
