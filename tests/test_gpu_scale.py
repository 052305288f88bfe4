"""GPU parity at BASELINE scale on the exact paths bench.py times.

* The device-resident SINR path (torch CUDA tensors; the call bench.py times)
  and the pinned-host-buffer path (the e2e call, group chunks over copy and
  compute streams) on ALL of C2 (64 groups x 272 subcarriers) and C2d, element
  by element against the oracle's run_compressed_pipeline on the same factors
  (proj/src/sinr.cpp:296-326).
* C4 (the headline) on 8 groups over all 3276 subcarriers, compared on a
  strided subset; C3 and C5 likewise.
* Tucker at C3/C4/C5 on 4 groups (C4: 5 sweeps, others 20) against the
  oracle's own groupwise_solve (decompose.cpp:309-373): NMSE within 1e-6 for
  every trace entry, and the oracle objective evaluated on the GPU factors.
* bench.py's self-check (parity_sample) on a C2 run.
"""
import os

import numpy as np
import pytest

import paper_2401_09792_b200 as gw
from oracle import oracle as O
from tests.helpers import baseline_inputs, dims_of, rel_err, serving_singular_values, sinr_cluster_err

pytestmark = pytest.mark.gpu

SINR_TOL = {"c128": 1e-9, "c64": 1e-4}
NT = max(1, min(32, len(os.sched_getaffinity(0))))


def _gpu_factors(ctx, cfg, X, sweeps):
    torch = pytest.importorskip("torch")
    Xd = torch.from_numpy(X).cuda()
    fac = ctx.groupwise_solve(cfg.topology(), Xd, cfg.ranks(), sweeps, early_stop=False)
    return Xd, fac


def _oracle_sinr(cfg, fac_np_C, fac_np_G, tau, fidx):
    co = O.coeffs_from_tau(tau, cfg.freqs()[fidx])
    want, sig = O.sinr_compressed(dims_of(cfg), fac_np_C.astype(np.complex128), fac_np_G.astype(np.complex128), co,
                                  cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=NT)
    return want, sig


@pytest.mark.parametrize("name", ["C2", "C2d"])
def test_full_c2_device_and_host_paths(ctx, name):
    torch = pytest.importorskip("torch")
    cfg = gw.CONFIGS[name]
    X, _, tau = baseline_inputs(cfg)
    assert X.shape[0] == cfg.groups == 64
    Xd, fac = _gpu_factors(ctx, cfg, X, 4)
    taud = torch.from_numpy(tau).cuda()
    freqs = torch.from_numpy(cfg.freqs()).cuda()
    # device-resident path (the one bench.py times), all groups x all subcarriers
    rep_d = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=taud, freqs=freqs)
    torch.cuda.synchronize()
    Cn, Gn = fac.delay.cpu().numpy(), fac.cores.cpu().numpy()
    want, wsig = _oracle_sinr(cfg, Cn, Gn, tau, np.arange(cfg.F))
    assert (rep_d.status.cpu().numpy() == 0).all()
    got = rep_d.sinr.cpu().numpy()
    assert got.shape == want.shape == (64, cfg.F, cfg.J * cfg.K, cfg.L)
    assert rel_err(got, want).max() <= SINR_TOL[cfg.dtype]
    assert rel_err(rep_d.signal_power.cpu().numpy(), wsig).max() <= 10 * SINR_TOL[cfg.dtype]
    # host-buffer path (the e2e call): pinned torch and plain numpy
    for Ch, Gh, th, fh in ((fac.delay.cpu().pin_memory(), fac.cores.cpu().pin_memory(),
                            torch.from_numpy(tau).pin_memory(), torch.from_numpy(cfg.freqs()).pin_memory()),
                           (Cn, Gn, tau, cfg.freqs())):
        rep_h = ctx.run_compressed_pipeline(cfg.topology(), gw.GroupwiseFactorSet(None, None, Ch, Gh), cfg.ranks(),
                                            tau=th, freqs=fh)
        st = rep_h.status.numpy() if hasattr(rep_h.status, "numpy") else rep_h.status
        assert (np.asarray(st) == 0).all()
        hs = rep_h.sinr.numpy() if hasattr(rep_h.sinr, "numpy") else rep_h.sinr
        # same kernels on the same inputs: bit-identical to the device-resident result
        np.testing.assert_array_equal(np.asarray(hs), got)


@pytest.mark.parametrize("name,ngroups,nf", [("C4", 8, 48), ("C3", 8, 48), ("C5", 8, 48)])
def test_large_config_sinr_all_subcarriers(ctx, name, ngroups, nf):
    """All subcarriers computed on the device; a strided subset compared with the oracle."""
    torch = pytest.importorskip("torch")
    cfg = gw.CONFIGS[name]
    X, _, tau = baseline_inputs(cfg, ngroups)
    Xd, fac = _gpu_factors(ctx, cfg, X, 1)
    rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=torch.from_numpy(tau).cuda(),
                                      freqs=torch.from_numpy(cfg.freqs()).cuda())
    torch.cuda.synchronize()
    assert tuple(rep.sinr.shape) == (ngroups, cfg.F, cfg.J * cfg.K, cfg.L)
    assert int(rep.status.ne(0).sum()) == 0
    fidx = np.unique(np.r_[np.linspace(0, cfg.F - 1, nf).astype(np.int64), cfg.F - 1])
    Cn, Gn = fac.delay.cpu().numpy(), fac.cores.cpu().numpy()
    want, _ = _oracle_sinr(cfg, Cn, Gn, tau, fidx)
    got = rep.sinr.cpu().numpy()[:, fidx]
    # per-stream within 1e-4; streams of a near-degenerate serving singular pair (relative gap < 2 %,
    # where the per-stream split is ill-conditioned in H~) are compared through their cluster sum
    err, raw, nclust = sinr_cluster_err(got, want, serving_singular_values(cfg, Cn, Gn, tau, fidx))
    assert err <= SINR_TOL[cfg.dtype], (err, raw, nclust)
    assert raw <= 50 * SINR_TOL[cfg.dtype], (err, raw, nclust)


@pytest.mark.parametrize("name,sweeps", [("C3", 20), ("C4", 5), ("C5", 20)])
def test_large_config_tucker_nmse(ctx, name, sweeps):
    """4 groups: every trace entry's NMSE within 1e-6 of the oracle's own solve, early-stop iteration
    counts equal, and the oracle objective (explicit reconstruction) on the GPU factors equal to the
    GPU's reported objective."""
    cfg = gw.CONFIGS[name]
    X, X128, _ = baseline_inputs(cfg, 4)
    fo = O.alternating_solve(dims_of(cfg), X128, sweeps, early_stop=False, nthreads=NT)
    res = ctx.groupwise_solve(cfg.topology(), X, cfg.ranks(), sweeps, early_stop=False)
    nm_g = np.asarray(res.trace) / np.asarray(res.energy)[:, None]
    nm_o = fo["trace"] / fo["energy"][:, None]
    assert np.max(np.abs(nm_g - nm_o)) <= 1e-6
    f_o, _ = O.objective(dims_of(cfg), X128[0], res.rx[0].astype(np.complex128), res.tx[0].astype(np.complex128),
                         res.delay[0].astype(np.complex128))
    assert abs(f_o / fo["energy"][0] - nm_g[0, -1]) <= 1e-6


def test_bench_self_check_on_c2(ctx):
    """bench.py's parity_sample on a real timed-path output (C2)."""
    torch = pytest.importorskip("torch")
    import bench
    cfg = gw.CONFIGS["C2"]
    X, _, tau = baseline_inputs(cfg, 4)
    Xd, fac = _gpu_factors(ctx, cfg, X, cfg.sweeps)
    rep = ctx.run_compressed_pipeline(cfg.topology(), fac, cfg.ranks(), tau=torch.from_numpy(tau).cuda(),
                                      freqs=torch.from_numpy(cfg.freqs()).cuda())
    out = bench.parity_sample(O, cfg, fac, Xd, tau, rep, groups=2, nfreq=16, nthreads=NT)
    assert out["ok"], out


def test_rank_sweep_c5_matches_oracle(ctx):
    """run_sweep (runner.cpp:193-211) over the C5 transmit rank on 4 groups x 64 subcarriers: R_s is the closed
    form, e_c equals the oracle's mean relative error between ITS full-size and compressed SINR on the GPU's
    factors (metrics.cpp:36-56), and the NMSE falls as the rank grows."""
    torch = pytest.importorskip("torch")
    from paper_2401_09792_b200 import metrics, sweep
    cfg = gw.CONFIGS["C5"]
    X, X128, tau = baseline_inputs(cfg, 4)
    freqs = cfg.freqs()[:64]
    Xd = torch.from_numpy(X).cuda()
    rows = sweep.run_sweep(ctx, cfg.topology(), cfg.ranks(), "n", [16, 64], Xd, torch.from_numpy(tau).cuda(),
                           torch.from_numpy(freqs).cuda(), sweeps=4, repetitions=1)
    assert [r.value for r in rows] == [16, 64]
    assert rows[0].nmse > rows[1].nmse
    dims_full = dims_of(cfg)
    co = O.coeffs_from_tau(tau, freqs)
    want_full, _ = O.sinr_full(dims_full, X128, co, cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=NT)
    for r in rows:
        rk = gw.CompressionRanks(cfg.m, r.value, cfg.p)
        assert r.r_s == pytest.approx(metrics.storage_ratio(cfg.topology(), rk))
        fac = ctx.groupwise_solve(cfg.topology(), Xd, rk, 4, early_stop=False)
        d = dict(dims_full, n=r.value)
        want_c, _ = O.sinr_compressed(d, fac.delay.cpu().numpy().astype(np.complex128),
                                      fac.cores.cpu().numpy().astype(np.complex128), co, cfg.sigma, cfg.L,
                                      O.SCOPE_PAPER, nthreads=NT)
        e_oracle = metrics.sinr_error(want_full, want_c)
        assert abs(r.e_c - e_oracle) <= 1e-4 * max(e_oracle, 1e-3), (r.e_c, e_oracle)


@pytest.mark.parametrize("name,dt,tol", [("C2", np.complex128, 1e-12), ("C2", np.complex64, 2e-6),
                                         ("C4", np.complex128, 1e-12), ("C4", np.complex64, 2e-6)])
@pytest.mark.parametrize("mode", [1, 2, 3])
def test_mode_product_baseline_shapes(ctx, name, dt, tol, mode):
    """gwt::mode_product (tensor.cpp:96-116) at the BASELINE tensor shapes and ranks: a batch of channel tensors
    [P, N, M] times U^H-shaped factors (rank x dim), against the oracle's mode_product on the same values."""
    cfg = gw.CONFIGS[name]
    rng = np.random.default_rng(17 + mode)
    M, N, P = cfg.M, cfg.N, cfg.P
    rank = (cfg.m, cfg.n, cfg.p)[mode - 1]
    d = (M, N, P)[mode - 1]
    b = 3
    X = (rng.standard_normal((b, P, N, M)) + 1j * rng.standard_normal((b, P, N, M))).astype(dt)
    U = (rng.standard_normal((rank, d)) + 1j * rng.standard_normal((rank, d))).astype(dt)
    Y = ctx.mode_product(X, U, mode)
    assert Y.dtype == dt
    for i in range(b):
        want = O.mode_product(np.transpose(X[i].astype(np.complex128), (2, 1, 0)), U.astype(np.complex128), mode)
        got = np.transpose(Y[i], (2, 1, 0))
        assert got.shape == want.shape
        assert np.max(np.abs(got - want)) <= tol * np.abs(want).max()
