"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of the Eigen-free C++ restatement of the reference
(`oracle/gwt_oracle.cpp`, following /root/reference/proj/src/*.cpp; see the
header of gwt_oracle.hpp for how parity is pinned). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline legs may import this.
Arrays are numpy complex128 in the product's layouts.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

SCOPE_FULL = 0
SCOPE_PAPER = 1


class OracleError(Exception):
    """Raised with the reference's exception text; .kind is 'invalid_argument' or 'runtime_error'."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.kind = {1: "invalid_argument", 2: "runtime_error"}.get(code, "error")


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _call(fn, *args):
    err = C.create_string_buffer(1024)
    rc = fn(*args, err, C.c_int(1024))
    if rc != 0:
        raise OracleError(rc, err.value.decode())


def generate_reference(J, K, M, N, P, seed, rays=4, tap_decay=0.7, rician=10.0, coeff_decay=0.8):
    """Reference generator (channel.cpp:154-180). Returns X [links,P,N,M] and coeffs [links,P]."""
    links = J * J * K
    X = np.zeros((links, P, N, M), np.complex128)
    c = np.zeros((links, P), np.complex128)
    _call(lib().orc_generate_reference, C.c_int(J), C.c_int(K), C.c_int(M), C.c_int(N), C.c_int(P), C.c_int(rays),
          C.c_double(tap_decay), C.c_double(rician), C.c_double(coeff_decay), C.c_ulonglong(seed), _p(X), _p(c))
    return X, c


def generate_baseline(J, K, M, N, P, ngroups, seed=0, group0=0, dtype=np.complex128, pdp_decay=0.3,
                      max_delay=1e-6, nthreads=None):
    """BASELINE.json generator (oracle/gen_baseline.cpp), bit-identical to the product's.
    Returns X [g, links, P, N, M] (complex128 or complex64) and tau [g, links, P]."""
    links = J * J * K
    X = np.empty((ngroups, links, P, N, M), dtype)
    tau = np.empty((ngroups, links, P), np.float64)
    rc = lib().orc_generate_baseline(C.c_int(J), C.c_int(K), C.c_int(M), C.c_int(N), C.c_int(P),
                                     C.c_longlong(group0), C.c_longlong(ngroups), C.c_ulonglong(seed),
                                     C.c_double(pdp_decay), C.c_double(max_delay),
                                     C.c_int(1 if X.dtype == np.complex64 else 0), _p(X), _p(tau),
                                     C.c_int(nthreads or os.cpu_count() or 1))
    if rc != 0:
        raise OracleError(1, "generate_baseline: invalid topology")
    return X, tau


def heev(a):
    a = _c128(a)
    n = a.shape[0]
    w = np.zeros(n)
    v = np.zeros((n, n), np.complex128, order="F")
    af = np.asfortranarray(a)
    _call(lib().orc_heev, C.c_int(n), _p(af), _p(w), _p(v))
    return w, v


def leading_eigenvectors(a, count):
    af = np.asfortranarray(_c128(a))
    n = af.shape[0]
    out = np.zeros((n, count), np.complex128, order="F")
    _call(lib().orc_leading_eigenvectors, C.c_int(n), _p(af), C.c_int(count), _p(out))
    return out


def truncated_svd(a, count):
    af = np.asfortranarray(_c128(a))
    r, c = af.shape
    u = np.zeros((r, count), np.complex128, order="F")
    s = np.zeros(count)
    v = np.zeros((c, count), np.complex128, order="F")
    _call(lib().orc_truncated_svd, C.c_int(r), C.c_int(c), _p(af), C.c_int(count), _p(u), _p(s), _p(v))
    return u, s, v


def mode_product(x, u, mode):
    """x: numpy array indexed x[i1,i2,i3] (stored mode-1 fastest via Fortran order)."""
    xf = np.asfortranarray(_c128(x))
    uf = np.asfortranarray(_c128(u))
    dims = list(xf.shape)
    dims[mode - 1] = uf.shape[0]
    y = np.zeros(dims, np.complex128, order="F")
    _call(lib().orc_mode_product, C.c_int(xf.shape[0]), C.c_int(xf.shape[1]), C.c_int(xf.shape[2]), _p(xf),
          C.c_int(uf.shape[0]), C.c_int(uf.shape[1]), _p(uf), C.c_int(mode), _p(y))
    return y


def contract_mode3(x, c):
    xf = np.asfortranarray(_c128(x))
    cc = _c128(c)
    h = np.zeros(xf.shape[:2], np.complex128, order="F")
    _call(lib().orc_contract_mode3, C.c_int(xf.shape[0]), C.c_int(xf.shape[1]), C.c_int(xf.shape[2]), _p(xf),
          C.c_int(cc.size), _p(cc), _p(h))
    return h


def hosvd(x, m, n, p):
    xf = np.asfortranarray(_c128(x))
    d1, d2, d3 = xf.shape
    A = np.zeros((d1, m), np.complex128, order="F")
    B = np.zeros((d2, n), np.complex128, order="F")
    Cc = np.zeros((d3, p), np.complex128, order="F")
    G = np.zeros((m, n, p), np.complex128, order="F")
    _call(lib().orc_hosvd, C.c_int(d1), C.c_int(d2), C.c_int(d3), _p(xf), C.c_int(m), C.c_int(n), C.c_int(p),
          _p(A), _p(B), _p(Cc), _p(G))
    return A, B, Cc, G


def hooi(x, m, n, p, sweeps):
    xf = np.asfortranarray(_c128(x))
    d1, d2, d3 = xf.shape
    A = np.zeros((d1, m), np.complex128, order="F")
    B = np.zeros((d2, n), np.complex128, order="F")
    Cc = np.zeros((d3, p), np.complex128, order="F")
    G = np.zeros((m, n, p), np.complex128, order="F")
    tr = np.zeros(sweeps + 1)
    it = C.c_int(0)
    _call(lib().orc_hooi, C.c_int(d1), C.c_int(d2), C.c_int(d3), _p(xf), C.c_int(m), C.c_int(n), C.c_int(p),
          C.c_int(sweeps), _p(A), _p(B), _p(Cc), _p(G), _p(tr), C.byref(it))
    return A, B, Cc, G, tr, it.value


def reconstruct(A, B, Cc, G):
    M, m = A.shape
    N, n = B.shape
    P, p = Cc.shape
    X = np.zeros((M, N, P), np.complex128, order="F")
    _call(lib().orc_reconstruct, C.c_int(M), C.c_int(N), C.c_int(P), C.c_int(m), C.c_int(n), C.c_int(p),
          _p(np.asfortranarray(_c128(A))), _p(np.asfortranarray(_c128(B))), _p(np.asfortranarray(_c128(Cc))),
          _p(np.asfortranarray(_c128(G))), _p(X))
    return X


def alternating_solve(dims, X, sweeps, early_stop=True, pooled=False, init=None, nthreads=1):
    """dims: dict J,K,M,N,P,m,n,p. X: [ngroups, links, P, N, M] complex128 (product layout).

    Returns dict with A [g,users,m,M], B [g,J,n,N], C [g,links,p,P], G [g,links,p,n,m],
    trace [g, sweeps+1], iters [g], energy [g]."""
    d = dims
    J, K, M, N, P, m, n, p = (d[k] for k in ("J", "K", "M", "N", "P", "m", "n", "p"))
    X = _c128(X)
    g = X.shape[0]
    users, links = J * K, J * J * K
    out = dict(
        A=np.zeros((g, users, m, M), np.complex128), B=np.zeros((g, J, n, N), np.complex128),
        C=np.zeros((g, links, p, P), np.complex128), G=np.zeros((g, links, p, n, m), np.complex128),
        trace=np.zeros((g, sweeps + 1)), iters=np.zeros(g, np.int32), energy=np.zeros(g))
    iA = iB = iC = None
    if init is not None:
        iA, iB, iC = (_c128(init[k]) for k in ("A", "B", "C"))
    _call(lib().orc_alternating_solve, *(C.c_int(v) for v in (J, K, M, N, P, m, n, p)), C.c_longlong(g), _p(X),
          C.c_int(sweeps), C.c_int(int(early_stop)), C.c_int(int(pooled)), _p(iA), _p(iB), _p(iC),
          C.c_int(nthreads), _p(out["A"]), _p(out["B"]), _p(out["C"]), _p(out["G"]), _p(out["trace"]),
          _p(out["iters"]), _p(out["energy"]))
    return out


def objective(dims, X, A, B, Cc):
    """One group. Returns (f, g): residual and captured energy."""
    d = dims
    f = C.c_double(0)
    gg = C.c_double(0)
    _call(lib().orc_objective, *(C.c_int(d[k]) for k in ("J", "K", "M", "N", "P", "m", "n", "p")), _p(_c128(X)),
          _p(_c128(A)), _p(_c128(B)), _p(_c128(Cc)), C.byref(f), C.byref(gg))
    return f.value, gg.value


def update_gram(which, dims, X, A, B, Cc, a, b=0, c=0):
    d = dims
    size = {0: d["M"], 1: d["N"], 2: d["P"]}[which]
    out = np.zeros((size, size), np.complex128, order="F")
    _call(lib().orc_update_gram, C.c_int(which), *(C.c_int(d[k]) for k in ("J", "K", "M", "N", "P", "m", "n", "p")),
          _p(_c128(X)), _p(_c128(A)), _p(_c128(B)), _p(_c128(Cc)), C.c_int(a), C.c_int(b), C.c_int(c), _p(out))
    return out


def coeffs_from_tau(tau, freqs):
    """c_q(f) = exp(+j 2 pi f tau_q). tau: [g, links, P]; freqs [F] -> [g, F, links, P]."""
    ph = np.einsum("f,glp->gflp", np.asarray(freqs, np.float64), np.asarray(tau, np.float64))
    ph = ph - np.floor(ph)
    return np.exp(2j * np.pi * ph)


def sinr_compressed(dims, Cd, G, coeffs, sigma, L, scope=SCOPE_PAPER, nthreads=1, with_ledger=False):
    """Cd: [g, links, p, P]; G: [g, links, p, n, m]; coeffs [g, F, links, P].

    Returns sinr, signal [g, F, users, L] (and ledger[6] if requested)."""
    d = dims
    J, K, P, m, n, p = (d[k] for k in ("J", "K", "P", "m", "n", "p"))
    coeffs = _c128(coeffs)
    g, F = coeffs.shape[:2]
    users = J * K
    sinr = np.zeros((g, F, users, L))
    sig = np.zeros_like(sinr)
    led = np.zeros(6, np.int64)
    _call(lib().orc_sinr_compressed, C.c_int(J), C.c_int(K), C.c_int(P), C.c_int(m), C.c_int(n), C.c_int(p),
          C.c_int(L), C.c_double(sigma), C.c_int(scope), C.c_longlong(g), _p(_c128(Cd)), _p(_c128(G)), _p(coeffs),
          C.c_longlong(F), C.c_int(nthreads), _p(sinr), _p(sig), _p(led))
    return (sinr, sig, led) if with_ledger else (sinr, sig)


def sinr_full(dims, X, coeffs, sigma, L, scope=SCOPE_PAPER, nthreads=1, with_ledger=False):
    d = dims
    J, K, M, N, P = (d[k] for k in ("J", "K", "M", "N", "P"))
    coeffs = _c128(coeffs)
    g, F = coeffs.shape[:2]
    users = J * K
    sinr = np.zeros((g, F, users, L))
    sig = np.zeros_like(sinr)
    led = np.zeros(6, np.int64)
    _call(lib().orc_sinr_full, C.c_int(J), C.c_int(K), C.c_int(M), C.c_int(N), C.c_int(P), C.c_int(L),
          C.c_double(sigma), C.c_int(scope), C.c_longlong(g), _p(_c128(X)), _p(coeffs), C.c_longlong(F),
          C.c_int(nthreads), _p(sinr), _p(sig), _p(led))
    return (sinr, sig, led) if with_ledger else (sinr, sig)


def evaluate_assembled(J, K, L, sigma, H, scope=SCOPE_PAPER):
    """H: [links, N, M] (column-major M x N per link)."""
    H = _c128(H)
    links, N, M = H.shape
    users = J * K
    sinr = np.zeros((users, L))
    sig = np.zeros_like(sinr)
    _call(lib().orc_evaluate_assembled, C.c_int(J), C.c_int(K), C.c_int(M), C.c_int(N), C.c_int(L),
          C.c_double(sigma), C.c_int(scope), _p(H), _p(sinr), _p(sig))
    return sinr, sig


# ---------------------------------------------------------------------------
# parity metrics (checker side)
def serving_singular_values(cfg, Cd, G, tau, fidx):
    """Singular values of every user's serving compressed channel H~_iij(f) (binary64 rebuild of the given
    factors), [g, F, users, min(m, n)] descending."""
    J, K, m, n, p, P = cfg.J, cfg.K, cfg.m, cfg.n, cfg.p, cfg.P
    g = Cd.shape[0]
    links = J * J * K
    co = coeffs_from_tau(tau, cfg.freqs()[fidx])
    C128 = np.asarray(Cd, np.complex128).reshape(g, links, p, P)
    G128 = np.asarray(G, np.complex128).reshape(g, links, p, n, m)
    serving = [(i * J + i) * K + j for i in range(J) for j in range(K)]
    d = np.einsum("glqP,gflP->gflq", C128[:, serving], np.conj(co[:, :, serving]))
    H = np.einsum("glqnm,gflq->gflnm", G128[:, serving], d)
    return np.linalg.svd(H, compute_uv=False)


def sinr_cluster_err(got, want, sv, gap=2e-2):
    """Parity of per-stream SINR with near-degenerate serving singular pairs handled as clusters.

    Where two consecutive serving singular values are within `gap` (relative), the split of the
    per-stream SINR between those streams is ill-conditioned (a relative perturbation e of H~ rotates
    the singular pair by ~e sigma^2 / (sigma_r^2 - sigma_r+1^2)); there the cluster sum of
    gamma = SINR / (1 + SINR) (rotation invariant) is compared instead. Returns (max relative error
    over well-separated streams and cluster sums, max raw per-stream error, number of clustered items)."""
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    L = got.shape[-1]
    s = np.asarray(sv)[..., :L]
    close = np.zeros(got.shape, bool)
    if L > 1:
        c = (s[..., :-1] - s[..., 1:]) <= gap * s[..., :-1]
        close[..., :-1] |= c
        close[..., 1:] |= c
    raw = np.abs(got - want) / np.abs(want)
    err = np.where(close, 0.0, raw)
    gg, gw_ = got / (1 + got), want / (1 + want)
    # cluster label: runs of consecutive 'close' streams
    lab = np.zeros(got.shape, np.int64)
    for r in range(1, L):
        lab[..., r] = lab[..., r - 1] + (~(close[..., r] & close[..., r - 1] & ((s[..., r - 1] - s[..., r]) <= gap * s[..., r - 1]))).astype(np.int64)
    worst = err.max() if err.size else 0.0
    idx = np.argwhere(close.any(-1))
    for ix in map(tuple, idx):
        for cl in np.unique(lab[ix][close[ix]]):
            sel = (lab[ix] == cl) & close[ix]
            a, b = gg[ix][sel].sum(), gw_[ix][sel].sum()
            worst = max(worst, abs(a - b) / abs(b))
    return float(worst), float(raw.max()), int(len(idx))


# ---------------------------------------------------------------------------
# oracle/_ref: the reference's own sources compiled against the Eigen-subset shim (oracle/Makefile `ref`)

_REF_PATH = os.path.join(_HERE, "_ref", "libgwtref.so")
_ref = None


def ref_available() -> bool:
    if os.path.exists(_REF_PATH):
        return True
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
        return os.path.exists(_REF_PATH)
    return False


def ref_lib():
    global _ref
    if _ref is None:
        if not ref_available():
            raise OSError("oracle/_ref/libgwtref.so not built (needs /root/reference)")
        _ref = C.CDLL(_REF_PATH)
        _ref.ref_model_name.restype = C.c_char_p
    return _ref


def ref_groupwise_solve(dims, X, sweeps, pooled=False):
    """The reference's gwt::groupwise_solve (its own stop rule) on each group of X [g, links, P, N, M]."""
    d = dims
    J, K, M, N, P, m, n, p = (d[k] for k in ("J", "K", "M", "N", "P", "m", "n", "p"))
    X = _c128(X)
    g = X.shape[0]
    users, links = J * K, J * J * K
    out = dict(A=np.zeros((g, users, m, M), np.complex128), B=np.zeros((g, J, n, N), np.complex128),
               C=np.zeros((g, links, p, P), np.complex128), G=np.zeros((g, links, p, n, m), np.complex128),
               trace=np.zeros((g, sweeps + 1)), iters=np.zeros(g, np.int32))
    _call(ref_lib().ref_groupwise_solve, *(C.c_int(v) for v in (J, K, M, N, P, m, n, p)), C.c_longlong(g), _p(X),
          C.c_int(sweeps), C.c_int(int(pooled)), _p(out["A"]), _p(out["B"]), _p(out["C"]), _p(out["G"]),
          _p(out["trace"]), _p(out["iters"]))
    return out


def ref_sinr_compressed(dims, Cd, G, coeffs, sigma, L, scope=SCOPE_PAPER):
    d = dims
    J, K, P, m, n, p = (d[k] for k in ("J", "K", "P", "m", "n", "p"))
    coeffs = _c128(coeffs)
    g, F = coeffs.shape[:2]
    sinr = np.zeros((g, F, J * K, L))
    sig = np.zeros_like(sinr)
    led = np.zeros(6, np.int64)
    _call(ref_lib().ref_sinr_compressed, *(C.c_int(v) for v in (J, K, P, m, n, p, L)), C.c_double(sigma),
          C.c_int(scope), C.c_longlong(g), _p(_c128(Cd)), _p(_c128(G)), _p(coeffs), C.c_longlong(F), _p(sinr), _p(sig),
          _p(led))
    return sinr, sig, led


def ref_sinr_full(dims, X, coeffs, sigma, L, scope=SCOPE_PAPER):
    d = dims
    J, K, M, N, P = (d[k] for k in ("J", "K", "M", "N", "P"))
    coeffs = _c128(coeffs)
    g, F = coeffs.shape[:2]
    sinr = np.zeros((g, F, J * K, L))
    sig = np.zeros_like(sinr)
    _call(ref_lib().ref_sinr_full, *(C.c_int(v) for v in (J, K, M, N, P, L)), C.c_double(sigma), C.c_int(scope),
          C.c_longlong(g), _p(_c128(X)), _p(coeffs), C.c_longlong(F), _p(sinr), _p(sig))
    return sinr, sig


def ref_generate_channel_set(J, K, M, N, P, seed, rays=4, tap_decay=0.7, rician=10.0, coeff_decay=0.8):
    links = J * J * K
    X = np.zeros((links, P, N, M), np.complex128)
    c = np.zeros((links, P), np.complex128)
    _call(ref_lib().ref_generate_channel_set, *(C.c_int(v) for v in (J, K, M, N, P, rays)), C.c_double(tap_decay),
          C.c_double(rician), C.c_double(coeff_decay), C.c_ulonglong(seed), _p(X), _p(c))
    return X, c


def ref_save_archive(path, model, dims, A, B, Cd, G, coeffs):
    d = dims
    _call(ref_lib().ref_save_archive, str(path).encode(), C.c_int(model),
          *(C.c_int(d[k]) for k in ("J", "K", "M", "N", "P", "m", "n", "p")), _p(_c128(A)), _p(_c128(B)),
          _p(_c128(Cd)), _p(_c128(G)), _p(_c128(coeffs)))


def ref_model_name(kind):
    return ref_lib().ref_model_name(C.c_int(kind)).decode()


def ref_model_from_name(name):
    err = C.create_string_buffer(256)
    rc = ref_lib().ref_model_from_name(name.encode(), err, C.c_int(256))
    if rc < 0:
        raise OracleError(-1 - rc, err.value.decode())
    return rc
