"""Python mirror of the reference's hot-path API (gwt:: in /root/reference/proj/include/gwtucker).

Same names, argument meaning and error behaviour as the reference, batched over
independent channel groups (and subcarriers), executed by the B200 kernels
through the C ABI (include/gwt_b200.h). Arrays may be numpy arrays or torch
tensors: CUDA tensors run zero-copy on device (GWT_MEM_DEVICE); host arrays are
copied in and out inside the call (GWT_MEM_HOST). Complex dtype selects the
arithmetic: complex64 -> fp32 kernels (fp64 m x m solves), complex128 -> fp64.

Errors: the reference throws std::invalid_argument / std::runtime_error; here
those surface as ``InvalidArgument`` (a ValueError) and ``NumericalError`` (a
RuntimeError) with the reference's message text.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

try:  # torch is plumbing only (device memory, streams); numpy works too
    import torch
except Exception:  # pragma: no cover
    torch = None


class InvalidArgument(ValueError):
    pass


class NumericalError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


SCOPE = {"full": L.GWT_SCOPE_FULL, "paper_experiment": L.GWT_SCOPE_PAPER}

# per-item status -> (exception, reference message) (sinr.cpp:23-43, 205-227)
ITEM_ERRORS = {
    1: (NumericalError, "woodbury_inverse_apply: covariance is numerically singular"),
    2: (NumericalError, "woodbury_inverse_apply: covariance is numerically singular (condition estimate above 1e14)"),
    3: (NumericalError, "sinr: interference-plus-noise power is negative for stream {stream} (numerically invalid "
                        "configuration)"),
    4: (InvalidArgument, "woodbury_inverse_apply: non-finite input"),
}


class ModelKind(enum.IntEnum):
    """gwt::ModelKind (decompose.hpp:12): which factor-sharing model a solve / archive uses."""
    individual = 0
    shared = 1
    groupwise = 2


def model_name(model: ModelKind) -> str:
    """gwt::model_name (decompose.cpp:42-49)."""
    try:
        return ModelKind(model).name
    except ValueError:
        return "unknown"


def model_from_name(name: str) -> ModelKind:
    """gwt::model_from_name (decompose.cpp:51-56); throws the reference's invalid_argument text."""
    if name in ModelKind.__members__:
        return ModelKind[name]
    raise InvalidArgument(f"unknown model '{name}' (expected individual, shared or groupwise)")


@dataclass
class SystemTopology:
    """gwt::SystemTopology (channel.hpp:13-27)."""
    num_cells: int
    users_per_cell: int
    rx_antennas: int
    tx_antennas: int
    num_taps: int
    num_streams: int = 1
    noise_std: float = 0.1

    @property
    def num_users(self):
        return self.num_cells * self.users_per_cell

    @property
    def num_links(self):
        return self.num_cells * self.num_cells * self.users_per_cell

    def c(self):
        return L.Topology(self.num_cells, self.users_per_cell, self.rx_antennas, self.tx_antennas, self.num_taps,
                          self.num_streams, float(self.noise_std))


@dataclass
class CompressionRanks:
    """gwt::CompressionRanks (decompose.hpp:18-24)."""
    m: int
    n: int
    p: int

    def c(self):
        return L.Ranks(self.m, self.n, self.p)


@dataclass
class GroupwiseFactorSet:
    """gwt::GroupwiseFactorSet + SolveTrace (decompose.hpp:33-68), batched over groups.

    rx [g, users, m, M] (col-major M x m per user), tx [g, J, n, N], delay [g, links, p, P],
    cores [g, links, p, n, m]; trace [g, sweeps+1]; iterations_run [g]; energy [g] = sum ||X||^2."""
    rx: object
    tx: object
    delay: object
    cores: object
    trace: object = None
    iterations_run: object = None
    energy: object = None


@dataclass
class SinrReport:
    """gwt::SinrReport (sinr.hpp:51-62), batched: sinr/signal_power [g, F, users, L], status [g, F, users]."""
    sinr: object
    signal_power: object
    status: object
    ledger: L.Ledger = field(default_factory=L.Ledger)
    stage_ms: tuple = ()

    def raise_first_error(self):
        """Rethrow the reference's exception for the first failing (subcarrier, user) in reference order."""
        st = self.status.cpu().numpy() if hasattr(self.status, "cpu") else np.asarray(self.status)
        code = st & 0xFF  # status code; code 3 carries the first failing stream in bits 8+
        bad = np.flatnonzero((code != 0) & (code != 5))
        if bad.size:
            v = int(st.reshape(-1)[bad[0]])
            exc, msg = ITEM_ERRORS[v & 0xFF]
            raise exc(msg.format(stream=v >> 8))

    @property
    def rank_deficient(self):
        """Items whose interfering anchor had a zero singular value among its L kept streams (status 5): the
        reference's SVD completes that precoder with arbitrary null-space columns, which the Gram route cannot
        reproduce; the reference raises nothing there, so neither does raise_first_error."""
        st = self.status.cpu().numpy() if hasattr(self.status, "cpu") else np.asarray(self.status)
        return (st & 0xFF) == 5


# ---------------------------------------------------------------------------
# array plumbing

def _is_torch(a):
    return torch is not None and isinstance(a, torch.Tensor)


def _dtype_code(a):
    if _is_torch(a):
        if a.dtype == torch.complex64:
            return L.GWT_C64
        if a.dtype == torch.complex128:
            return L.GWT_C128
    else:
        if a.dtype == np.complex64:
            return L.GWT_C64
        if a.dtype == np.complex128:
            return L.GWT_C128
    raise InvalidArgument(f"complex64 or complex128 array expected, got {a.dtype}")


def _mem(a):
    return L.GWT_MEM_DEVICE if (_is_torch(a) and a.is_cuda) else L.GWT_MEM_HOST


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        if not a.is_contiguous():
            raise InvalidArgument("arrays must be contiguous")
        return C.c_void_p(a.data_ptr())
    if not a.flags["C_CONTIGUOUS"]:
        raise InvalidArgument("arrays must be contiguous")
    return C.c_void_p(a.ctypes.data)


def _like(ref, shape, kind):
    """Allocate an output next to `ref`: kind 'c' (ref's complex dtype), 'f64', 'i32'."""
    if _is_torch(ref):
        dt = {"c": ref.dtype, "f64": torch.float64, "i32": torch.int32}[kind]
        pin = (not ref.is_cuda) and ref.is_pinned()
        return torch.empty(shape, dtype=dt, device=ref.device, pin_memory=pin)
    dt = {"c": ref.dtype, "f64": np.float64, "i32": np.int32}[kind]
    return np.empty(shape, dtype=dt)


def _as_f64(ref, a):
    """Real binary64 side arrays (tau, freqs) in the same memory space as `ref`."""
    if a is None:
        return None
    if _is_torch(ref):
        t = a if _is_torch(a) else torch.as_tensor(np.asarray(a, np.float64))
        return t.to(device=ref.device, dtype=torch.float64).contiguous()
    return np.ascontiguousarray(np.asarray(a.cpu().numpy() if _is_torch(a) else a, np.float64))


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


class Context:
    """Owns a gwt_ctx (CUDA stream, workspaces). One per host thread."""

    _bound = None

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = C.c_void_p()
        rc = self.lib.gwt_ctx_create(C.byref(h), device)
        if rc == L.GWT_NO_DEVICE:
            raise CudaError("gwt: no CUDA device available (the B200 path has no CPU fallback)")
        if rc != L.GWT_OK:
            raise CudaError(f"gwt_ctx_create failed with status {rc}")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.gwt_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def use_stream(self, stream_handle: int | None):
        """Bind the context to a CUDA stream handle; None restores the context's own stream. Handle 0 is the
        legacy default stream and is passed as cudaStreamLegacy (the C ABI maps NULL to the own stream)."""
        if stream_handle is None:
            self.lib.gwt_ctx_set_stream(self.h, None)
        else:
            self.lib.gwt_ctx_set_stream(self.h, C.c_void_p(stream_handle if stream_handle else _CUDA_STREAM_LEGACY))
        self._bound = stream_handle

    def use_torch_stream(self):
        """Run on torch's current CUDA stream so torch events bracket our kernels."""
        self.use_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def _bind(self, *arrays):
        """Calls with torch CUDA tensors run on torch's current stream, so torch work queued before the call
        (copies, transposes, allocator reuse) is ordered before our kernels; host-only calls keep the
        context's own stream."""
        if any(_is_torch(a) and a.is_cuda for a in arrays if a is not None):
            h = torch.cuda.current_stream(self.device).cuda_stream
            if h != self._bound:
                self.use_stream(h)
        elif self._bound is not None:
            self.use_stream(None)

    @property
    def launches(self) -> int:
        return int(self.lib.gwt_ctx_launch_count(self.h))

    def stage_ms(self):
        buf = (C.c_double * 8)()
        self.lib.gwt_ctx_stage_times(self.h, buf)
        return tuple(buf)

    def check(self, rc):
        if rc == L.GWT_OK:
            return
        msg = self.lib.gwt_last_error(self.h).decode()
        if rc == L.GWT_INVALID_ARGUMENT:
            raise InvalidArgument(msg)
        if rc == L.GWT_RUNTIME_ERROR:
            raise NumericalError(msg)
        raise CudaError(msg)

    # ------------------------------------------------------------------ solvers
    def groupwise_solve(self, topo: SystemTopology, X, ranks: CompressionRanks, sweeps: int, init=None,
                        early_stop: bool = True, pooled: bool = False) -> GroupwiseFactorSet:
        """gwt::groupwise_solve (decompose.hpp:126-128; pooled=True is gwt::shared_solve :132-134).

        X: [groups, links, P, N, M] complex. init: GroupwiseFactorSet warm start (rx, tx, delay)."""
        J, K, M, N, P = topo.num_cells, topo.users_per_cell, topo.rx_antennas, topo.tx_antennas, topo.num_taps
        users, links = J * K, J * J * K
        if tuple(X.shape[1:]) != (links, P, N, M):
            raise InvalidArgument("channel set: inconsistent tensor dims")
        g = X.shape[0]
        m, n, p = ranks.m, ranks.n, ranks.p
        flags = (L.GWT_SOLVE_EARLY_STOP if early_stop else 0) | (L.GWT_SOLVE_POOLED if pooled else 0)
        if init is not None:
            flags |= L.GWT_SOLVE_INIT
            if (tuple(init.rx.shape) != (g, users, m, M) or tuple(init.tx.shape) != (g, J, n, N)
                    or tuple(init.delay.shape) != (g, links, p, P)):
                raise InvalidArgument("solver init: factor set shape does not match channels/ranks")
            A = init.rx.clone() if _is_torch(init.rx) else np.array(init.rx, copy=True)
            B = init.tx.clone() if _is_torch(init.tx) else np.array(init.tx, copy=True)
            Cd = init.delay.clone() if _is_torch(init.delay) else np.array(init.delay, copy=True)
        else:
            A = _like(X, (g, users, max(m, 1), M), "c")
            B = _like(X, (g, J, max(n, 1), N), "c")
            Cd = _like(X, (g, links, max(p, 1), P), "c")
        G = _like(X, (g, links, max(p, 1), max(n, 1), max(m, 1)), "c")
        trace = _like(X, (g, max(sweeps, 0) + 1), "f64")
        iters = _like(X, (g,), "i32")
        energy = _like(X, (g,), "f64")
        self._bind(X, A, B, Cd)
        rc = self.lib.gwt_groupwise_solve(self.h, C.byref(topo.c()), C.byref(ranks.c()), g, _dtype_code(X), _mem(X),
                                          _ptr(X), sweeps, flags, _ptr(A), _ptr(B), _ptr(Cd), _ptr(G), _ptr(trace),
                                          _ptr(iters), _ptr(energy))
        self.check(rc)
        return GroupwiseFactorSet(A, B, Cd, G, trace, iters, energy)

    def shared_solve(self, topo, X, ranks, sweeps, init=None, early_stop=True):
        """gwt::shared_solve (decompose.hpp:132-134): one rx and one tx factor per group."""
        return self.groupwise_solve(topo, X, ranks, sweeps, init=init, early_stop=early_stop, pooled=True)

    def individual_solve(self, topo, X, ranks, sweeps, init: GroupwiseFactorSet | None = None,
                         early_stop: bool = True):
        """gwt::individual_solve (decompose.cpp:389-435): independent per-link HOOI, optionally warm-started
        from a groupwise solution. Runs as the batched solver on J=K=1 systems (one per link).

        Returns dict: rx [g, links, m, M], tx [g, links, n, N], delay [g, links, p, P], cores [g, links, p, n, m],
        trace [g, sweeps+1] (per-sweep sum over links; stopped links hold their final value),
        iterations_run [g] (max over links), link_trace [g, links, sweeps+1]."""
        J, K = topo.num_cells, topo.users_per_cell
        g, links = X.shape[0], X.shape[1]
        one = SystemTopology(1, 1, topo.rx_antennas, topo.tx_antennas, topo.num_taps, 1, topo.noise_std)
        Xl = X.reshape((g * links, 1) + tuple(X.shape[2:]))
        ini = None
        if init is not None:
            ks = np.arange(links) // (J * K)
            us = np.arange(links) % (J * K)
            def per_link(arr, idx):
                a = arr[:, idx]
                return a.reshape((g * links, 1) + tuple(a.shape[2:]))
            ini = GroupwiseFactorSet(per_link(init.rx, us), per_link(init.tx, ks), init.delay.reshape(
                (g * links, 1) + tuple(init.delay.shape[2:])), None)
            if _is_torch(X):
                ini = GroupwiseFactorSet(*(torch.as_tensor(np.ascontiguousarray(x.cpu().numpy() if _is_torch(x) else x),
                                                           device=X.device) for x in (ini.rx, ini.tx, ini.delay)), None)
            else:
                ini = GroupwiseFactorSet(*(np.ascontiguousarray(x.cpu().numpy() if _is_torch(x) else x)
                                           for x in (ini.rx, ini.tx, ini.delay)), None)
        r = self.groupwise_solve(one, Xl.contiguous() if _is_torch(Xl) else np.ascontiguousarray(Xl), ranks, sweeps,
                                 init=ini, early_stop=early_stop)
        sh = lambda a: a.reshape((g, links) + tuple(a.shape[2:]))
        tr = r.trace.reshape(g, links, -1)
        it = r.iterations_run.reshape(g, links)
        return dict(rx=sh(r.rx), tx=sh(r.tx), delay=sh(r.delay), cores=sh(r.cores), link_trace=tr,
                    trace=tr.sum(1), iterations_run=it.max(1), energy=r.energy.reshape(g, links).sum(1))

    # ------------------------------------------------------------------ SINR
    def run_compressed_pipeline(self, topo: SystemTopology, factors: GroupwiseFactorSet, ranks: CompressionRanks,
                                scope: str = "paper_experiment", tau=None, freqs=None, coeffs=None,
                                raise_errors: bool = False) -> SinrReport:
        """gwt::run_compressed_pipeline (sinr.hpp:136-137) batched over groups and F coefficient grids.

        Either (tau [g, links, P] seconds, freqs [F] Hz) with c_q(f) = exp(+j 2 pi f tau_q), or explicit
        coeffs [g, F, links, P] complex (the reference's ChannelSet::coeffs, one grid per subcarrier)."""
        if scope not in SCOPE:
            raise InvalidArgument(f"unknown interference scope '{scope}'")
        Cd, G = factors.delay, factors.cores
        g = G.shape[0]
        users = topo.num_users
        ledger = L.Ledger()
        if coeffs is not None:
            F = coeffs.shape[1]
            sinr = _like(G, (g, F, users, topo.num_streams), "f64")
            sig = _like(G, (g, F, users, topo.num_streams), "f64")
            st = _like(G, (g, F, users), "i32")
            self._bind(G, Cd, coeffs)
            rc = self.lib.gwt_sinr_compressed_coeffs(self.h, C.byref(topo.c()), C.byref(ranks.c()), g,
                                                     _dtype_code(G), _mem(G), _ptr(Cd), _ptr(G), _ptr(coeffs), F,
                                                     SCOPE[scope], _ptr(sinr), _ptr(sig), _ptr(st), C.byref(ledger))
        else:
            tau = _as_f64(G, tau)
            freqs = _as_f64(G, freqs)
            F = freqs.shape[0]
            sinr = _like(G, (g, F, users, topo.num_streams), "f64")
            sig = _like(G, (g, F, users, topo.num_streams), "f64")
            st = _like(G, (g, F, users), "i32")
            self._bind(G, Cd, tau, freqs)
            rc = self.lib.gwt_sinr_compressed(self.h, C.byref(topo.c()), C.byref(ranks.c()), g, _dtype_code(G),
                                              _mem(G), _ptr(Cd), _ptr(G), _ptr(tau), _ptr(freqs), F, SCOPE[scope],
                                              _ptr(sinr), _ptr(sig), _ptr(st), C.byref(ledger))
        self.check(rc)
        rep = SinrReport(sinr, sig, st, ledger, self.stage_ms())
        if raise_errors:
            rep.raise_first_error()
        return rep

    def run_full_pipeline(self, topo: SystemTopology, X, scope: str = "paper_experiment", tau=None, freqs=None,
                          coeffs=None, raise_errors: bool = False) -> SinrReport:
        """gwt::run_full_pipeline (sinr.hpp:134) batched over groups and F coefficient grids: SINR on the
        uncompressed channels H(f) = X x3 c(f)^* (the comparator for the paper's e_c and R_t)."""
        if scope not in SCOPE:
            raise InvalidArgument(f"unknown interference scope '{scope}'")
        g = X.shape[0]
        users, L_ = topo.num_users, topo.num_streams
        ledger = L.Ledger()
        if coeffs is not None:
            F = coeffs.shape[1]
            tau_p = freqs_p = None
        else:
            tau, freqs = _as_f64(X, tau), _as_f64(X, freqs)
            F = freqs.shape[0]
            tau_p, freqs_p = _ptr(tau), _ptr(freqs)
        sinr = _like(X, (g, F, users, L_), "f64")
        sig = _like(X, (g, F, users, L_), "f64")
        st = _like(X, (g, F, users), "i32")
        self._bind(X, coeffs, tau, freqs)
        rc = self.lib.gwt_sinr_full(self.h, C.byref(topo.c()), g, _dtype_code(X), _mem(X), _ptr(X), tau_p, freqs_p,
                                    _ptr(coeffs), F, SCOPE[scope], _ptr(sinr), _ptr(sig), _ptr(st), C.byref(ledger))
        self.check(rc)
        rep = SinrReport(sinr, sig, st, ledger, self.stage_ms())
        if raise_errors:
            rep.raise_first_error()
        return rep

    def assemble_compressed(self, topo, ranks, delay, cores, tau=None, freqs=None, coeffs=None):
        """Batched gwt::assemble_channel_compressed (channel.hpp:78-79): H~ [g, F, links, n, m]."""
        g = cores.shape[0]
        if coeffs is not None:
            F = coeffs.shape[1]
            tau_p = freqs_p = None
        else:
            tau, freqs = _as_f64(cores, tau), _as_f64(cores, freqs)
            F = freqs.shape[0]
            tau_p, freqs_p = _ptr(tau), _ptr(freqs)
        H = _like(cores, (g, F, topo.num_links, ranks.n, ranks.m), "c")
        self._bind(cores, delay, coeffs, tau, freqs)
        rc = self.lib.gwt_assemble_compressed(self.h, C.byref(topo.c()), C.byref(ranks.c()), g, _dtype_code(cores),
                                              _mem(cores), _ptr(delay), _ptr(cores), tau_p, freqs_p, _ptr(coeffs), F,
                                              _ptr(H))
        self.check(rc)
        return H

    # ------------------------------------------------------------------ linalg
    def leading_eigenvectors(self, H, count: int, with_values: bool = False):
        """Batched gwt::leading_eigenvectors (linalg.hpp:16). H [batch, n, n] Hermitian (natural indexing).
        Returns vectors [batch, n, count] (columns descending, phase-normalised) and optionally eigenvalues."""
        b, n = H.shape[0], H.shape[-1]
        Hc = H.transpose(-1, -2).contiguous() if _is_torch(H) else np.ascontiguousarray(np.swapaxes(H, -1, -2))
        out = _like(H, (b, count, n), "c")
        ev = _like(H, (b, count), "f64") if with_values else None
        self._bind(Hc)
        rc = self.lib.gwt_leading_eigenvectors(self.h, n, count, b, _dtype_code(H), _mem(H), _ptr(Hc), _ptr(out),
                                               _ptr(ev))
        self.check(rc)
        vec = out.transpose(-1, -2) if _is_torch(out) else np.swapaxes(out, -1, -2)
        return (vec, ev) if with_values else vec

    def woodbury_inverse_apply(self, Q, sigma: float):
        """Batched gwt::woodbury_inverse_apply (sinr.hpp:121-122, sinr.cpp:205-227): Q [batch, m, m] Hermitian
        covariances (complex128, natural indexing). Returns (T [batch, m, m] = Q^-1 (Q - sigma^2 I),
        inv_sigma_sq). Device Cholesky with the reference's checks; raises the reference's errors for the
        first failing matrix."""
        b, m = Q.shape[0], Q.shape[-1]
        if _is_torch(Q):
            Qc = Q.to(dtype=torch.complex128).transpose(-1, -2).contiguous()
        else:
            Qc = np.ascontiguousarray(np.swapaxes(np.asarray(Q, dtype=np.complex128), -1, -2))
        if not sigma > 0.0:
            raise InvalidArgument("woodbury_inverse_apply: sigma must be > 0")
        eye = (torch.eye(m, dtype=Qc.dtype, device=Qc.device) if _is_torch(Qc) else np.eye(m, dtype=Qc.dtype))
        Bc = Qc - (sigma * sigma) * eye  # RHS Q - sigma^2 I (column-major like Qc; the shift is symmetric)
        Bc = Bc.contiguous() if _is_torch(Bc) else np.ascontiguousarray(Bc)
        T = _like(Qc, (b, m, m), "c")
        st = _like(Qc, (b,), "i32")
        self._bind(Qc, Bc)
        rc = self.lib.gwt_hpd_solve(self.h, m, m, b, _mem(Qc), _ptr(Qc), _ptr(Bc), 1, _ptr(T), _ptr(st))
        self.check(rc)
        sth = st.cpu().numpy() if _is_torch(st) else st
        bad = np.nonzero(sth)[0]
        if bad.size:
            code = int(sth[bad[0]])
            if code == 4:
                raise InvalidArgument("woodbury_inverse_apply: non-finite input")
            raise NumericalError("woodbury_inverse_apply: covariance is numerically singular" +
                                  (" (condition estimate above 1e14)" if code == 2 else ""))
        T = T.transpose(-1, -2) if _is_torch(T) else np.swapaxes(T, -1, -2)
        return T, 1.0 / (sigma * sigma)

    def mode_product(self, X, U, mode: int):
        """Batched gwt::mode_product (tensor.hpp:68-70): X [batch, d3, d2, d1] (mode-1 fastest), U natural
        [rows, dim(mode)] shared by the batch. Returns Y with dim(mode) replaced by rows."""
        b, d3, d2, d1 = X.shape
        rows, dm = U.shape
        if dm != (d1, d2, d3)[mode - 1] if 1 <= mode <= 3 else True:
            if not 1 <= mode <= 3:
                raise InvalidArgument(f"mode_product: mode must be 1, 2 or 3, got {mode}")
            raise InvalidArgument(f"mode_product: matrix has {dm} cols but tensor mode {mode} has size "
                                  f"{(d1, d2, d3)[mode - 1]}")
        Uc = (U.transpose(-1, -2).contiguous() if _is_torch(U) else np.ascontiguousarray(np.swapaxes(U, -1, -2)))
        o = [d1, d2, d3]
        o[mode - 1] = rows
        Y = _like(X, (b, o[2], o[1], o[0]), "c")
        self._bind(X, Uc)
        rc = self.lib.gwt_mode_product(self.h, _dtype_code(X), _mem(X), b, d1, d2, d3, _ptr(X), rows, _ptr(Uc), mode,
                                       _ptr(Y))
        self.check(rc)
        return Y

    def reconstruct(self, topo, ranks, factors: GroupwiseFactorSet):
        """gwt::reconstruct (decompose.hpp:84) per link: X^ [g, links, P, N, M]."""
        G = factors.cores
        g = G.shape[0]
        X = _like(G, (g, topo.num_links, topo.num_taps, topo.tx_antennas, topo.rx_antennas), "c")
        self._bind(G, factors.rx, factors.tx, factors.delay)
        rc = self.lib.gwt_reconstruct(self.h, C.byref(topo.c()), C.byref(ranks.c()), g, _dtype_code(G), _mem(G),
                                      _ptr(factors.rx), _ptr(factors.tx), _ptr(factors.delay), _ptr(G), _ptr(X))
        self.check(rc)
        return X


def flop_estimate(topo: SystemTopology, ranks: CompressionRanks, path: str = "compressed") -> L.Ledger:
    """gwt::flop_estimate (sinr.hpp:148-149), closed form on the host."""
    out = L.Ledger()
    rc = L.load().gwt_flop_estimate(C.byref(topo.c()), C.byref(ranks.c()), 0 if path == "full" else 1, C.byref(out))
    if rc != 0:
        raise InvalidArgument("flop_estimate: invalid topology or ranks")
    return out


def generate_channels(topo: SystemTopology, ngroups: int, seed: int = 0, dtype=np.complex128, group0: int = 0,
                      pdp_decay: float = 0.3, max_delay: float = 1e-6, nthreads: int = 8, out=None):
    """BASELINE.json generator. Returns numpy X [g, links, P, N, M] and tau [g, links, P]."""
    links = topo.num_links
    shape = (ngroups, links, topo.num_taps, topo.tx_antennas, topo.rx_antennas)
    X = out if out is not None else np.empty(shape, dtype)
    tau = np.empty((ngroups, links, topo.num_taps), np.float64)
    code = L.GWT_C64 if X.dtype == np.complex64 else L.GWT_C128
    rc = L.load().gwt_generate_channels(C.byref(topo.c()), group0, ngroups, seed, pdp_decay, max_delay, code,
                                        C.c_void_p(X.ctypes.data), C.c_void_p(tau.ctypes.data), nthreads)
    if rc != 0:
        raise InvalidArgument("generate_channels: invalid topology")
    return X, tau
