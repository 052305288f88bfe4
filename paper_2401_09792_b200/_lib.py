"""ctypes binding of the C ABI in include/gwt_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``)
into ``paper_2401_09792_b200/_build/libgwt_b200.so``. There is no CPU
fallback: importing without the library raises, and every call fails loudly
when no CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GWT_LIB_PATH") or os.path.join(HERE, "_build", "libgwt_b200.so")  # override: profiling builds

GWT_OK, GWT_INVALID_ARGUMENT, GWT_RUNTIME_ERROR, GWT_CUDA_ERROR, GWT_NO_DEVICE = range(5)
GWT_C64, GWT_C128 = 0, 1
GWT_MEM_HOST, GWT_MEM_DEVICE = 0, 1
GWT_SCOPE_FULL, GWT_SCOPE_PAPER = 0, 1
GWT_SOLVE_EARLY_STOP, GWT_SOLVE_POOLED, GWT_SOLVE_INIT = 1, 2, 4

# every symbol include/gwt_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "gwt_ctx_create", "gwt_ctx_destroy", "gwt_last_error", "gwt_ctx_set_stream", "gwt_ctx_launch_count",
    "gwt_ctx_stage_times", "gwt_groupwise_solve", "gwt_sinr_compressed", "gwt_sinr_compressed_coeffs",
    "gwt_assemble_compressed", "gwt_leading_eigenvectors", "gwt_reconstruct", "gwt_flop_estimate",
    "gwt_generate_channels", "gwt_mode_product", "gwt_sinr_full", "gwt_hpd_solve",
)


class Topology(C.Structure):
    """gwt_topology == gwt::SystemTopology (channel.hpp:13-27)."""
    _fields_ = [("num_cells", C.c_int32), ("users_per_cell", C.c_int32), ("rx_antennas", C.c_int32),
                ("tx_antennas", C.c_int32), ("num_taps", C.c_int32), ("num_streams", C.c_int32),
                ("noise_std", C.c_double)]


class Ranks(C.Structure):
    """gwt_ranks == gwt::CompressionRanks (decompose.hpp:18-24)."""
    _fields_ = [("m", C.c_int32), ("n", C.c_int32), ("p", C.c_int32)]


class Ledger(C.Structure):
    """gwt_ledger == gwt::FlopLedger (flops.hpp:10-31)."""
    _fields_ = [("reconstruct", C.c_int64), ("precoder", C.c_int64), ("covariance", C.c_int64),
                ("inverse", C.c_int64), ("filter", C.c_int64), ("sinr", C.c_int64)]

    def total(self):
        return self.reconstruct + self.precoder + self.covariance + self.inverse + self.filter + self.sinr


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"gwt B200 library not built: {LIB_PATH} missing (run `make` or __graft_entry__.build())")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, u32, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.POINTER(C.c_double)
    P_T, P_R, P_L = C.POINTER(Topology), C.POINTER(Ranks), C.POINTER(Ledger)
    sig = {
        "gwt_ctx_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
        "gwt_ctx_destroy": (None, [vp]),
        "gwt_last_error": (C.c_char_p, [vp]),
        "gwt_ctx_set_stream": (C.c_int, [vp, vp]),
        "gwt_ctx_launch_count": (i64, [vp]),
        "gwt_ctx_stage_times": (C.c_int, [vp, vp]),
        "gwt_groupwise_solve": (C.c_int, [vp, P_T, P_R, i64, C.c_int, C.c_int, vp, i32, u32, vp, vp, vp, vp, vp, vp,
                                          vp]),
        "gwt_sinr_compressed": (C.c_int, [vp, P_T, P_R, i64, C.c_int, C.c_int, vp, vp, vp, vp, i64, C.c_int, vp, vp,
                                          vp, P_L]),
        "gwt_sinr_compressed_coeffs": (C.c_int, [vp, P_T, P_R, i64, C.c_int, C.c_int, vp, vp, vp, i64, C.c_int, vp,
                                                 vp, vp, P_L]),
        "gwt_assemble_compressed": (C.c_int, [vp, P_T, P_R, i64, C.c_int, C.c_int, vp, vp, vp, vp, vp, i64, vp]),
        "gwt_leading_eigenvectors": (C.c_int, [vp, i32, i32, i64, C.c_int, C.c_int, vp, vp, vp]),
        "gwt_reconstruct": (C.c_int, [vp, P_T, P_R, i64, C.c_int, C.c_int, vp, vp, vp, vp, vp]),
        "gwt_flop_estimate": (C.c_int, [P_T, P_R, i32, P_L]),
        "gwt_sinr_full": (C.c_int, [vp, P_T, i64, C.c_int, C.c_int, vp, vp, vp, vp, i64, C.c_int, vp, vp, vp, P_L]),
        "gwt_mode_product": (C.c_int, [vp, C.c_int, C.c_int, i64, i32, i32, i32, vp, i32, vp, i32, vp]),
        "gwt_hpd_solve": (C.c_int, [vp, i32, i32, i64, C.c_int, vp, vp, i32, vp, vp]),
        "gwt_generate_channels": (C.c_int, [P_T, i64, i64, C.c_uint64, C.c_double, C.c_double, C.c_int, vp, vp,
                                            i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
