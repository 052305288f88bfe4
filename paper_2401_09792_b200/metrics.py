"""Paper metrics R_s, e_c, R_t (reference proj/src/metrics.cpp:9-66).

Host-side scalar arithmetic over SINR reports; used for reporting, not a hot loop."""
from __future__ import annotations

import numpy as np

from .api import CompressionRanks, InvalidArgument, SystemTopology


def storage_counts(topo: SystemTopology, ranks: CompressionRanks, model: str = "groupwise"):
    """(original, compressed) complex-value counts (metrics.cpp:9-34)."""
    J, K, M, N, P = topo.num_cells, topo.users_per_cell, topo.rx_antennas, topo.tx_antennas, topo.num_taps
    m, n, p = ranks.m, ranks.n, ranks.p
    original = J * J * K * M * N * P
    per_link = m * n * p + P * p
    if model == "groupwise":
        comp = J * J * K * per_link + J * K * M * m + J * N * n
    elif model == "shared":
        comp = J * J * K * per_link + M * m + N * n
    elif model == "individual":
        comp = J * J * K * (per_link + M * m + N * n)
    else:
        raise InvalidArgument(f"unknown model '{model}' (expected individual, shared or groupwise)")
    return original, comp


def storage_ratio(topo, ranks, model="groupwise") -> float:
    o, c = storage_counts(topo, ranks, model)
    return o / c


def sinr_error(full, compressed) -> float:
    """Mean relative per-stream SINR error e_c (metrics.cpp:36-56); raises on a zero full-path SINR."""
    f = np.asarray(full, np.float64).reshape(-1)
    c = np.asarray(compressed, np.float64).reshape(-1)
    if f.shape != c.shape:
        raise InvalidArgument("sinr_error: reports cover different (user, stream) sets")
    z = np.flatnonzero(f == 0.0)
    if z.size:
        raise InvalidArgument(f"sinr_error: full-path SINR is zero at flat index {int(z[0])}; relative error undefined")
    return float(np.mean(np.abs(f - c) / np.abs(f)))


def speedup(t_full: float, t_compressed: float) -> float:
    """R_t = t_full / t_compressed (metrics.cpp:58-66)."""
    if not (t_full > 0.0) or not (t_compressed > 0.0):
        raise InvalidArgument("speedup: durations must be positive")
    return t_full / t_compressed
