"""Shared test helpers: seeded BASELINE inputs, layout conversions, error metrics."""
import numpy as np

import paper_2401_09792_b200 as gw
from oracle import oracle as O


def dims_of(cfg_or_topo, ranks=None):
    if isinstance(cfg_or_topo, gw.BaselineConfig):
        t, r = cfg_or_topo.topology(), cfg_or_topo.ranks()
    else:
        t, r = cfg_or_topo, ranks
    return dict(J=t.num_cells, K=t.users_per_cell, M=t.rx_antennas, N=t.tx_antennas, P=t.num_taps,
                m=r.m, n=r.n, p=r.p)


def baseline_inputs(cfg, ngroups=None, seed=0):
    """X in the config's dtype plus the complex128 upcast the oracle sees (identical values)."""
    g = cfg.groups if ngroups is None else ngroups
    X, tau = gw.generate_channels(cfg.topology(), g, seed=seed, dtype=np.complex128)
    if cfg.dtype == "c64":
        X = X.astype(np.complex64)
    return X, X.astype(np.complex128), tau


def rel_err(a, b, floor=0.0):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.abs(b), floor)


def to_np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


serving_singular_values = O.serving_singular_values
sinr_cluster_err = O.sinr_cluster_err
