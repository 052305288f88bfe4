"""BASELINE.json configurations C1..C5 under the SURVEY.md §8(d) mapping.

One BASELINE "group of G channels" = one independent reference ChannelSet with
J=2 cells and K=G/4 users per cell (J^2 K = G links, G/2 users), interference
scope paper_experiment. Nr, Nt, K(submatrices) map to M, N, P. Subcarrier s is
at f_s = s * 30 kHz; sigma = 10^(-SNR/20).
"""
from __future__ import annotations

from dataclasses import dataclass

# Dependency-free on purpose: bench.py's CPU reference arm loads this file by path so that it never
# imports the product package (the topology()/ranks() helpers import the API lazily).

SUBCARRIER_SPACING_HZ = 30e3
MAX_DELAY_S = 1e-6
PDP_DECAY = 0.3


@dataclass(frozen=True)
class BaselineConfig:
    name: str
    M: int
    N: int
    P: int
    G: int          # channels (links) per group
    groups: int
    F: int          # subcarriers
    m: int
    n: int
    p: int
    L: int
    snr_db: float
    dtype: str      # "c64" | "c128"
    sweeps: int = 20

    @property
    def J(self):
        return 2

    @property
    def K(self):
        return self.G // 4

    @property
    def sigma(self):
        return 10.0 ** (-self.snr_db / 20.0)

    def topology(self):
        from .api import SystemTopology
        return SystemTopology(self.J, self.K, self.M, self.N, self.P, self.L, self.sigma)

    def ranks(self):
        from .api import CompressionRanks
        return CompressionRanks(self.m, self.n, self.p)

    def freqs(self):
        import numpy as np
        return np.arange(self.F, dtype=np.float64) * SUBCARRIER_SPACING_HZ

    @property
    def users(self):
        return self.groups * self.J * self.K

    @property
    def links(self):
        return self.groups * self.G


CONFIGS = {
    "C1": BaselineConfig("C1", 4, 32, 24, 8, 4, 64, 4, 16, 8, 4, 10.0, "c128"),
    "C2": BaselineConfig("C2", 4, 64, 32, 16, 64, 272, 4, 24, 12, 4, 10.0, "c64"),
    "C2d": BaselineConfig("C2d", 4, 64, 32, 16, 64, 272, 4, 24, 12, 4, 10.0, "c128"),
    "C3": BaselineConfig("C3", 8, 128, 48, 32, 256, 1632, 8, 40, 16, 4, 15.0, "c64"),
    "C4": BaselineConfig("C4", 8, 256, 64, 64, 512, 3276, 8, 64, 24, 8, 10.0, "c64"),
    "C5": BaselineConfig("C5", 4, 128, 64, 32, 1024, 816, 4, 64, 16, 4, 10.0, "c64"),
}
