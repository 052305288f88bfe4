"""Rank sweep of the storage / error trade-off on the B200 path (reference run_sweep, proj/src/runner.cpp:193-211,
and run_experiment's scoring, runner.cpp:115-140; BASELINE configs[4] = C5: Tucker n in {16, 32, 64, 96},
p in {8, 16, 32}, 20 ALS sweeps each).

For every value along one axis ('n' or 'p', the other rank fixed) the groups are compressed on the device
(groupwise_solve, fixed sweeps), both SINR pipelines run on the device — the compressed path
(run_compressed_pipeline) and the full-size comparator on the uncompressed tensors (run_full_pipeline) —
and the row carries the reference's SweepRow fields: the storage ratio R_s (metrics.cpp:9-34), the
measured speedup R_t = t_full / t_compressed (metrics.cpp:58-66; median of `repetitions` device-timed runs
after one discarded warm-up, runner.cpp:123-134), and the mean per-stream SINR error e_c
(metrics.cpp:36-56); plus the NMSE of the fit and both SINR throughputs. The report writers (sweep.csv) are
control plane and out of scope; `sweep_csv_text` gives the same columns for callers that want them.
"""
from __future__ import annotations

import dataclasses
import statistics
import time

import numpy as np

from . import metrics
from .api import CompressionRanks, InvalidArgument


@dataclasses.dataclass
class SweepRow:
    """gwt::SweepRow (runner.hpp:24-29) plus the fit and throughput of the point."""
    value: int
    r_s: float
    r_t: float
    e_c: float
    nmse: float = 0.0
    t_full_ms: float = 0.0
    t_compressed_ms: float = 0.0
    tucker_ms: float = 0.0


def _timed(ctx, fn, repetitions):
    """One discarded warm-up, then the median of `repetitions` runs, each bracketed by device syncs."""
    import torch
    out = fn()
    ts = []
    for _ in range(max(1, repetitions)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return out, statistics.median(ts)


def run_sweep(ctx, topo, ranks: CompressionRanks, axis: str, values, X, tau, freqs, sweeps: int = 20,
              repetitions: int = 3, scope: str = "paper_experiment"):
    """Rows for `values` along `axis` ('n' or 'p'); X [g, links, P, N, M] (device tensors for the timing),
    tau [g, links, P], freqs [F]. Raises the reference's invalid_argument text for a bad axis."""
    if axis not in ("n", "p"):
        raise InvalidArgument("run_sweep: config has no sweep axis")
    import torch
    full, t_full = _timed(ctx, lambda: ctx.run_full_pipeline(topo, X, scope=scope, tau=tau, freqs=freqs), repetitions)
    f_sinr = full.sinr.cpu().numpy() if hasattr(full.sinr, "cpu") else np.asarray(full.sinr)
    rows = []
    for v in values:
        r = dataclasses.replace(ranks, **{axis: int(v)})
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fac = ctx.groupwise_solve(topo, X, r, sweeps, early_stop=False)
        torch.cuda.synchronize()
        t_tucker = (time.perf_counter() - t0) * 1e3
        rep, t_comp = _timed(ctx, lambda: ctx.run_compressed_pipeline(topo, fac, r, scope=scope, tau=tau,
                                                                       freqs=freqs), repetitions)
        c_sinr = rep.sinr.cpu().numpy() if hasattr(rep.sinr, "cpu") else np.asarray(rep.sinr)
        tr = fac.trace.cpu().numpy() if hasattr(fac.trace, "cpu") else np.asarray(fac.trace)
        en = fac.energy.cpu().numpy() if hasattr(fac.energy, "cpu") else np.asarray(fac.energy)
        rows.append(SweepRow(value=int(v), r_s=metrics.storage_ratio(topo, r), r_t=metrics.speedup(t_full, t_comp),
                             e_c=metrics.sinr_error(f_sinr, c_sinr), nmse=float(tr[:, -1].sum() / en.sum()),
                             t_full_ms=t_full, t_compressed_ms=t_comp, tucker_ms=t_tucker))
    return rows


def sweep_csv_text(rows) -> str:
    """sweep.csv as the reference writes it (runner.cpp:288-298): header `axis,Rs,Rt,ec`, then
    `%d,%.6f,%.6f,%.8f` per row."""
    return "axis,Rs,Rt,ec\n" + "".join(f"{r.value},{r.r_s:.6f},{r.r_t:.6f},{r.e_c:.8f}\n" for r in rows)
