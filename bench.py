#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric) — one JSON line on rank 0.

Workload: BASELINE.json configs[1] (C2): Nr=4, Nt=64, K=32 submatrices, G=16
channels/group, 64 groups, 272 subcarriers, ranks (4,24,12), complex64, MMSE
SINR at 10 dB, 4 streams (J=2, K=G/4 mapping, paper_experiment scope;
DESIGN.md §2). A "step" is one pass of the compressed-form SINR stage
(rebuild + precoder + MMSE over all groups x subcarriers) — the headline
metric "SINR evals/sec" (one eval = one user x one subcarrier, all streams).
The Tucker stage (groupwise_solve, 20 fixed sweeps, all groups) is timed in
the same run and reported under "tucker" (Tucker channels/sec).

Multi-GPU (torchrun): weak scaling — each rank compresses and evaluates its
own C2-sized block of groups (group offset rank*64); no data-path collective;
one NCCL all_reduce of a small stats vector at the end; times are max over ranks.

--impl reference: times the reference algorithm's CPU implementation (the
oracle restatement — the reference itself needs Eigen, absent here) on this
host's cores for the same metric/config.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["hbm_gbs"], "measured", d
    except Exception:
        return 6650.0, "fallback", {}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region (NVML, ~2 ms period)."""

    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, device):
        self.device = device
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.mx.append(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.N = None
        return self

    def _run(self):
        N = self.N
        get_r = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons", None) or N.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop.is_set():
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = get_r(self.h)
                for b, name in self.BITS.items():
                    if r & b:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self.stop.set()
        if self.N is not None:
            self.t.join(timeout=1)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml"}


# ---------------------------------------------------------------------------
# algorithmic cost model

def sinr_costs(cfg, cs):
    """Per-kernel algorithmic (flops, flop pipe, bytes) for one SINR step over the whole batch."""
    J, m, n, p, P, L = cfg.J, cfg.m, cfg.n, cfg.p, cfg.P, cfg.L
    links, users, F, g = cfg.G, cfg.G // 2, cfg.F, cfg.groups
    S = J
    wp = "fp32" if cs == 8 else "fp64"
    rebuild = (8 * (m * n * p + P * p) * links * F * g, wp,
               (cs * m * n * links * F + cs * (m * n * p + P * p) * links + 8 * P * links) * g)
    pair_gram = (8 * S * m * m * n * users * F * g, "fp64",
                 (cs * m * n * (2 * J - 1) * users * F + 16 * S * m * m * users * F) * g)
    # eig (cyclic Jacobi, ~6 sweeps) + covariance/Cholesky/solves, estimated fp64 flops per (user, subcarrier)
    jac = 6 * (m * (m - 1) // 2) * 48 * m
    mmse = 8 * (L * m * m + (S - 1) * 2 * m ** 3 + m ** 3 // 3 + L * m * m // 2)
    Lp = (L + 1) // 2 * 2
    small = ((jac + mmse) * users * F * g, "fp64",
             (16 * S * m * m + 8 * (Lp + 2 * m * L) * (1 + (S - 1)) + 16 * L + 4) * users * F * g)
    return dict(rebuild=rebuild, pair_gram=pair_gram, small=small)


def binding_roofline(flops, pipe, nbytes, ms, hbm, peaks_t):
    """t_roof = max(bytes/BW, flops/peak); report the binding resource's achieved rate vs its peak."""
    t = ms * 1e-3
    t_b = nbytes / (hbm * 1e9)
    t_f = flops / (peaks_t[pipe] * 1e12) if flops else 0.0
    if t_b >= t_f:
        ach = nbytes / t / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm}
    ach = flops / t / 1e12
    return {"bound": pipe, "achieved": ach, "peak": peaks_t[pipe], "unit": "TFLOP/s", "frac": ach / peaks_t[pipe]}


def cublas_peaks(dev):
    """Measured FP32 (SGEMM, TF32 off) and FP64 (DGEMM) cuBLAS throughput on this GPU, best of a few
    square GEMMs timed with CUDA events: the achievable CUDA-core ceilings SURVEY.md §8(d) asks for
    beside the derived 148 SM x clock peaks (cuBLAS is a measuring tool here, not on the hot path)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    out = {}
    for name, dt, n, reps in (("sgemm_tflops", torch.float32, 8192, 5), ("dgemm_tflops", torch.float64, 4096, 3)):
        a = torch.randn(n, n, dtype=dt, device=dev)
        b = torch.randn(n, n, dtype=dt, device=dev)
        torch.matmul(a, b)
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = 2.0 * n ** 3 / (best * 1e-3) / 1e12
        del a, b
    torch.backends.cuda.matmul.allow_tf32 = prev
    return out


def tucker_flops(cfg):
    """Canonical-order flops of one groupwise_solve (init + S sweeps) per SURVEY.md §8(d)."""
    M, N, P, m, n, p, S = cfg.M, cfg.N, cfg.P, cfg.m, cfg.n, cfg.p, cfg.sweeps
    init = M * M * N * P + N * N * M * P + P * P * M * N
    rx = min(M * N * P * n + M * n * P * p, M * N * P * p + M * N * p * n) + M * M * n * p
    tx = min(m * M * N * P + m * N * P * p, M * N * P * p + m * M * N * p) + N * N * m * p
    de = min(m * M * N * P + m * n * N * P, M * N * P * n + m * M * n * P) + P * P * m * n
    obj = m * n * P * p
    return 8 * (init + S * (rx + tx + de + obj)) * cfg.links


# ---------------------------------------------------------------------------

def run_reference(args, cfg):
    import paper_2401_09792_b200 as gw
    from oracle import oracle as O
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    topo = cfg.topology()
    dims = dict(J=cfg.J, K=cfg.K, M=cfg.M, N=cfg.N, P=cfg.P, m=cfg.m, n=cfg.n, p=cfg.p)
    # bounded sample of the same workload: 2*cores groups x 64 subcarriers per step
    gs = min(cfg.groups, 2 * cores)
    fs = min(cfg.F, 64)
    X, tau = gw.generate_channels(topo, gs, seed=0, dtype=np.complex128)
    if cfg.dtype == "c64":
        X = X.astype(np.complex64).astype(np.complex128)
    fo = O.alternating_solve(dims, X, 2, early_stop=False, nthreads=cores)
    co = O.coeffs_from_tau(tau, cfg.freqs()[:fs])
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        O.sinr_compressed(dims, fo["C"], fo["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=cores)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
    evals = gs * fs * cfg.J * cfg.K
    v = evals / statistics.median(times)
    t0 = time.perf_counter()
    O.alternating_solve(dims, X[: min(gs, cores)], cfg.sweeps, early_stop=False, nthreads=cores)
    tuck = min(gs, cores) * cfg.G / (time.perf_counter() - t0)
    line = {
        "impl": "reference", "metric": "SINR evals/sec", "value": v, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64)",
        "data": "synthetic (BASELINE.json generator, seed 0)",
        "config": {"workload": cfg.name, "groups": cfg.groups, "subcarriers": cfg.F, "ranks": [cfg.m, cfg.n, cfg.p],
                   "streams": cfg.L, "snr_db": cfg.snr_db, "scope": "paper_experiment"},
        "cpu_baseline": {"value": v, "unit": "evals/s", "cores": cores, "kind": "port",
                         "sample": f"{gs} groups x {fs} subcarriers per step (of {cfg.groups} x {cfg.F}); "
                                   "oracle C++ restatement, one group per std::thread"},
        "e2e": {"value": v, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "tucker": {"value": tuck, "unit": "channels/s", "sample": f"{min(gs, cores)} groups x {cfg.sweeps} sweeps"},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_leg(cfg, cores):
    """Oracle (port) on the host, bounded sample ~10 s; rank 0 at N=1 only."""
    import paper_2401_09792_b200 as gw
    from oracle import oracle as O
    dims = dict(J=cfg.J, K=cfg.K, M=cfg.M, N=cfg.N, P=cfg.P, m=cfg.m, n=cfg.n, p=cfg.p)
    gs = min(cfg.groups, 2 * cores)
    fs = min(cfg.F, 64)
    X, tau = gw.generate_channels(cfg.topology(), gs, seed=0, dtype=np.complex128)
    if cfg.dtype == "c64":
        X = X.astype(np.complex64).astype(np.complex128)
    t0 = time.perf_counter()
    fo = O.alternating_solve(dims, X, cfg.sweeps, early_stop=False, nthreads=cores)
    t_tuck = time.perf_counter() - t0
    co = O.coeffs_from_tau(tau, cfg.freqs()[:fs])
    t0 = time.perf_counter()
    O.sinr_compressed(dims, fo["C"], fo["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER, nthreads=cores)
    t_s = time.perf_counter() - t0
    return {"value": gs * fs * cfg.J * cfg.K / t_s, "unit": "evals/s", "cores": cores, "kind": "port",
            "sample": f"SINR: {gs} groups x {fs} subcarriers; Tucker: {gs} groups x {cfg.sweeps} sweeps "
                      f"(oracle C++ restatement in fp64, one group per std::thread)",
            "tucker_channels_per_s": gs * cfg.G / t_tuck}


def main():
    args = parse()
    import paper_2401_09792_b200 as gw
    cfg = gw.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    ctx = gw.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.use_torch_stream()
    topo, ranks = cfg.topology(), cfg.ranks()
    npdt = np.complex64 if cfg.dtype == "c64" else np.complex128
    cs = 8 if cfg.dtype == "c64" else 16

    # inputs: this rank's block of groups, resident in HBM
    Xh, tau_h = gw.generate_channels(topo, cfg.groups, seed=0, dtype=np.complex128, group0=rank * cfg.groups)
    Xh = Xh.astype(npdt)
    X = torch.from_numpy(Xh).to(dev)
    tau = torch.from_numpy(tau_h).to(dev)
    freqs = torch.from_numpy(cfg.freqs()).to(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---------------- Tucker stage (device-resident), fixed 20 sweeps
    fac = None
    for _ in range(max(1, args.warmup // 2)):
        fac = ctx.groupwise_solve(topo, X, ranks, cfg.sweeps, early_stop=False)
    barrier()
    tt = []
    tucker_steps = max(2, min(args.steps, 5))
    for _ in range(tucker_steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fac = ctx.groupwise_solve(topo, X, ranks, cfg.sweeps, early_stop=False)
        e1.record(stream)
        e1.synchronize()
        tt.append(e0.elapsed_time(e1))
    tucker_stage = ctx.stage_ms()
    # reference stop rule (decompose.cpp:363-368: stop once decrease < 1e-10 * energy), timed the same way
    es_ms, es_iters = [], None
    for it in range(4):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fes = ctx.groupwise_solve(topo, X, ranks, cfg.sweeps, early_stop=True)
        e1.record(stream)
        e1.synchronize()
        if it > 0:
            es_ms.append(e0.elapsed_time(e1))
        if os.environ.get("GWT_BENCH_DEBUG"):
            print("early-stop solve ms", e0.elapsed_time(e1), ctx.stage_ms()[:3], file=sys.stderr)
        it_ = fes.iterations_run
        es_iters = np.asarray(it_.cpu() if hasattr(it_, "cpu") else it_)
    barrier()

    # ---------------- SINR stage (the step), device-resident inputs
    for _ in range(args.warmup):
        rep = ctx.run_compressed_pipeline(topo, fac, ranks, tau=tau, freqs=freqs)
    barrier()
    launches0 = ctx.launches
    step_ms, st_acc = [], np.zeros(8)
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            rep = ctx.run_compressed_pipeline(topo, fac, ranks, tau=tau, freqs=freqs)
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            st_acc += np.array(rep.stage_ms)
        barrier()
        t_wall = time.perf_counter() - t_wall
    launches = ctx.launches - launches0
    ms = float(np.mean(step_ms))
    st_acc /= args.steps
    # The headline loop runs the groups on 2 overlapping stream lanes, so per-kernel durations there
    # include inter-lane contention; the roofline is taken from a single-lane timed loop (same inputs,
    # L2 flushed) whose per-stage kernel times sum to its step time.
    prev = os.environ.get("GWT_SINR_DEV_LANES")
    os.environ["GWT_SINR_DEV_LANES"] = "1"
    st_acc = np.zeros(8)
    rl_steps = max(10, min(args.steps, 50))
    rl_ms = []
    for _ in range(3):  # warm: the single-lane call sizes lane 0's workspaces for all groups
        ctx.run_compressed_pipeline(topo, fac, ranks, tau=tau, freqs=freqs)
    torch.cuda.synchronize()
    for _ in range(rl_steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rep1 = ctx.run_compressed_pipeline(topo, fac, ranks, tau=tau, freqs=freqs)
        e1.record(stream)
        e1.synchronize()
        rl_ms.append(e0.elapsed_time(e1))
        st_acc += np.array(rep1.stage_ms)
    st_acc /= rl_steps
    if prev is None:
        del os.environ["GWT_SINR_DEV_LANES"]
    else:
        os.environ["GWT_SINR_DEV_LANES"] = prev
    tk = float(np.mean(tt))
    stats = torch.tensor([ms, tk, float(rep.status.ne(0).sum())], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)  # only collective: max-over-ranks times + status
    ms, tk, bad = stats.tolist()
    evals = cfg.groups * cfg.F * cfg.J * cfg.K * world
    value = evals / (ms * 1e-3)

    # ---------------- paper metrics on this workload: full-size SINR on the raw
    # channels (same kernels, cores = X, delay = I) vs the compressed step; R_t, e_c, R_s
    from paper_2401_09792_b200 import metrics as pm
    for _ in range(2):
        full = ctx.run_full_pipeline(topo, X, tau=tau, freqs=freqs)
    fms = []
    for _ in range(max(3, min(args.steps, 10))):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        full = ctx.run_full_pipeline(topo, X, tau=tau, freqs=freqs)
        e1.record(stream)
        e1.synchronize()
        fms.append(e0.elapsed_time(e1))
    paper = {"R_t_gpu": float(np.mean(fms)) / ms, "t_full_ms": float(np.mean(fms)), "t_compressed_ms": ms,
             "e_c": pm.sinr_error(full.sinr.cpu().numpy(), rep.sinr.cpu().numpy()),
             "R_s": pm.storage_ratio(topo, ranks),
             "note": "paper Table 2 (groupwise, 3GPP J=21) reports R_t 6.19 / R_s 6.16 / e_c 9.4% on other data"}

    # ---------------- e2e through the public API with pinned host buffers
    Ch = rep_in = None
    Ch = fac.delay.cpu().pin_memory()
    Gh = fac.cores.cpu().pin_memory()
    tauh = torch.from_numpy(tau_h).pin_memory()
    fh = torch.from_numpy(cfg.freqs()).pin_memory()
    ctx_h = gw.Context(local)
    e2e_ms = []
    for it in range(max(args.warmup, 1) + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fh_fac = gw.GroupwiseFactorSet(None, None, Ch, Gh)
        rep_h = ctx_h.run_compressed_pipeline(topo, fh_fac, ranks, tau=tauh, freqs=fh)
        t1 = time.perf_counter()
        if it >= max(args.warmup, 1):
            e2e_ms.append((t1 - t0) * 1e3)
    if os.environ.get("GWT_BENCH_DEBUG"):
        print("e2e_ms", [round(x, 3) for x in e2e_ms], file=sys.stderr)
    e2e_t = torch.tensor([float(np.mean(e2e_ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    h2d = Ch.numel() * cs + Gh.numel() * cs + tauh.numel() * 8 + fh.numel() * 8
    d2h = rep_h.sinr.numel() * 8 * 2 + rep_h.status.numel() * 4
    # Tucker e2e: host X in, factors out
    Xpin = torch.from_numpy(Xh).pin_memory()
    fac_h = ctx_h.groupwise_solve(topo, Xpin, ranks, cfg.sweeps, early_stop=False)  # warm (workspaces, pinned outs)
    t0 = time.perf_counter()
    for _ in range(2):
        fac_h = ctx_h.groupwise_solve(topo, Xpin, ranks, cfg.sweeps, early_stop=False)
    tuck_e2e_ms = (time.perf_counter() - t0) * 1e3 / 2
    ctx_h.close()

    # ---------------- roofline of the dominant SINR kernel (binding resource), all stages listed
    hbm, peak_kind, pk = peaks()
    clk_max = pk.get("sm_max_mhz", 1965.0)
    cublas = cublas_peaks(dev)
    peaks_t = {"fp32": 148 * 128 * 2 * clk_max * 1e6 / 1e12, "fp64": 148 * 64 * 2 * clk_max * 1e6 / 1e12}
    costs = sinr_costs(cfg, cs)
    stage = {"rebuild": st_acc[4], "pair_gram": st_acc[5], "small": st_acc[6]}
    kern = {"rebuild": "k_rebuild_rb", "pair_gram": "k_pair_gram_gf", "small": "k_small_fused"}
    per_stage = {}
    for k_, ms_k in stage.items():
        fl, pipe, by = costs[k_]
        r = binding_roofline(fl, pipe, by, ms_k, hbm, peaks_t)
        r.update(kernel=kern[k_], ms=round(ms_k, 4), alg_bytes=int(by), alg_flops=int(fl))
        if r["bound"] in ("fp32", "fp64"):  # same achieved rate against the cuBLAS ceiling measured in this run
            r["frac_vs_cublas"] = r["achieved"] / cublas["sgemm_tflops" if r["bound"] == "fp32" else "dgemm_tflops"]
        per_stage[k_] = r
    dom = max(stage, key=stage.get)
    roof = dict(per_stage[dom])
    # measured DRAM traffic per launch of the dominant kernel from the committed ncu capture (same config)
    traffic = None
    try:
        tj = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01_traffic.json")))
        if tj.get("config") == args.config:
            traffic = tj["bytes_per_launch"].get(kern[dom])
    except (OSError, ValueError, KeyError):
        traffic = None
    roof.update(traffic=traffic, traffic_source="profiles/r01_traffic.json" if traffic else None, peak_source={"hbm": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                                           "fp32": "derived: 148 SM x 128 FMA/clk x 2 x max clock (not measured)",
                                           "fp64": "derived: 148 SM x 64 DFMA/clk x 2 x max clock (not measured)"}[roof["bound"]],
                stage_share={k_: round(v / max(sum(stage.values()), 1e-9), 3) for k_, v in stage.items()},
                timing="per-stage CUDA events of a single-lane timed loop (ms_per_step_single_lane); the headline "
                       "value overlaps 2 group lanes",
                ms_per_step_single_lane=round(float(np.mean(rl_ms)), 4),
                stages=per_stage)
    tfl = tucker_flops(cfg) * world
    fp32_peak = peaks_t["fp32" if cs == 8 else "fp64"]
    tucker = {"value": cfg.links * world / (tk * 1e-3), "unit": "channels/s", "ms_per_solve": tk,
              "sweeps": cfg.sweeps, "mode": "fixed sweeps (no early stop)",
              "algorithmic_tflops": tfl / (tk * 1e-3) / 1e12,
              "roofline": {"bound": "fp32-cuda-core", "achieved": tfl / (tk * 1e-3) / 1e12, "peak": fp32_peak,
                           "unit": "TFLOP/s", "frac": tfl / (tk * 1e-3) / 1e12 / fp32_peak,
                           "frac_vs_cublas": tfl / (tk * 1e-3) / 1e12 / cublas["sgemm_tflops" if cs == 8 else "dgemm_tflops"],
                           "peak_source": "derived 148 SMs x 128 FFMA x 2 x max clock (not measured)"},
              "stage_ms": {"init_obj": tucker_stage[1], "sweeps": tucker_stage[2]},
              "early_stop": {"mode": "reference stop rule (decrease < 1e-10 * energy)",
                             "ms_per_solve": float(np.mean(es_ms)),
                             "value": cfg.links * world / (float(np.mean(es_ms)) * 1e-3),
                             "iterations_mean": float(es_iters.mean()), "iterations_max": int(es_iters.max())},
              "e2e_ms": tuck_e2e_ms, "e2e_h2d_bytes": Xh.nbytes,
              "e2e_d2h_bytes": sum(int(np.prod(a.shape)) * cs for a in (fac_h.rx, fac_h.tx, fac_h.delay, fac_h.cores))}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_leg(cfg, os.cpu_count() or 1)
    if rank == 0:
        line = {
            "metric": "SINR evals/sec", "value": value, "unit": "evals/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "c64 (fp32 rebuild/products; fp64 Grams and m x m solves)",
            "data": "synthetic (BASELINE.json generator: 1 ray/tap ULA, exp PDP 0.3, tau U(0,1us), seed 0)",
            "config": {"workload": cfg.name, "groups_per_gpu": cfg.groups, "subcarriers": cfg.F,
                       "dims": [cfg.M, cfg.N, cfg.P], "ranks": [cfg.m, cfg.n, cfg.p], "streams": cfg.L,
                       "snr_db": cfg.snr_db, "scope": "paper_experiment", "J": cfg.J, "K": cfg.K,
                       "parallelism": f"group-sharded x{world}", "l2": "flushed (256 MB write) between steps"},
            "e2e": {"value": evals / (e2e_t.item() * 1e-3), "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches),
            "roofline": roof,
            "cpu_baseline": cpu,
            "tucker": tucker,
            "paper_metrics": paper,
            "clocks": clk.summary(),
            "cublas_peaks": cublas,
            "status_nonzero": int(bad),
            "wall_s_timed": t_wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
