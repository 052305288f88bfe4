"""Group sharding across ranks: independent channel groups,
contiguous blocks per rank, no data-path collective. The only collective is
one all_reduce of a small statistics vector at the end (NCCL over NVLink on
GPUs, gloo in the CPU tests)."""
from __future__ import annotations


def group_range(rank: int, world: int, ngroups: int) -> tuple[int, int]:
    """Contiguous block [g0, g1) of `ngroups` for `rank` of `world` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world) or ngroups < 0:
        raise ValueError("group_range: invalid rank/world/ngroups")
    base, extra = divmod(ngroups, world)
    g0 = rank * base + min(rank, extra)
    return g0, g0 + base + (1 if rank < extra else 0)


SUM_KEYS = ("nmse_num", "nmse_den", "evals", "links", "bad_items")
MAX_KEYS = ("max_sinr_rel_err", "max_ms", "max_tucker_ms")


def reduce_stats(stats: dict, device=None) -> dict:
    """All-reduce a stats dict across the default process group: sums for SUM_KEYS, maxima for MAX_KEYS."""
    import torch
    import torch.distributed as dist
    s = torch.tensor([float(stats.get(k, 0.0)) for k in SUM_KEYS], dtype=torch.float64, device=device)
    m = torch.tensor([float(stats.get(k, 0.0)) for k in MAX_KEYS], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(s, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    out = {k: v for k, v in zip(SUM_KEYS, s.tolist())}
    out.update({k: v for k, v in zip(MAX_KEYS, m.tolist())})
    return out
