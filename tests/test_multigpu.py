"""N>1 host logic on CPU (gloo, world_size 2): bench.py's own group partition
(bench.shard_plan), per-rank input generation and bench.py's end-of-run stats
reduction (bench.reduce_run_stats / whole_job_value), checked against a
single-process run of the same work."""
import os
import socket

import numpy as np
import pytest

from paper_2401_09792_b200.shard import group_range, reduce_stats


def test_group_range_partitions():
    for n in (0, 1, 4, 7, 64, 512):
        for w in (1, 2, 3, 4, 8):
            blocks = [group_range(r, w, n) for r in range(w)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(b[1] == c[0] for b, c in zip(blocks, blocks[1:]))
            sizes = [b[1] - b[0] for b in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        group_range(2, 2, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import bench
    import paper_2401_09792_b200 as gw
    from oracle import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = gw.CONFIGS["C1"]
    g0, g1 = bench.shard_plan(cfg, rank, world)
    X, tau = gw.generate_channels(cfg.topology(), g1 - g0, seed=0, group0=g0)
    d = bench.dims_of(cfg)
    fo = O.alternating_solve(d, X, 3, early_stop=False)
    co = O.coeffs_from_tau(tau, cfg.freqs()[:4])
    sinr, _ = O.sinr_compressed(d, fo["C"], fo["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER)
    stats = bench.reduce_run_stats({"nmse_num": fo["trace"][:, -1].sum(), "nmse_den": fo["energy"].sum(),
                                    "links": (g1 - g0) * cfg.G, "evals": (g1 - g0) * 4 * cfg.J * cfg.K,
                                    "bad_items": 0, "max_ms": 1.0 + rank, "max_tucker_ms": 10.0 * (rank + 1),
                                    "max_sinr_rel_err": 1e-12 * (rank + 1)})
    q.put((rank, dict(stats, whole=bench.whole_job_value(cfg, stats), block=(g0, g1), sinr=sinr)))
    dist.destroy_process_group()


def test_bench_shard_plan_covers_c4():
    import bench
    import paper_2401_09792_b200 as gw
    cfg = gw.CONFIGS["C4"]
    for w in (1, 2, 4, 8):
        blocks = [bench.shard_plan(cfg, r, w) for r in range(w)]
        assert [b[1] - b[0] for b in blocks] == [cfg.groups // w] * w
        assert blocks[0][0] == 0 and blocks[-1][1] == cfg.groups


def test_gloo_world2_sharded_equals_single():
    import torch.multiprocessing as mp

    import paper_2401_09792_b200 as gw
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = gw.CONFIGS["C1"]
    X, _ = gw.generate_channels(cfg.topology(), cfg.groups, seed=0)
    d = dict(J=cfg.J, K=cfg.K, M=cfg.M, N=cfg.N, P=cfg.P, m=cfg.m, n=cfg.n, p=cfg.p)
    fo = O.alternating_solve(d, X, 3, early_stop=False)
    co = O.coeffs_from_tau(_, cfg.freqs()[:4])
    sinr, _s = O.sinr_compressed(d, fo["C"], fo["G"], co, cfg.sigma, cfg.L, O.SCOPE_PAPER)
    assert res[0]["block"] == (0, 2) and res[1]["block"] == (2, 4)
    # the sharded per-group results are the single-process ones (groups are independent)
    assert np.array_equal(np.concatenate([res[0]["sinr"], res[1]["sinr"]]), sinr)
    for r in (0, 1):
        s = res[r]
        assert s["links"] == cfg.links
        assert s["evals"] == cfg.groups * 4 * cfg.J * cfg.K
        assert s["max_ms"] == 2.0 and s["max_tucker_ms"] == 20.0 and s["max_sinr_rel_err"] == 2e-12
        assert abs(s["nmse_num"] - fo["trace"][:, -1].sum()) <= 1e-9 * s["nmse_num"]
        assert abs(s["nmse_den"] - fo["energy"].sum()) <= 1e-12 * s["nmse_den"]
        w = s["whole"]
        assert w["value"] == s["evals"] / 2e-3 and w["tucker"] == cfg.links / 20e-3
