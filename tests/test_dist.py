"""Multi-rank host logic of bench.py (replicas only: barrier + max-over-ranks timing) with the gloo
backend, world size 2, on CPU."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    r, w, lr = bench.dist_env()
    dist.init_process_group("gloo", rank=r, world_size=w)
    dist.barrier()
    ms = 10.0 + 5.0 * rank                          # rank 1 is the slow one
    m = bench.reduce_max(ms, w, "cpu")
    rate = bench.aggregate_rate(w, 8192 * 8192, 100, m)
    dist.barrier()
    dist.destroy_process_group()
    out.put((r, w, lr, m, rate))


def test_two_rank_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[:3] for r in res] == [(0, 2, 0), (1, 2, 1)]
    assert res[0][3] == res[1][3] == 15.0            # every rank sees the slowest rank's time
    assert res[0][4] == pytest.approx(2 * 8192 * 8192 * 100 / 0.015)


def test_single_rank_identity():
    import bench
    assert bench.reduce_max(3.0, 1) == 3.0
    assert bench.aggregate_rate(1, 100, 10, 1000.0) == 1000.0
