"""Multi-rank host logic of bench.py on CPU: world_size 2 over gloo (127.0.0.1).

The GPU path shards independent actuation sequences across ranks with no data-path collective;
the only collective gathers per-rank device times, and the job time is the max over ranks
(DESIGN.md 7).  This test runs that gather and the throughput arithmetic in two processes."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    per_rank_ms = [100.0 + 50.0 * rank, 7.0 * (rank + 1)]      # rank 1 is the slow one
    allv = bench.gather_rank_values(per_rank_ms, world, "cpu")
    v = bench.job_throughput(allv[:, 0], world, steps=4)
    out.put((rank, allv.tolist(), v))
    dist.destroy_process_group()


def test_two_rank_gather_and_throughput():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, allv, v in res:
        assert allv == [[100.0, 7.0], [150.0, 14.0]]          # every rank sees every rank
        # 2 ranks x 4 frames x 20 iterations in the slowest rank's 150 ms
        assert v == pytest.approx(2 * 4 * 20 / 0.150)
