"""Multi-rank host logic of bench.py on CPU: world_size 2 over gloo (127.0.0.1).

The GPU path shards the C4 sequences round-robin (rank r owns j = r mod P) with no data-path
collective; the collectives gather per-rank device times / units (the job time is the max over
ranks) and per-sequence position checksums, whose combined digest must not depend on P
(SURVEY.md 8(e)).  This test runs that host logic in two processes."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_positions(j):
    """Stand-in for sequence j's final positions (depends on j only, like a real trajectory)."""
    return np.random.default_rng(500 + j).standard_normal((7, 3))


def _worker(rank, world, port, n_seq, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import scenes
    mine = scenes.c4_assignment(n_seq, rank, world)
    per_rank = [100.0 + 50.0 * rank, 7.0 * (rank + 1), float(len(mine) * 4)]   # rank 1 is slow
    allv = bench.gather_rank_values(per_rank, world, "cpu")
    v = bench.job_throughput(allv[:, 0], allv[:, 2])
    by_seq = bench.gather_checksums([(j, bench.seq_checksum(_fake_positions(j))) for j in mine], world, "cpu",
                                    n_seq)
    out.put((rank, mine, allv.tolist(), v, bench.combined_checksum(by_seq)))
    dist.destroy_process_group()


def test_two_rank_assignment_gather_throughput_checksums():
    import bench
    import scenes
    n_seq = 9
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_seq, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # round-robin j mod P: disjoint, covering, balanced to within one
    assert res[0][1] == [0, 2, 4, 6, 8] and res[1][1] == [1, 3, 5, 7]
    for rank, mine, allv, v, digest in res:
        assert allv == [[100.0, 7.0, 20.0], [150.0, 14.0, 16.0]]      # every rank sees every rank
        # 20 + 16 sequence-iterations in the slowest rank's 150 ms
        assert v == pytest.approx(36 / 0.150)
    # the combined checksum equals the single-process (P = 1) one and both ranks agree
    single = bench.combined_checksum({j: bench.seq_checksum(_fake_positions(j)) for j in range(n_seq)})
    assert res[0][4] == res[1][4] == single
    # and it detects a single changed trajectory
    bad = {j: bench.seq_checksum(_fake_positions(j)) for j in range(n_seq)}
    x = _fake_positions(3)
    x[0, 0] = np.nextafter(x[0, 0], 1.0)
    bad[3] = bench.seq_checksum(x)
    assert bench.combined_checksum(bad) != single
    assert scenes.c4_assignment(64, 3, 8) == list(range(3, 64, 8))
