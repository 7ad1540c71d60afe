"""Multi-process path of bench.py (replicas) on CPU with gloo, world size 2."""
import os
import socket
import sys

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r timed (10 + r) ms and processed 100 * (r + 1) decisions
        mx, sm = bench.reduce_max_sum([10.0 + rank], [100.0 * (rank + 1)])
        r2, w2, l2 = bench.dist_env()
        q.put((rank, mx, sm, r2, w2))
    finally:
        dist.destroy_process_group()


def test_replica_reduction_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, mx, sm, r2, w2 in res:
        assert mx == [11.0]          # max over ranks of the device time
        assert sm == [300.0]         # whole-job work = sum over ranks
        assert r2 == rank and w2 == 2


def test_reference_arm_other_ranks_exit_without_work(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench.main(["--impl", "reference", "--steps", "1", "--warmup", "3"]) == 0
    assert capsys.readouterr().out == ""


def test_bytes_per_decision():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.b_dec(16) == 260 and bench.b_dec(20) == 324
