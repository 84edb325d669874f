"""N>1 path on CPU: world_size-2 gloo process group (the GPU bench runs the
same code over NCCL).  Requests are data-parallel replicas — one request per
rank, no data-path collective — so the only exchange is the end-of-run
aggregation: total tokens and the slowest rank's time."""

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import bench

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = bench.aggregate_ranks(100 + rank, 10.0 * (rank + 1), 0.5 + rank, world, "cpu")
        P = bench.prompts(2, 1000, 16, rank)
        out.put((rank, res, P))
    finally:
        dist.destroy_process_group()


def test_two_rank_aggregation_and_replica_prompts():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict()
    for _ in procs:
        rank, res, P = q.get(timeout=120)
        got[rank] = (res, P)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in (0, 1):
        tokens, ms, e2e = got[r][0]
        assert tokens == 201.0          # 100 + 101 tokens over both replicas
        assert ms == 20.0               # slowest rank's device time
        assert e2e == 1.5
    assert got[0][1] != got[1][1]       # each replica decodes its own synthetic request


def test_single_rank_aggregation_is_identity():
    import bench

    assert bench.aggregate_ranks(7, 3.0, 0.25, 1, "cpu") == (7.0, 3.0, 0.25)
