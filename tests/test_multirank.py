"""bench.py's multi-rank host logic (replicas only) on the CPU with gloo,
world size 2: the timed region is the max over ranks and the value aggregates all ranks."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local_ms = 100.0 + 50.0 * rank           # rank 1 is the slow one
    ms = bench.max_over_ranks(local_ms)
    value = bench.job_throughput(1e6, 4, world, ms)
    out[rank] = (ms, value, bench.dist_env())
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_job_throughput_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        ms, value, env = res[rank]
        assert ms == 150.0                             # max over ranks, identical everywhere
        assert value == pytest.approx(1e6 * 4 * world / 0.150)
        assert env == (world, rank, 0)                 # WORLD_SIZE / RANK read from the env


def test_single_process_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(12.5) == 12.5
    assert bench.job_throughput(10.0, 2, 1, 1000.0) == 20.0
