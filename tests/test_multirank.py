"""The bench's N>1 path (independent replicas, max-over-ranks device time,
summed work) on CPU with gloo, world_size 2."""
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    ms, n = bench.reduce_over_ranks(10.0 * (rank + 1), 100 + rank, dist, "cpu")
    out[rank] = (ms, n)
    dist.destroy_process_group()


def test_reduce_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    man = ctx.Manager()
    out = man.dict()
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, start_method="spawn", join=True)
    assert out[0] == (20.0, 201.0) and out[1] == (20.0, 201.0)
