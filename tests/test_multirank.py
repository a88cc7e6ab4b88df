"""Multi-rank host logic of the replicas mode on CPU (gloo, world_size 2):
per-rank instances differ, the job time is the max over ranks, and the
whole-job throughput counts every rank's units."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2105_11788_b200 import workloads as W
    inst = W.lifted_quotient(2000, 100, 8, 3, 2, 2, seed=rank)
    local_ms = 10.0 * (rank + 1)
    ms = bench.reduce_max(local_ms)
    value = bench.job_throughput(inst.n + inst.m, 3, world, ms)
    out[rank] = (ms, value, int(inst.src[:50].sum()))
    dist.destroy_process_group()


def test_replicas_aggregation_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    (ms0, v0, h0), (ms1, v1, h1) = out[0], out[1]
    assert ms0 == ms1 == 20.0                  # max over ranks
    assert v0 == v1 == pytest.approx((2000 + 2000 * 4) * 3 * 2 / 0.020)
    assert h0 != h1                            # each rank refines its own instance


def test_single_process_reduce_is_identity():
    import bench
    assert bench.reduce_max(3.5) == 3.5
    assert bench.job_throughput(10, 2, 1, 1000.0) == 20.0
