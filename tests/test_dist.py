"""N>1 host logic of bench.py on CPU: world-size-2 gloo process group.

The conv path shards as independent replicas: each rank runs
its own stack with its own seed, the job time is the max over ranks and the
value aggregates all ranks' layers. No data-path collective exists to test.
"""

import os
import socket
import sys
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t_max = bench.world_max(10.0 + 5.0 * rank, world, "cpu")  # rank 1 is the slow one
    value = bench.job_value(20, 4, t_max, world)
    dist.barrier()
    q.put((rank, t_max, value))
    dist.destroy_process_group()


def test_world2_max_over_ranks_and_job_value():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t_max, value in out:
        assert t_max == 15.0  # every rank sees the slowest rank's time
        assert value == pytest.approx(2 * 20 * 4 / 15e-3)  # both replicas' layers over that time


def test_world1_is_identity():
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.world_max(3.5, 1, "cpu") == 3.5
    assert bench.job_value(20, 2, 4.0, 1) == pytest.approx(10000.0)
