"""The N > 1 path of bench.py on CPU: world_size-2 gloo process group,
weak-scaling shard assignment and the max-over-ranks timing reduction."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    mine = bench.shard(25, rank, world)
    t = 1.0 + rank * 0.5           # pretend per-rank device seconds
    tmax = bench.reduce_max(t)
    bench.barrier()
    out.put((rank, mine, tmax, bench.dist_env()))
    dist.destroy_process_group()


def test_gloo_world2_shards_and_max_reduce():
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
    (r0, s0, m0, e0), (r1, s1, m1, e1) = res
    assert s0 + s1 == list(range(25)) and not set(s0) & set(s1)
    assert m0 == m1 == 1.5
    assert e0 == (0, 0, 2) and e1 == (1, 1, 2)


@pytest.mark.parametrize("n,world", [(25, 1), (25, 2), (25, 8), (3, 8), (1000, 7)])
def test_shard_partitions(n, world):
    import sys
    sys.path.insert(0, ROOT)
    import bench
    parts = [bench.shard(n, r, world) for r in range(world)]
    flat = [i for p in parts for i in p]
    assert flat == list(range(n))
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
