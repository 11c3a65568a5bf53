"""The N > 1 path of bench.py on CPU: world_size-2 gloo process group, the
shared FIFO of batch claims (dynamic placement of the 256-image pool over
the ranks), and the max/sum-over-ranks reductions of the timing."""

import os
import socket

import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import random
    import sys
    import time
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    claims = bench.Claims(True)
    bench.barrier()
    mine = []
    rng = random.Random(rank)
    for _ in range(10):                 # rank 1 is slower: it should claim later ids
        mine.append(claims.next())
        time.sleep(rng.random() * 0.002 * (1 + 3 * rank))
    t = 1.0 + rank * 0.5                # pretend per-rank device seconds
    tmax = bench.reduce_max(t)
    tsum = bench.reduce_sum(len(mine))
    bench.barrier()
    out.put((rank, mine, tmax, tsum, bench.dist_env()))
    dist.destroy_process_group()


def test_gloo_world2_dynamic_claims_and_reductions():
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
    (r0, c0, m0, s0, e0), (r1, c1, m1, s1, e1) = res
    # every claim distinct, together exactly the FIFO prefix 0..19
    assert sorted(c0 + c1) == list(range(20))
    assert c0 == sorted(c0) and c1 == sorted(c1)          # each rank's claims in FIFO order
    assert m0 == m1 == 1.5 and s0 == s1 == 20
    assert e0 == (0, 0, 2) and e1 == (1, 1, 2)


def test_local_claims_and_batches():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    c = bench.Claims(False)
    assert [c.next() for _ in range(5)] == [0, 1, 2, 3, 4]
    cfg = bench.CONFIGS["c5"]
    assert bench.POOL_IMAGES // cfg["images"] == 8       # 256 images in batches of 32
