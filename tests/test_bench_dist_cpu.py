"""bench.py's multi-rank plumbing on CPU (world_size 2, gloo): the timed value is
the max over ranks, and the data-parallel split covers every sequence once
(BASELINE configs[4] "MLGRU scan batch-split")."""
import os
import socket
import sys

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, bench.max_over_ranks(10.0 + rank * 5.0, world, "cpu")))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: 15.0, 1: 15.0}


def test_split_sequences_covers_batch():
    sys.path.insert(0, ROOT)
    import bench
    for B, world in [(32, 8), (8, 3), (5, 8), (16, 1)]:
        seen = []
        for r in range(world):
            f, n = bench.split_sequences(B, world, r)
            seen += list(range(f, f + n))
        assert seen == list(range(B))
