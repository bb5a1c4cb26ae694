"""Sequence-parallel MLGRU scan, host side (gloo, CPU; reading C23; tern.h block_prefill_sp).

Each process takes its contiguous token slice (paper_2406_02528_b200.shard.seq_slice),
forms its slice aggregate (A = prod f, B = the recurrence from 0, left to right) with the
ORACLE's scan, all-gathers the aggregates over gloo exactly where the library calls its
all-gather callback, composes the earlier ranks' aggregates in rank order into its
boundary state, scans its slice sequentially from it and composes through every slice for
the final state.  The gathered result must equal the oracle's W-slice scan
(O.scan_slices / O.scan_seqpar) bit for bit on every rank: the partition, the exchange and
the composition order are what the GPU path runs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2406_02528_b200 import shard

T, NCH = 257, 6


def _inputs():
    rng = np.random.default_rng(3)
    f = O.sigmoid_c((rng.standard_normal((NCH, T)) * 2).astype(np.float32))
    c = rng.standard_normal((NCH, T)).astype(np.float32)
    h0 = rng.standard_normal(NCH).astype(np.float32)
    return f, c, h0


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        f, c, h0 = _inputs()
        t0, t1 = shard.seq_slice(T, world, rank)
        agg = np.zeros((2, NCH), np.float32)
        for ch in range(NCH):
            A = np.float32(1.0)
            for t in range(t0, t1):
                A = np.float32(A * f[ch, t])
            agg[0, ch] = A
            agg[1, ch] = O.scan_seq(f[ch, t0:t1], c[ch, t0:t1], 0.0)[-1] if t1 > t0 else 0.0
        send = torch.from_numpy(agg)
        recv = [torch.empty_like(send) for _ in range(world)]
        dist.all_gather(recv, send)                               # the one exchange
        hin, hfin = h0.copy(), h0.copy()
        for j in range(world):                                    # compose in rank order
            if j == rank:
                hin = hfin.copy()
            Aj, Bj = recv[j].numpy()
            hfin = (Aj * hfin + Bj).astype(np.float32)
        h = np.stack([O.scan_seq(f[ch, t0:t1], c[ch, t0:t1], float(hin[ch]))
                      if t1 > t0 else np.zeros(0, np.float32) for ch in range(NCH)])
        q.put((rank, ((t0, t1), h, hfin)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_seq_slice_partition():
    for T_, W in ((2048, 8), (257, 3), (3, 4), (0, 2)):
        sl = [shard.seq_slice(T_, W, r) for r in range(W)]
        assert sl[0][0] == 0 and sl[-1][1] == T_
        assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
        assert max(b - a for a, b in sl) - min(b - a for a, b in sl) <= 1
    with pytest.raises(ValueError):
        shard.seq_slice(10, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_seqpar_scan_equals_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    f, c, h0 = _inputs()
    for ch in range(NCH):
        href, hf = O.scan_seqpar(f[ch], c[ch], world, float(h0[ch]))
        got = np.concatenate([res[r][1][ch] for r in range(world)])
        assert np.array_equal(got, href)
        for r in range(world):
            assert res[r][2][ch] == hf
