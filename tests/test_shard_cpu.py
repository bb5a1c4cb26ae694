"""Output-feature sharding, host side (world_size 2, gloo, CPU).

Each process takes rank r of paper_2406_02528_b200.shard.plan(), computes its
slice of every BitLinear of a block with the ORACLE (ternary rows of the full
matrices, i.e. the full-matrix scale), and gathers o', x1, p and y
over gloo exactly where the library calls its all-gather callback (tern.h
tern_shard).  The gathered result must equal the unsharded oracle block bit for
bit, for prefill and a decode step continuing the sharded state: the partition
and the composition are what the GPU path runs.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2406_02528_b200 import shard, synth

D, LW, B, T = 256, 512, 2, 9


def _block_latents():
    g = synth.generator(7)
    return {k: v.numpy() for k, v in synth.latent_block(D, LW, g).items()}


def _gather(part):
    """all-gather along the last (feature) axis in rank order."""
    t = torch.from_numpy(np.ascontiguousarray(part))
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return torch.cat(out, dim=-1).numpy()


def _sharded_block(lat, x, H_shard, rank, world, gate):
    """One block with rank's slices + gathers; returns (y_full, new H_shard)."""
    p = shard.plan(D, LW, world, rank)
    c0, c1 = p["ch"]
    g0, g1 = p["gl"]
    t, m = {}, {}
    for k in lat:
        t[k], m[k] = O.ternarize(lat[k])   # full-matrix scale (one per matrix)
    Bx, Tx, _ = x.shape
    X = x.reshape(Bx * Tx, D)
    fh = O.bitlinear(X, t["f"][c0:c1], m["f"]).reshape(Bx, Tx, -1)
    ch = O.bitlinear(X, t["c"][c0:c1], m["c"]).reshape(Bx, Tx, -1)
    gh = O.bitlinear(X, t["g"][c0:c1], m["g"]).reshape(Bx, Tx, -1)
    op, H_shard = O.mlgru_scan(fh, ch, gh, H_shard, gate_mode=gate)
    op_full = _gather(op.reshape(Bx * Tx, -1))                        # gather 1: o'
    x1_s = X[:, c0:c1] + O.bitlinear(op_full, t["o"][c0:c1], m["o"])
    x1 = _gather(x1_s)                                                # gather 2: x1
    gg = O.bitlinear(x1, t["gate"][g0:g1], m["gate"])
    uu = O.bitlinear(x1, t["up"][g0:g1], m["up"])
    p_s = O.silu_mul(gg, uu)
    p_full = _gather(p_s)                                             # gather 3: p
    y_s = x1[:, c0:c1] + O.bitlinear(p_full, t["down"][c0:c1], m["down"])
    y = _gather(y_s)                                                  # gather 4: y
    return y.reshape(Bx, Tx, D), H_shard


def _allreduce_i64(a):
    t = torch.from_numpy(np.ascontiguousarray(a.astype(np.int64)))
    dist.all_reduce(t)
    return t.numpy()


def _rowpar_bitlinear(x_r, t_cols, m_w, K, eps=1e-6):
    """Row-parallel BitLinear on rank's input slice x_r: the row
    moments are exchanged (binary64 partials summed in rank order), the slice is
    quantized with the shared r / absmax and its int32 products with
    the weight columns are all-reduced (exact) before the dequantization."""
    x64 = x_r.astype(np.float64)
    ss = _gather(np.sum(x64 * x64, axis=1, keepdims=True))    # [M][world] partials
    mx = _gather(np.max(np.abs(x_r), axis=1, keepdims=True).astype(np.float32))
    ss_tot = np.zeros(ss.shape[0])
    for r in range(ss.shape[1]):
        ss_tot = ss_tot + ss[:, r]
    r32 = (1.0 / np.sqrt(ss_tot / K + eps)).astype(np.float32)
    amax = (np.max(mx, axis=1) * r32).astype(np.float32)
    y = (x_r * r32[:, None]).astype(np.float32)
    sc = np.where(amax > 0, np.float32(127.0) / np.where(amax > 0, amax, 1), 0).astype(np.float32)
    v = (y * sc[:, None]).astype(np.float32)
    q = np.clip(np.sign(v) * np.floor(np.abs(v) + np.float32(0.5)), -128, 127).astype(np.int64)
    acc = _allreduce_i64(q @ t_cols.astype(np.int64).T)
    deq = np.where(amax > 0, (amax / np.float32(127.0)).astype(np.float32), 0).astype(np.float32)
    return (acc.astype(np.float32) * (deq * np.float32(m_w))[:, None]).astype(np.float32)


def _megatron_block(lat, x, H_shard, rank, world, gate):
    """Megatron-paired block (tern_shard.megatron): f|c|g and gate|up column-parallel,
    o and down row-parallel with int32 all-reduces; x1 and y come out whole."""
    p = shard.plan(D, LW, world, rank)
    c0, c1 = p["ch"]
    g0, g1 = p["gl"]
    t, m = {}, {}
    for k in lat:
        t[k], m[k] = O.ternarize(lat[k])
    Bx, Tx, _ = x.shape
    X = x.reshape(Bx * Tx, D)
    fh = O.bitlinear(X, t["f"][c0:c1], m["f"]).reshape(Bx, Tx, -1)
    ch = O.bitlinear(X, t["c"][c0:c1], m["c"]).reshape(Bx, Tx, -1)
    gh = O.bitlinear(X, t["g"][c0:c1], m["g"]).reshape(Bx, Tx, -1)
    op, H_shard = O.mlgru_scan(fh, ch, gh, H_shard, gate_mode=gate)
    o = _rowpar_bitlinear(op.reshape(Bx * Tx, -1), t["o"][:, c0:c1], m["o"], D)
    x1 = (X + o).astype(np.float32)
    gg = O.bitlinear(x1, t["gate"][g0:g1], m["gate"])
    uu = O.bitlinear(x1, t["up"][g0:g1], m["up"])
    p_s = O.silu_mul(gg, uu)
    dn = _rowpar_bitlinear(p_s, t["down"][:, g0:g1], m["down"], LW)
    y = (x1 + dn).astype(np.float32)
    return y.reshape(Bx, Tx, D), H_shard


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O.set_threads(1)
        lat = _block_latents()
        g = synth.generator(11)
        x = synth.hidden((B, T + 1, D), g).numpy()
        res = {}
        for gate in (0, 1):
            ds = shard.plan(D, LW, world, rank)["ds"]
            Hs = np.zeros((B, ds), np.float32)
            y0, Hs = _sharded_block(lat, x[:, :T], Hs, rank, world, gate)   # prefill
            y1, Hs = _sharded_block(lat, x[:, T:], Hs, rank, world, gate)   # decode step
            res[gate] = (y0, y1, _gather(Hs))
            Hm = np.zeros((B, ds), np.float32)
            m0, Hm = _megatron_block(lat, x[:, :T], Hm, rank, world, gate)
            m1, Hm = _megatron_block(lat, x[:, T:], Hm, rank, world, gate)
            res[("mega", gate)] = (m0, m1, _gather(Hm))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plan_partitions_and_validates():
    parts = [shard.plan(2048, 5632, 8, r) for r in range(8)]
    assert [p["ch"] for p in parts] == [(256 * r, 256 * (r + 1)) for r in range(8)]
    assert [p["gl"] for p in parts] == [(704 * r, 704 * (r + 1)) for r in range(8)]
    assert shard.plan(1024, 2816, 1, 0) == {"ds": 1024, "ls": 2816, "ch": (0, 1024),
                                             "gl": (0, 2816)}
    with pytest.raises(ValueError):
        shard.plan(256, 688, 2, 0)      # l/world = 344 is not a multiple of 16
    with pytest.raises(ValueError):
        shard.plan(192, 512, 2, 0)      # d/world = 96 is not a multiple of 64
    with pytest.raises(ValueError):
        shard.plan(256, 512, 2, 2)


def test_shard_latents_rows():
    lat = {k: torch.arange(n * k_, dtype=torch.float32).reshape(n, k_)
           for k, (n, k_) in synth.weight_shapes(256, 512).items()}
    s1 = shard.shard_latents(lat, 256, 512, 2, 1)
    assert torch.equal(s1["f"], lat["f"][128:256]) and torch.equal(s1["down"], lat["down"][128:])
    assert torch.equal(s1["gate"], lat["gate"][256:512]) and s1["up"].shape == (256, 256)


def test_two_rank_gloo_sharded_block_equals_unsharded_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lat = _block_latents()
    ob = O.OracleBlock(lat, D, LW)
    g = synth.generator(11)
    x = synth.hidden((B, T + 1, D), g).numpy()
    for gate in (0, 1):
        H = np.zeros((B, D), np.float32)
        y0, H = O.block(ob, x[:, :T], H, gate_mode=gate)
        y1, H = O.block(ob, x[:, T:], H, gate_mode=gate)
        for r in range(world):
            g0, g1, Hg = out[r][gate]
            assert np.array_equal(g0, y0), f"prefill rank {r} gate {gate}"
            assert np.array_equal(g1, y1), f"decode rank {r} gate {gate}"
            assert np.array_equal(Hg, H), f"state rank {r} gate {gate}"
            m0, m1, Hm = out[r][("mega", gate)]   # Megatron pairing (f1(ii))
            assert np.array_equal(m0, y0), f"megatron prefill rank {r} gate {gate}"
            assert np.array_equal(m1, y1), f"megatron decode rank {r} gate {gate}"
            assert np.array_equal(Hm, H), f"megatron state rank {r} gate {gate}"
