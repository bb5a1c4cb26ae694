"""Output-feature sharding through the C ABI on one GPU (tern.h tern_shard):
`world` virtual ranks run as host threads, each on its own stream with its own
shard of every weight, exchanging o', x1, p and y through the library's
all-gather callback (shard.ThreadAllGather: CUDA events + copies, no kernel
waits on another).  Every rank's output must be bit-identical to the unsharded
library path, and that one must match the oracle's unsharded stack (O.stack,
prefill then decode, north_star tolerances; in practice bit-exact): gathers
move values unchanged, int32 sums are exact and every norm sees the full row.
"""
import threading

import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu


def _run(world, cfg, T, n_dec, B, gather_q=False, norm=0, megatron=False):
    from paper_2406_02528_b200 import _lib as L
    from paper_2406_02528_b200 import model, shard
    L.load()
    ref = model.Stack.random(cfg, device="cuda", gen_device="cpu", norm=norm,
                             keep_latents=cfg.L)
    x = synth.hidden((B, T + n_dec, cfg.d), synth.generator(3), cfg.dtype).cuda()
    hs = ref.new_state(B)
    ys = [ref.prefill(x[:, :T].contiguous(), hs)]
    for t in range(T, T + n_dec):
        ys.append(ref.decode(x[:, t].contiguous(), hs).unsqueeze(1))
    torch.cuda.synchronize()
    yref = torch.cat(ys, 1)
    # the unsharded result against the oracle's unsharded stack (prefill, then decode steps)
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l)
          for lat in ref.latents]
    xo = x.float().cpu().numpy()
    bf = cfg.dtype == "bf16"
    with O.norm_mode(norm):
        Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
        yo, Hs = O.stack(ob, xo[:, :T], Hs, bf16=bf, eps=cfg.eps)
        outs = [yo]
        for t in range(T, T + n_dec):
            yt, Hs = O.stack(ob, xo[:, t:t + 1], Hs, bf16=bf, eps=cfg.eps)
            outs.append(yt)
    yo = np.concatenate(outs, 1)
    g = yref.float().cpu().numpy()
    tol = 2e-2 if bf else 1e-4
    rms = np.sqrt((yo.astype(np.float64) ** 2).mean(-1, keepdims=True))
    assert np.all(np.abs(g - yo) <= tol * np.maximum(np.abs(yo), 1e-2 * rms)), \
        f"unsharded CUDA vs oracle: max abs err {np.abs(g - yo).max()}"

    gather = shard.ThreadAllGather(world)
    stacks = [model.Stack.random(cfg, device="cuda", gen_device="cpu", shard=(r, gather, gather_q, megatron),
                                 norm=norm)
              for r in range(world)]
    outs, errs = [None] * world, []

    def worker(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                st = stacks[r]
                h = st.new_state(B)
                xr = x.clone()
                gather.register(xr)
                o = [st.prefill(xr[:, :T].contiguous(), h)]
                for t in range(T, T + n_dec):
                    o.append(st.decode(xr[:, t].contiguous(), h).unsqueeze(1))
                s.synchronize()
                outs[r] = torch.cat(o, 1)
        except Exception as e:   # re-raised in the main thread
            errs.append(e)
            gather.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    for r in range(world):   # sharded == unsharded (bit for bit) == oracle (tolerance above)
        assert torch.equal(outs[r], yref), f"rank {r} differs from the unsharded path"


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_block_prefill_decode_bit_identical(world):
    cfg = synth.Config("shard", 2, 512, 1024, "f32", 21, 2, 40, 2, 3)
    _run(world, cfg, T=40, n_dec=3, B=2)


def test_sharded_bf16_batch1_decode():
    cfg = synth.Config("shard_bf16", 1, 256, 512, "bf16", 22, 1, 33, 1, 4)
    _run(2, cfg, T=33, n_dec=4, B=1)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype,norm", [("f32", 0), ("bf16", 1)])
def test_sharded_int8_code_gathers(world, dtype, norm):
    """tern_shard.gather_q: o', x1 and p cross the ranks as int8
    codes after a binary64 moment exchange; prefill (M = 80) and decode with B = 8
    run the tensor-core path that uses it.  Equal to the unsharded path (the moment
    sums differ only in order: reading C4)."""
    cfg = synth.Config("shard_q", 2, 512, 1024, dtype, 23, 8, 10, 8, 2)
    _run(world, cfg, T=10, n_dec=2, B=8, gather_q=True, norm=norm)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype,norm", [("f32", 0), ("bf16", 1)])
def test_megatron_paired_sharding(world, dtype, norm):
    """tern_shard.megatron: f|c|g and gate|up column-parallel, o and
    down row-parallel with the int32 partials of all outputs summed by the all-reduce
    callback (exact); prefill and decode (B = 1 takes the GEMV for f|c|g and the
    tensor-core path for the row-parallel BitLinears).  Equal to the unsharded path up to
    the order of the row-moment sums (reading C4)."""
    cfg = synth.Config("shard_mg", 2, 512, 1024, dtype, 29, 2, 40, 2, 3)
    _run(world, cfg, T=40, n_dec=3, B=2, norm=norm, megatron=True)
