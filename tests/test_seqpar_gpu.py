"""Sequence-parallel prefill (tern.h block_prefill_sp; SURVEY 8(f) f3's long-context
variant; reading C23) through the C ABI on one GPU: `world` virtual ranks as host threads,
each on its own stream holding one contiguous token slice of every sequence, exchanging the
scan's slice aggregates through the library's all-gather callback (shard.ThreadAllGather:
CUDA events + copies, no kernel waits on another).  Every rank's outputs and the final
states must equal the oracle's W-slice scan (O.scan_slices) bit for bit; world = 1 must
equal block_prefill.
"""
import threading

import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu


def _stack(cfg, keep):
    from paper_2406_02528_b200 import model
    return model.Stack.random(cfg, device="cuda", gen_device="cpu", keep_latents=keep)


def _run_sp(st, x, world, B):
    from paper_2406_02528_b200 import shard
    T = x.shape[1]
    gather = shard.ThreadAllGather(world)
    outs, states, errs = [None] * world, [None] * world, []

    def worker(r):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                t0, t1 = shard.seq_slice(T, world, r)
                xr = x[:, t0:t1].contiguous()
                h = st.new_state(B)
                y = st.prefill_sp(xr, h, gather, r)
                s.synchronize()
                outs[r] = y.clone()
                states[r] = [hh.clone() for hh in h]
        except Exception as e:   # re-raised in the main thread
            errs.append(e)
            gather.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return torch.cat(outs, 1), states


def _oracle(st, cfg, x, world, gate=0):
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in st.latents]
    Hs = [np.zeros((x.shape[0], cfg.d), np.float32) for _ in ob]
    with O.scan_slices(world):
        y, Hs = O.stack(ob, x.float().cpu().numpy(), Hs, bf16=(cfg.dtype == "bf16"), gate_mode=gate)
    return y, Hs


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("world,B,T", [(2, 2, 256), (4, 1, 300), (3, 2, 130), (8, 1, 64)])
def test_seqpar_prefill_matches_oracle(dtype, world, B, T):
    cfg = synth.Config("sp", 2, 256, 688, dtype, 31 + world, B, T, B, 0)
    st = _stack(cfg, 2)
    x = synth.hidden((B, T, cfg.d), synth.generator(5 + world), dtype).cuda()
    y, states = _run_sp(st, x, world, B)
    yo, Ho = _oracle(st, cfg, x, world)
    assert np.array_equal(y.float().cpu().numpy(), yo)
    for r in range(world):                       # the same final state on every rank
        for h, ho in zip(states[r], Ho):
            assert np.array_equal(h.cpu().numpy(), ho), f"rank {r}"


def test_seqpar_world1_equals_block_prefill():
    B, T = 2, 200
    cfg = synth.Config("sp1", 2, 256, 688, "f32", 7, B, T, B, 0)
    st = _stack(cfg, 0)
    x = synth.hidden((B, T, cfg.d), synth.generator(9), "f32").cuda()
    y1, s1 = _run_sp(st, x, 1, B)
    h = st.new_state(B)
    y = st.prefill(x, h)
    torch.cuda.synchronize()
    assert torch.equal(y1, y) and all(torch.equal(a, b) for a, b in zip(s1[0], h))


def test_seqpar_then_decode_close_to_sequential():
    """The W-slice prefill differs from the sequential one only by the reassociated boundary
    states: slice 0's outputs are bit-identical, the rest and the decode steps that follow
    (from the composed state) agree within the chunked-scan tolerance."""
    B, T, world = 1, 512, 4
    cfg = synth.Config("spd", 2, 256, 688, "f32", 11, B, T, B, 0)
    st = _stack(cfg, 0)
    x = synth.hidden((B, T + 3, cfg.d), synth.generator(13), "f32").cuda()
    ysp, states = _run_sp(st, x[:, :T].contiguous(), world, B)
    h = st.new_state(B)
    yseq = st.prefill(x[:, :T].contiguous(), h)
    torch.cuda.synchronize()
    assert torch.equal(ysp[:, :T // world], yseq[:, :T // world])
    assert torch.allclose(ysp, yseq, rtol=1e-3, atol=1e-3)
    hs = states[0]
    for t in range(T, T + 3):
        a = st.decode(x[:, t].contiguous(), hs).clone()
        b = st.decode(x[:, t].contiguous(), h).clone()
        assert torch.allclose(a, b, rtol=1e-3, atol=1e-3)


def test_seqpar_rank_without_tokens():
    """world > T: ranks with an empty slice still join every exchange (identity aggregate)."""
    B, T, world = 1, 3, 4
    cfg = synth.Config("spe", 1, 256, 688, "f32", 17, B, T, B, 0)
    st = _stack(cfg, 1)
    x = synth.hidden((B, T, cfg.d), synth.generator(19), "f32").cuda()
    y, states = _run_sp(st, x, world, B)
    yo, Ho = _oracle(st, cfg, x, world)
    assert np.array_equal(y.cpu().numpy(), yo)
    for r in range(world):
        assert np.array_equal(states[r][0].cpu().numpy(), Ho[0])
