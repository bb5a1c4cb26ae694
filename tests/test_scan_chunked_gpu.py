"""The chunked prefill scan (tern.h tern_mlgru.num_chunks = 4; "parallel
scan", reading C23 for the composition): each channel's sequence is cut into 4 contiguous
chunks [j T/4, (j+1) T/4) that run concurrently from their composed boundary states.  The
oracle computes the same composition literally (O.scan_slices(4): chunk aggregates from
h = 0, composed in chunk order, each chunk scanned from its boundary, final state = the
composition through every chunk), so the GPU must match it BIT FOR BIT; against the
sequential definition the scan differs only by reassociation (S4: within 1e-5 relative for
h, pinned on the oracle side in tests/test_oracle_pins.py).
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu


def _run(cfg, B, T, num_chunks, gate=0, n_blocks=1):
    from paper_2406_02528_b200 import _lib as L
    from paper_2406_02528_b200 import model
    L.load()
    st = model.Stack.random(cfg, device="cuda", gen_device="cpu", keep_latents=n_blocks,
                            n_blocks=n_blocks, gate=gate, num_chunks=num_chunks)
    x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 5), cfg.dtype)
    hs = st.new_state(B)
    y = st.prefill(x.cuda(), hs)
    torch.cuda.synchronize()
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in st.latents]
    return st, x, y, hs, ob


@pytest.mark.parametrize("nch", [4, 8])
@pytest.mark.parametrize("dtype,B,T,gate", [("f32", 1, 2048, 0), ("bf16", 1, 2048, 1),
                                            ("f32", 2, 1030, 1), ("bf16", 3, 517, 0),
                                            ("f32", 1, 9, 0), ("f32", 1, 4, 0)])
def test_chunked_scan_equals_oracle_composition(dtype, B, T, gate, nch):
    """num_chunks = 4 and 8 through block_prefill (ragged chunks: T = 1030, 517, 9 are not
    multiples of nch x 64; T = 4: one step per chunk, or none for half of the 8), both gate
    modes, fp32 and bf16: y and the per-block state equal O.stack under O.scan_slices(nch)
    bit for bit.  (d = 256: the cluster kernel, 8 groups of 32 channels.)"""
    cfg = synth.Config("chk", 1, 256, 688, dtype, 61, B, T, B, 0)
    st, x, y, hs, ob = _run(cfg, B, T, nch, gate)
    assert st.blocks[0].scan_chunks(B, T) == nch
    with O.scan_slices(nch):
        yo, Ho = O.stack(ob, x.float().numpy(), [np.zeros((B, cfg.d), np.float32)],
                         bf16=(dtype == "bf16"), gate_mode=gate)
    assert np.array_equal(y.float().cpu().numpy(), yo)
    assert np.array_equal(hs[0].cpu().numpy(), Ho[0])


def test_chunked_scan_at_c2_batch1():
    """The c2 width at batch 1 x 2048 (P:198's workload) with num_chunks = 4 through 2 blocks:
    bit for bit the oracle's 4-slice composition; the first block's final state within S4's
    1e-5 of the sequential recurrence's; auto (num_chunks = 0) resolves to the sequential
    scan (measured faster)."""
    cfg = synth.CONFIGS["c2"]
    B, T = 1, 2048
    st, x, y, hs, ob = _run(cfg, B, T, 4, n_blocks=2)
    assert st.blocks[0].scan_chunks(B, T) == 4
    with O.scan_slices(4):
        yo, Ho = O.stack(ob, x.float().numpy(), [np.zeros((B, cfg.d), np.float32)] * 2)
    assert np.array_equal(y.float().cpu().numpy(), yo)
    for i in range(2):
        assert np.array_equal(hs[i].cpu().numpy(), Ho[i])
    with O.scan_slices(4):
        _, H4 = O.stack(ob[:1], x.float().numpy(), [np.zeros((B, cfg.d), np.float32)])
    _, Hseq = O.stack(ob[:1], x.float().numpy(), [np.zeros((B, cfg.d), np.float32)])
    assert np.all(np.abs(H4[0] - Hseq[0]) <= 1e-5 * np.maximum(np.abs(Hseq[0]), 1e-2))
    st0, *_ = _run(synth.Config("auto", 1, 256, 688, "f32", 63, 1, 8, 1, 0), 1, 8, 0)
    assert st0.blocks[0].scan_chunks(1, 4096) == 1


def test_eight_chunks_at_c2_batch1_and_fallbacks():
    """num_chunks = 8 at the c2 width, batch 1 x 2048 through 2 blocks: bit for bit the
    oracle's 8-slice composition; beyond 8 x 512 steps (T = 4104) it resolves to the exact
    sequential scan and then equals the sequential oracle."""
    cfg = synth.CONFIGS["c2"]
    st, x, y, hs, ob = _run(cfg, 1, 2048, 8, n_blocks=2)
    assert st.blocks[0].scan_chunks(1, 2048) == 8
    with O.scan_slices(8):
        yo, Ho = O.stack(ob, x.float().numpy(), [np.zeros((1, cfg.d), np.float32)] * 2)
    assert np.array_equal(y.float().cpu().numpy(), yo)
    for i in range(2):
        assert np.array_equal(hs[i].cpu().numpy(), Ho[i])
    cfg2 = synth.Config("chk8", 1, 256, 688, "f32", 64, 1, 4104, 1, 0)
    st2, x2, y2, hs2, ob2 = _run(cfg2, 1, 4104, 8)
    assert st2.blocks[0].scan_chunks(1, 4104) == 1
    yo2, Ho2 = O.stack(ob2, x2.float().numpy(), [np.zeros((1, cfg2.d), np.float32)])
    assert np.array_equal(y2.float().cpu().numpy(), yo2)
    assert np.array_equal(hs2[0].cpu().numpy(), Ho2[0])


def test_num_chunks_one_stays_exact():
    """num_chunks = 1 forces the exact sequential scan even where auto would chunk."""
    cfg = synth.Config("chk1", 1, 256, 688, "f32", 62, 1, 1100, 1, 0)
    st, x, y, hs, ob = _run(cfg, 1, 1100, 1)
    assert st.blocks[0].scan_chunks(1, 1100) == 1
    yo, Ho = O.stack(ob, x.float().numpy(), [np.zeros((1, cfg.d), np.float32)])
    assert np.array_equal(y.float().cpu().numpy(), yo)
    assert np.array_equal(hs[0].cpu().numpy(), Ho[0])
