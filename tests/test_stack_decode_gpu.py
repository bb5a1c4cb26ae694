"""Whole-stack persistent decode (tern.h stack_decode) through the C ABI.

One decode step through all blocks runs as ONE cooperative kernel with grid barriers
between the 4 dependent BitLinear phases of every block.  Its arithmetic is the decode
GEMV's, so it must be bit-identical to the per-block path (block_decode x L), which
test_parity_gpu.py pins to the oracle; the oracle is also checked directly here.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_2406_02528_b200 import _lib
    _lib.load()
    return _lib


@pytest.fixture(scope="module")
def M():
    from paper_2406_02528_b200 import model
    return model


def f32np(t):
    return t.detach().float().cpu().numpy()


def _stack(M, cfg, n_blocks, gate, extras=False, keep=0):
    """Stack of n_blocks seeded blocks; extras adds non-unit gains and biases."""
    g = synth.generator(cfg.seed)
    blocks, kept = [], []
    for i in range(n_blocks):
        lat = synth.latent_block(cfg.d, cfg.l, g)
        gains, biases = None, None
        if extras:
            gg = synth.generator(cfg.seed * 100 + i)
            gains = {k: (1.0 + 0.25 * torch.randn(n, generator=gg)).cuda()
                     for k, n in (("x", cfg.d), ("o", cfg.d), ("x1", cfg.d), ("p", cfg.l))}
            biases = {k: (0.05 * torch.randn(cfg.d, generator=gg)).cuda()
                      for k in ("f", "c", "g", "o")}
        if i < keep:
            kept.append((lat, gains, biases))
        blocks.append(M.Block(lat, cfg.d, cfg.l, gate=gate, eps=cfg.eps, gains=gains,
                              biases=biases))
    st = M.Stack(blocks, cfg.d, cfg.l, synth.torch_dtype(cfg.dtype))
    st.link_blocks()
    return st, kept


def _run(st, xs, B, persistent, graph=False):
    states = st.new_state(B)
    ys = []
    if graph:
        st.persistent_decode = persistent
        gr, x_in, y_out = st.capture_decode(B, states)
        for x in xs:
            x_in.copy_(x)
            gr.replay()
            ys.append(y_out.clone())
    else:
        for x in xs:
            ys.append(st.decode(x, states, persistent=persistent).clone())
    torch.cuda.synchronize()
    return torch.stack(ys), [h.clone() for h in states]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("B", [1, 2, 3, 4])
@pytest.mark.parametrize("gate", [0, 1])
def test_persistent_equals_per_block(L, M, dtype, B, gate):
    cfg = synth.Config("sd", 3, 256, 688, dtype, 41 + B, B, 0, B, 5)
    st, _ = _stack(M, cfg, 3, gate, extras=(B == 3))
    xs = [synth.hidden((B, cfg.d), synth.generator(500 + t), dtype).cuda() for t in range(5)]
    yp, hp = _run(st, xs, B, True)
    yb, hb = _run(st, xs, B, False)
    assert torch.equal(yp, yb), "persistent decode output differs from block_decode"
    for a, b in zip(hp, hb):
        assert torch.equal(a, b), "persistent decode state differs"


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_persistent_vs_oracle_with_gains_and_biases(L, M, dtype):
    """Free-running 2-block stack, B = 3, non-unit gains and biases: oracle bit-exact."""
    B, n = 3, 4
    cfg = synth.Config("so", 2, 256, 688, dtype, 57, B, 0, B, n)
    st, kept = _stack(M, cfg, 2, 0, extras=True, keep=2)
    ob = []
    for lat, gains, biases in kept:
        ob.append(O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l,
                                gains={k: v.cpu().numpy() for k, v in gains.items()},
                                biases={k: v.cpu().numpy() for k, v in biases.items()}))
    xs = [synth.hidden((B, cfg.d), synth.generator(900 + t), dtype) for t in range(n)]
    yp, hp = _run(st, [x.cuda() for x in xs], B, True)
    Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
    bf = dtype == "bf16"
    for t in range(n):
        yo, Hs = O.stack(ob, f32np(xs[t])[:, None, :], Hs, bf16=bf)
        assert np.array_equal(f32np(yp[t]), yo[:, 0]), f"step {t}"
    for a, b in zip(hp, Hs):
        assert np.array_equal(a.cpu().numpy(), b)


def test_chunked_launches(L, M):
    """More than 32 blocks: the step is split into several persistent launches."""
    B = 2
    cfg = synth.Config("sc", 34, 128, 256, "f32", 61, B, 0, B, 3)
    st, _ = _stack(M, cfg, 34, 0)
    xs = [synth.hidden((B, cfg.d), synth.generator(700 + t), "f32").cuda() for t in range(3)]
    yp, hp = _run(st, xs, B, True)
    yb, hb = _run(st, xs, B, False)
    assert torch.equal(yp, yb)
    for a, b in zip(hp, hb):
        assert torch.equal(a, b)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_graph_captured_persistent(L, M, dtype):
    """The persistent step captured in a CUDA graph (memset + cooperative kernel) and
    replayed equals eager per-block decoding."""
    B = 1
    cfg = synth.Config("sg", 4, 512, 1408, dtype, 67, B, 0, B, 6)
    st, _ = _stack(M, cfg, 4, 0)
    xs = [synth.hidden((B, cfg.d), synth.generator(800 + t), dtype).cuda() for t in range(6)]
    yg, hg = _run(st, xs, B, True, graph=True)
    yb, hb = _run(st, xs, B, False)
    assert torch.equal(yg, yb)
    for a, b in zip(hg, hb):
        assert torch.equal(a, b)


def test_unsupported_shape_reports_and_falls_back(L, M):
    """B = 5 exceeds the persistent plan: the C call returns TERN_ERR_UNSUPPORTED with no
    side effects and Stack.decode takes the per-block path (same results)."""
    B = 5
    cfg = synth.Config("su", 2, 256, 688, "f32", 71, B, 0, B, 2)
    st, _ = _stack(M, cfg, 2, 0)
    x = synth.hidden((B, cfg.d), synth.generator(1), "f32").cuda()
    arr = st._stack_struct()
    ws = torch.zeros(L.tern_stack_decode_workspace(arr, B, torch.float32), dtype=torch.uint8,
                     device="cuda")
    y = torch.full_like(x, 7.0)
    states = st.new_state(B)
    assert L.stack_decode(arr, x, y, states, ws, allow_unsupported=True) == L.TERN_ERR_UNSUPPORTED
    torch.cuda.synchronize()
    assert torch.all(y == 7.0) and all(torch.all(h == 0) for h in states)
    yp, _ = _run(st, [x], B, True)
    yb, _ = _run(st, [x], B, False)
    assert torch.equal(yp, yb)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_batched_decode_with_gains_and_biases(L, M, dtype):
    """Batched decode (B = 24 > the GEMV limit: split-K GEMM + row-wise finalize with the
    next BitLinear's quant fused, k_fin.cu) with non-unit gains and biases: oracle bit-exact."""
    B, n = 24, 3
    cfg = synth.Config("bg", 2, 256, 688, dtype, 83, B, 0, B, n)
    st, kept = _stack(M, cfg, 2, 1, extras=True, keep=2)
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l,
                        gains={k: v.cpu().numpy() for k, v in gains.items()},
                        biases={k: v.cpu().numpy() for k, v in biases.items()})
          for lat, gains, biases in kept]
    xs = [synth.hidden((B, cfg.d), synth.generator(950 + t), dtype) for t in range(n)]
    old = L.tern_get_batched_fin()
    try:
        L.tern_set_batched_fin(True)
        yp, hp = _run(st, [x.cuda() for x in xs], B, False)
    finally:
        L.tern_set_batched_fin(old)
    yq, hq = _run(st, [x.cuda() for x in xs], B, False)   # quant + GEMM + epilogue path
    assert torch.equal(yp, yq) and all(torch.equal(a, b) for a, b in zip(hp, hq))
    Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
    for t in range(n):
        yo, Hs = O.stack(ob, f32np(xs[t])[:, None, :], Hs, bf16=(dtype == "bf16"), gate_mode=1)
        assert np.array_equal(f32np(yp[t]), yo[:, 0]), f"step {t}"
    for a, b in zip(hp, Hs):
        assert np.array_equal(a.cpu().numpy(), b)
