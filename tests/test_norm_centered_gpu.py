"""Centred norm variant (Alg. 1 rms_norm_fwd, PAPER.md P:330-332;
reading C22) through the C ABI against the oracle run in the same mode.

Every place the library normalizes a BitLinear input implements it: the prefill quant
kernel, the decode GEMV prologue, the batched-decode finalize and the persistent stack
kernel.  Rows carry a non-zero mean (x + 3) so that centring changes the codes.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu
CENT = 1


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


def shifted(shape, seed, dtype):
    x = synth.hidden(shape, synth.generator(seed), "f32") + 3.0
    return x.to(torch.bfloat16) if dtype == "bf16" else x


class norm_knob:
    def __init__(self, L, mode):
        self.L, self.mode = L, mode

    def __enter__(self):
        self.old = self.L.tern_get_norm_mode()
        self.L.tern_set_norm_mode(self.mode)

    def __exit__(self, *exc):
        self.L.tern_set_norm_mode(self.old)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("m,k", [(1, 256), (7, 688), (33, 1024), (5, 2816), (3, 6912), (300, 256)])
@pytest.mark.parametrize("with_gain", [False, True])
def test_quant_centered(L, m, k, dtype, with_gain):
    x = shifted((m, k), 70 + k, dtype)
    x[0, :] = 2.5                      # constant row: x - mu = 0 -> q = 0 (C7)
    gain = (1.0 + 0.3 * torch.randn(k, generator=synth.generator(3))) if with_gain else None
    kp = (k + 127) // 128 * 128
    q = torch.full((m, kp), 99, dtype=torch.int8, device="cuda")
    deq = torch.empty(m, device="cuda")
    qsum = torch.empty(m, dtype=torch.int32, device="cuda")
    r = torch.empty(m, device="cuda")
    a = torch.empty(m, device="cuda")
    with norm_knob(L, CENT):
        L.tern_quant(x.cuda(), q, deq, qsum, gain=None if gain is None else gain.cuda(),
                     inv_rms=r, absmax=a)
    torch.cuda.synchronize()
    with O.norm_mode(CENT):
        qo, do, ro, ao = O.quant_rows(f32np(x), gain=None if gain is None else gain.numpy())
    r_g = r.cpu().numpy()
    assert np.all(np.abs(r_g - ro) <= np.spacing(ro))
    same = r_g == ro
    assert same.mean() > 0.99
    qg = q.cpu().numpy()
    assert np.all(qg[:, k:] == 0)
    assert np.all(qg[0] == 0) and deq[0].item() == 0.0
    assert np.array_equal(qg[same, :k], qo[same])
    assert np.array_equal(deq.cpu().numpy()[same], do[same])
    assert np.array_equal(a.cpu().numpy()[same], ao[same])
    assert np.array_equal(qsum.cpu().numpy(), qg[:, :k].astype(np.int64).sum(1))
    if m > 1:
        with O.norm_mode(0):   # centring matters on these rows
            assert not np.array_equal(O.quant_rows(f32np(x))[0][1:], qo[1:])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("m,force_gemm", [(1, False), (3, False), (2, True), (130, False)])
def test_bitlinear_centered(L, M, m, force_gemm, dtype):
    k, n = 1024, 640
    W = synth.latent_matrix(n, k, synth.generator(41))
    pw = M.PackedWeight([W.cuda()])
    t, mw = O.ternarize(W.numpy())
    x = shifted((m, k), 43 + m, dtype)
    ydt = torch.bfloat16 if dtype == "bf16" else torch.float32
    y = torch.empty((m, n), dtype=ydt, device="cuda")
    old = L.tern_get_gemv_max_m()
    try:
        if force_gemm:
            L.tern_set_gemv_max_m(0)
        with norm_knob(L, CENT):
            L.bitlinear_fwd(x.cuda(), pw.struct, y)
        torch.cuda.synchronize()
    finally:
        L.tern_set_gemv_max_m(old)
    with O.norm_mode(CENT):
        ref = O.bitlinear(f32np(x), t, mw, bf16=(dtype == "bf16"))
    assert np.array_equal(f32np(y), ref)


def _stack(M, cfg, n_blocks, gate, extras=False):
    g = synth.generator(cfg.seed)
    blocks, ob = [], []
    for i in range(n_blocks):
        lat = synth.latent_block(cfg.d, cfg.l, g)
        gains = biases = None
        if extras:
            gg = synth.generator(cfg.seed * 100 + i)
            gains = {k: (1.0 + 0.25 * torch.randn(n, generator=gg)).cuda()
                     for k, n in (("x", cfg.d), ("o", cfg.d), ("x1", cfg.d), ("p", cfg.l))}
            biases = {k: (0.05 * torch.randn(cfg.d, generator=gg)).cuda() for k in ("f", "c", "g", "o")}
        ob.append(O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l,
                                gains=None if gains is None else {k: v.cpu().numpy() for k, v in gains.items()},
                                biases=None if biases is None else {k: v.cpu().numpy() for k, v in biases.items()}))
        blocks.append(M.Block(lat, cfg.d, cfg.l, gate=gate, eps=cfg.eps, gains=gains, biases=biases,
                              norm=CENT))
    st = M.Stack(blocks, cfg.d, cfg.l, synth.torch_dtype(cfg.dtype))
    st.link_blocks()
    return st, ob


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("gate", [0, 1])
def test_block_prefill_decode_centered(L, M, dtype, gate):
    """c0-shaped block (d=256, l=688): prefill (fused f|c|g+scan GEMM path) then
    decode (GEMV), free-running against the oracle in the centred mode."""
    B, T, n = 2, 128, 4
    cfg = synth.Config("nc", 2, 256, 688, dtype, 91, B, T, B, n)
    st, ob = _stack(M, cfg, 2, gate, extras=(gate == 1))
    x = shifted((B, T + n, cfg.d), 92, dtype)
    xd = x.cuda()
    states = st.new_state(B)
    ys = [st.prefill(xd[:, :T].contiguous(), states)]
    for t in range(T, T + n):
        ys.append(st.decode(xd[:, t].contiguous(), states).unsqueeze(1))
    torch.cuda.synchronize()
    bf = dtype == "bf16"
    Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
    xo = f32np(x)
    with O.norm_mode(CENT):
        y0, Hs = O.stack(ob, xo[:, :T], Hs, bf16=bf, gate_mode=gate)
        outs = [y0]
        for t in range(T, T + n):
            yt, Hs = O.stack(ob, xo[:, t:t + 1], Hs, bf16=bf, gate_mode=gate)
            outs.append(yt)
    assert np.array_equal(f32np(torch.cat(ys, 1)), np.concatenate(outs, 1))
    for h, ho in zip(states, Hs):
        assert np.array_equal(h.cpu().numpy(), ho)


@pytest.mark.parametrize("fin", [False, True])
def test_batched_decode_centered(L, M, fin):
    """B = 24 decode steps (split-K GEMM; with fin, the row-wise finalize quantizes
    each output row for the next BitLinear in the centred mode)."""
    B, n = 24, 3
    cfg = synth.Config("nb", 2, 256, 688, "f32", 95, B, 0, B, n)
    st, ob = _stack(M, cfg, 2, 0, extras=True)
    xs = [shifted((B, cfg.d), 960 + t, "f32") for t in range(n)]
    states = st.new_state(B)
    old = L.tern_get_batched_fin()
    try:
        L.tern_set_batched_fin(fin)
        ys = [st.decode(x.cuda(), states).clone() for x in xs]
        torch.cuda.synchronize()
    finally:
        L.tern_set_batched_fin(old)
    Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
    with O.norm_mode(CENT):
        for t in range(n):
            yo, Hs = O.stack(ob, f32np(xs[t])[:, None, :], Hs)
            assert np.array_equal(f32np(ys[t]), yo[:, 0]), f"step {t}"
    for h, ho in zip(states, Hs):
        assert np.array_equal(h.cpu().numpy(), ho)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_persistent_stack_decode_centered(L, M, dtype):
    """The one-launch stack decode (stack_decode) equals the per-block chain."""
    B, n = 2, 4
    cfg = synth.Config("ns", 3, 256, 688, dtype, 97, B, 0, B, n)
    st, _ = _stack(M, cfg, 3, 0, extras=True)
    xs = [shifted((B, cfg.d), 980 + t, dtype).cuda() for t in range(n)]
    out = {}
    for persistent in (True, False):
        states = st.new_state(B)
        out[persistent] = [st.decode(x, states, persistent=persistent).clone() for x in xs]
        out[persistent].append(torch.cat([h.clone() for h in states]))
        assert st.last_decode_path == ("persistent" if persistent else "per_block")
    torch.cuda.synchronize()
    for a, b in zip(out[True], out[False]):
        assert torch.equal(a, b)
