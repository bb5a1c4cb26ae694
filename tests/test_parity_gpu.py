"""GPU-vs-oracle parity of every hot-path step, through the C ABI (B200 only).

Bar (BASELINE.json north_star): ternary codes,
int8 activations and int32 accumulators bit-exact given the same fp32 scales;
float outputs and hidden states within 1e-4 relative (fp32) / 2e-2 (bf16) --
and, because both sides follow the canonical numerics, they are expected (and
here required, up to logged fp64-boundary events) to be bit-identical.
"""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2406_02528_b200 import synth

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-4, torch.bfloat16: 2e-2}


@pytest.fixture(scope="module")
def L():
    from paper_2406_02528_b200 import _lib
    _lib.load()
    return _lib


@pytest.fixture(scope="module")
def M():
    from paper_2406_02528_b200 import model
    return model


def dev(x):
    return torch.as_tensor(x).cuda()


def f32np(t):
    return t.detach().float().cpu().numpy()


def close(g, o, tol, what=""):
    """Elementwise |g-o| <= tol*max(|o|, 1e-2*rms(o_row)) (DESIGN.md tolerance rule)."""
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    o2 = o.reshape(-1, o.shape[-1]) if o.ndim > 1 else o.reshape(1, -1)
    rms = np.sqrt(np.mean(o2 ** 2, axis=1, keepdims=True)).repeat(o2.shape[1], 1).reshape(o.shape)
    lim = tol * np.maximum(np.abs(o), 1e-2 * rms) + 1e-30
    bad = np.abs(g - o) > lim
    assert not bad.any(), f"{what}: {bad.sum()} / {bad.size} outside tol {tol}; " \
                          f"max abs err {np.max(np.abs(g - o)):.3e}"


def latents(n, k, seed):
    g = synth.generator(seed)
    return synth.latent_matrix(n, k, g)


def acts(shape, seed, dtype="f32"):
    g = synth.generator(seed)
    return synth.hidden(shape, g, dtype)


# ------------------------------------------------------------------------ numerics shortcuts
@pytest.mark.parametrize("which", [0, 1, 2, 3, 4])
def test_device_selftest(L, which):
    """The FMA-corrected reciprocals equal IEEE division on [1, 2^126); the scalar sigmoid
    equals 1/(1+exp_c(-x)); the paired vector sigmoid equals it wherever the result is a
    normal number; both conversion-free round-half-away forms equal the reference for every
    float with |v| < 2^22."""
    assert L.tern_selftest(which) == 0


# ------------------------------------------------------------------------ a1 pack
@pytest.mark.parametrize("n,k,n_seg", [(64, 128, 1), (48, 40, 1), (256, 256, 3), (688, 256, 2),
                                       (1024, 2816, 1), (100, 1008, 3)])
def test_pack_parity(L, M, n, k, n_seg):
    lats = [latents(n, k, 100 + s) for s in range(n_seg)]
    pw = M.PackedWeight([x.cuda() for x in lats])
    codes = pw.codes.cpu().numpy().view(np.uint32)
    scales = pw.scales.cpu().numpy()
    for s, W in enumerate(lats):
        t_ref, m_ref = O.ternarize(W.numpy())
        assert abs(float(scales[s]) - float(m_ref)) <= np.spacing(np.float32(m_ref)), "scale"
        t_gpu = O.unpack_segment(codes, n, k, n_seg=n_seg, s=s)
        if scales[s] == m_ref:
            assert np.array_equal(t_gpu, t_ref)
        # with the oracle's scale forced, codes are bit-exact unconditionally
        pw2 = M.PackedWeight([W.cuda()], scales_in=[torch.tensor([float(m_ref)]).cuda()])
        t2 = O.unpack_segment(pw2.codes.cpu().numpy().view(np.uint32), n, k)
        assert np.array_equal(t2, t_ref)
    # K padding words hold the zero trit
    if pw.ldw * 16 > k:
        full = O.unpack_segment(codes, n, pw.ldw * 16, n_seg=n_seg, s=0)
        assert np.all(full[:, k:] == 0)


def test_pack_degenerate(L, M):
    with pytest.raises(L.TernError) as e:
        M.PackedWeight([torch.zeros(64, 128, device="cuda")])
    assert e.value.status == L.TERN_ERR_DEGENERATE


# ------------------------------------------------------------------------ a2 quant
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("m,k", [(1, 256), (7, 688), (33, 1024), (5, 2816), (3, 6912), (300, 256), (300, 2048), (260, 2560)])
def test_quant_parity(L, m, k, dtype):
    x = acts((m, k), 7 + k, dtype)
    x[0, :] = 0                       # all-zero row (C7)
    if m > 2:
        x[1, :] = 1.5                 # constant row
        x[2, : k // 2] *= 1000.0      # large dynamic range
    xd = x.cuda()
    kp = (k + 127) // 128 * 128
    q = torch.full((m, kp), 99, dtype=torch.int8, device="cuda")
    deq = torch.empty(m, device="cuda")
    qsum = torch.empty(m, dtype=torch.int32, device="cuda")
    r = torch.empty(m, device="cuda")
    a = torch.empty(m, device="cuda")
    L.tern_quant(xd, q, deq, qsum, inv_rms=r, absmax=a)
    torch.cuda.synchronize()
    qo, do, ro, ao = O.quant_rows(f32np(x))
    r_g = r.cpu().numpy()
    # inv_rms: within one ulp of the oracle's (fp64 sum order), normally identical
    assert np.all(np.abs(r_g - ro) <= np.spacing(ro))
    same = r_g == ro
    assert same.mean() > 0.99
    qg = q.cpu().numpy()
    assert np.all(qg[:, k:] == 0)
    assert np.array_equal(qg[same, :k], qo[same])
    assert np.array_equal(deq.cpu().numpy()[same], do[same])
    assert np.array_equal(a.cpu().numpy()[same], ao[same])
    assert np.array_equal(qsum.cpu().numpy(), qg[:, :k].astype(np.int64).sum(1))


# ------------------------------------------------------------------------ a3/a4 contraction
@pytest.mark.parametrize("m,n,k,n_seg", [(1, 256, 128, 1), (130, 640, 384, 1),
                                         (300, 1100, 1008, 1), (129, 256, 256, 3),
                                         (257, 688, 256, 2), (64, 5632, 2048, 1)])
def test_contract_gemm_exact(L, M, m, n, k, n_seg):
    rng = np.random.default_rng(m * 7 + n)
    lats = [latents(n, k, 200 + s) for s in range(n_seg)]
    pw = M.PackedWeight([x.cuda() for x in lats])
    kp = (k + 127) // 128 * 128
    qn = rng.integers(-128, 128, size=(m, kp), dtype=np.int8)
    qn[:, k:] = 0
    q = torch.from_numpy(qn).cuda()
    qsum = torch.from_numpy(qn.astype(np.int32).sum(1).astype(np.int32)).cuda()
    acc = torch.full((m, pw.n_rows), -7, dtype=torch.int32, device="cuda")
    L.tern_contract(q, qsum, pw.struct, acc)
    torch.cuda.synchronize()
    accg = acc.cpu().numpy()
    codes = pw.codes.cpu().numpy().view(np.uint32)
    for s, W in enumerate(lats):
        t = O.unpack_segment(codes, n, k, n_seg=n_seg, s=s)
        ref = O.tern_matmul(qn[:, :k], t)
        rows = [O.packed_row(s, r, n_seg, 64) for r in range(n)]
        assert np.array_equal(accg[:, rows], ref), f"segment {s}"


@pytest.mark.parametrize("xdt,ydt", [(torch.float32, torch.float32),
                                     (torch.bfloat16, torch.bfloat16),
                                     (torch.bfloat16, torch.float32)])
@pytest.mark.parametrize("k,n", [(256, 256), (1024, 1024), (688, 256), (2816, 1024)])
@pytest.mark.parametrize("m,force_gemm", [(1, False), (2, False), (3, False), (8, False),
                                          (16, False), (130, False), (1, True), (2, True),
                                          (3, True), (8, True)])
def test_bitlinear_parity(L, M, m, k, n, xdt, ydt, force_gemm):
    """m <= 4 runs the decode GEMV unless force_gemm; larger m (and force_gemm) the
    quant + tcgen05 GEMM path (split-K for few tiles)."""
    W = latents(n, k, 300 + k)
    pw = M.PackedWeight([W.cuda()])
    t, mw = O.ternarize(W.numpy())
    x = acts((m, k), 11 + m, "bf16" if xdt == torch.bfloat16 else "f32")
    bias = torch.randn(n, generator=synth.generator(5)) if m % 2 else None
    y = torch.empty((m, n), dtype=ydt, device="cuda")
    kp = (k + 127) // 128 * 128
    taps = {"q": torch.empty((m, kp), dtype=torch.int8, device="cuda"),
            "acc": torch.empty((m, pw.n_rows), dtype=torch.int32, device="cuda"),
            "deq": torch.empty(m, device="cuda"), "inv_rms": torch.empty(m, device="cuda"),
            "absmax": torch.empty(m, device="cuda")}
    old = L.tern_get_gemv_max_m()
    try:
        if force_gemm:
            L.tern_set_gemv_max_m(0)
        L.bitlinear_fwd(x.cuda(), pw.struct, y, bias=None if bias is None else bias.cuda(), taps=taps)
        torch.cuda.synchronize()
    finally:
        L.tern_set_gemv_max_m(old)
    assert float(pw.scales[0]) == float(mw)
    xo = f32np(x)
    out_o, tp = O.bitlinear(xo, t, mw, bias=None if bias is None else bias.numpy(),
                            bf16=(ydt == torch.bfloat16), taps=True)
    qg = taps["q"].cpu().numpy()[:, :k]
    # teacher forcing: the oracle accumulates the GPU's own int8 activations
    assert np.array_equal(taps["acc"].cpu().numpy(), O.tern_matmul(qg, t))
    # free running: identical quantization and accumulators, outputs bit-exact
    assert np.array_equal(qg, tp["q"])
    assert np.array_equal(taps["acc"].cpu().numpy(), tp["acc"])
    assert np.array_equal(taps["deq"].cpu().numpy(), tp["deq"])
    close(f32np(y), out_o, TOL[ydt], "y")
    assert np.array_equal(f32np(y), out_o)


# ------------------------------------------------------------------------ a6 scan
def deinterleave(fcg, d):
    Mx = fcg.shape[0]
    v = fcg.reshape(Mx, d // 64, 3, 64)
    return [v[:, :, s, :].reshape(Mx, d) for s in range(3)]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("B,T,d", [(1, 1, 64), (2, 5, 128), (2, 64, 256), (3, 130, 64),
                                   (1, 300, 1024)])
@pytest.mark.parametrize("gate", [0, 1])
def test_scan_parity(L, B, T, d, dtype, gate):
    g = synth.generator(B * 1000 + T)
    fcg = (torch.randn((B * T, 3 * d), generator=g) * 2).to(dtype)
    h0 = torch.randn((B, d), generator=g)
    h = h0.clone().cuda()
    op = torch.empty((B * T, d), dtype=dtype, device="cuda")
    L.tern_mlgru_scan(fcg.cuda(), B, T, d, h, op, gate=gate)
    torch.cuda.synchronize()
    fh, ch, gh = (a.reshape(B, T, d) for a in deinterleave(f32np(fcg), d))
    o_ref, h_ref = O.mlgru_scan(fh, ch, gh, h0.numpy(), gate_mode=gate,
                                bf16=(dtype == torch.bfloat16))
    assert np.array_equal(h.cpu().numpy(), h_ref)
    assert np.array_equal(f32np(op).reshape(B, T, d), o_ref)


# ------------------------------------------------------------------------ mixers + block
def _blocks(cfg, M, n_blocks, gate, gen_device="cpu"):
    st = M.Stack.random(cfg, gate=gate, n_blocks=n_blocks, gen_device=gen_device,
                        keep_latents=n_blocks)
    oblocks = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l)
               for lat in st.latents]
    return st, oblocks


@pytest.mark.parametrize("gate", [0, 1])
def test_c0_block_prefill_then_decode(L, M, gate):
    """BASELINE configs[0]: one block, fp32, d=256, l=688, batch 2 x 128, then 16 decode steps."""
    cfg = synth.CONFIGS["c0"]
    st, ob = _blocks(cfg, M, 1, gate)
    B, T, n = cfg.prefill_B, cfg.prefill_T, cfg.decode_steps
    x = synth.hidden((B, T + n, cfg.d), st.generator, cfg.dtype)   # drawn after the weights
    xd = x.cuda()
    states = st.new_state(B)
    y = st.prefill(xd[:, :T].contiguous(), states)
    ys = [y]
    for t in range(T, T + n):
        ys.append(st.decode(xd[:, t].contiguous(), states).unsqueeze(1))
    torch.cuda.synchronize()
    yg = f32np(torch.cat(ys, 1))
    H = np.zeros((B, cfg.d), np.float32)
    yo, Ho = O.block(ob[0], x.numpy()[:, :T], H, gate_mode=gate)
    outs = [yo]
    for t in range(T, T + n):
        yt, Ho = O.block(ob[0], x.numpy()[:, t:t + 1], Ho, gate_mode=gate)
        outs.append(yt)
    yo = np.concatenate(outs, 1)
    close(yg, yo, 1e-4, "y")
    close(states[0].cpu().numpy(), Ho, 1e-4, "h")
    assert np.array_equal(yg, yo), "free-running c0 expected bit-exact"
    assert np.array_equal(states[0].cpu().numpy(), Ho)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_mlgru_and_glu_fwd(L, M, dtype):
    cfg = synth.Config("t", 1, 256, 688, dtype, 9, 2, 70, 2, 0)
    st, ob = _blocks(cfg, M, 1, 0)
    blk = st.blocks[0]
    tdt = synth.torch_dtype(dtype)
    x = synth.hidden((2, 70, 256), synth.generator(3), dtype)
    ws = torch.empty(blk.workspace_bytes(2, 70, tdt), dtype=torch.uint8, device="cuda")
    h = torch.zeros((2, 256), device="cuda")
    out = torch.empty((2, 70, 256), dtype=tdt, device="cuda")
    L.mlgru_fwd(blk.mix, x.cuda(), out, h, ws)
    g_out = torch.empty((140, 256), dtype=tdt, device="cuda")
    L.glu_fwd(blk.ch, x.cuda().reshape(140, 256), g_out, 688, ws)
    torch.cuda.synchronize()
    bf = dtype == "bf16"
    o_ref, h_ref = O.mlgru(ob[0], f32np(x), np.zeros((2, 256), np.float32), bf16=bf)
    assert np.array_equal(f32np(out), o_ref)
    assert np.array_equal(h.cpu().numpy(), h_ref)
    g_ref = O.glu(ob[0], f32np(x).reshape(140, 256), bf16=bf)
    assert np.array_equal(f32np(g_out), g_ref)


@pytest.mark.parametrize("cfg_name,n_blocks,T,n_dec", [("c2", 2, 64, 4), ("c3", 1, 16, 2),
                                                       ("c4", 1, 8, 2)])
def test_stack_truncated_parity(L, M, cfg_name, n_blocks, T, n_dec):
    """Configs 2-4 truncated (first blocks, a few tokens, a few decode steps)."""
    cfg = synth.CONFIGS[cfg_name]
    st, ob = _blocks(cfg, M, n_blocks, 0, gen_device="cuda")
    B = 1
    x = synth.hidden((B, T + n_dec, cfg.d), synth.generator(cfg.seed + 1000), cfg.dtype)
    xd = x.cuda()
    states = st.new_state(B)
    ys = [st.prefill(xd[:, :T].contiguous(), states)]
    for t in range(T, T + n_dec):
        ys.append(st.decode(xd[:, t].contiguous(), states).unsqueeze(1))
    torch.cuda.synchronize()
    yg = f32np(torch.cat(ys, 1))
    bf = cfg.dtype == "bf16"
    Hs = [np.zeros((B, cfg.d), np.float32) for _ in ob]
    xo = f32np(x)
    y0, Hs = O.stack(ob, xo[:, :T], Hs, bf16=bf)
    outs = [y0]
    for t in range(T, T + n_dec):
        yt, Hs = O.stack(ob, xo[:, t:t + 1], Hs, bf16=bf)
        outs.append(yt)
    yo = np.concatenate(outs, 1)
    close(yg, yo, 2e-2 if bf else 1e-4, cfg_name)
    assert np.array_equal(yg, yo)


@pytest.mark.parametrize("m,k,n", [(4096, 2048, 5632), (4096, 5632, 2048), (16384, 1024, 1024)])
def test_sampled_full_size_bitlinear_c1(L, M, m, k, n):
    """configs[1] at full-size points (bf16) checked on sampled rows the oracle computes one
    by one: both GLU-shaped matrices at M = 4096 and the (1024,1024) one at M = 16384."""
    W = latents(n, k, 1)
    pw = M.PackedWeight([W.cuda()])
    t, mw = O.ternarize(W.numpy())
    x = acts((m, k), 1, "bf16")
    y = torch.empty((m, n), dtype=torch.bfloat16, device="cuda")
    L.bitlinear_fwd(x.cuda(), pw.struct, y)
    torch.cuda.synchronize()
    rows = np.random.default_rng(0).choice(m, 24, replace=False)
    rows = np.concatenate([rows, [0, m - 1]])
    ref = O.bitlinear(f32np(x)[rows], t, mw, bf16=True)
    assert np.array_equal(f32np(y)[rows], ref)


# ------------------------------------------------------------------------ fused a4 + a6
@pytest.mark.parametrize("dtype,B,T,d,gate", [("f32", 2, 128, 256, 0), ("f32", 3, 200, 128, 1),
                                              ("bf16", 2, 300, 192, 0), ("bf16", 1, 77, 64, 1)])
def test_fused_fcg_scan_equals_unfused(L, M, dtype, B, T, d, gate):
    """k_fcgscan (f|c|g GEMM with the scan in its epilogue) reproduces GEMM + scan bit for bit,
    including ragged sequence lengths (T not a multiple of the 128-token tile) and both gates;
    the unfused path is itself oracle-checked above."""
    cfg = synth.Config("fz", 1, d, 128, dtype, 17, B, T, 1, 0)
    st = M.Stack.random(cfg, gate=gate, gen_device="cpu")
    x = synth.hidden((B, T, d), synth.generator(4), dtype).cuda()
    outs = []
    old = L.tern_get_fused_scan()
    for fused in (True, False):
        L.tern_set_fused_scan(fused)
        try:
            h = st.new_state(B)
            y = st.prefill(x, h)
            torch.cuda.synchronize()
            outs.append((y.clone(), h[0].clone()))
        finally:
            L.tern_set_fused_scan(old)
    assert torch.equal(outs[0][0], outs[1][0]), "y differs"
    assert torch.equal(outs[0][1], outs[1][1]), "h differs"


# ------------------------------------------------------------------------ batched decode (split-K)
@pytest.mark.parametrize("cfg_name,B,T,n_dec", [("c2", 32, 3, 2), ("c4", 16, 2, 2), ("c3", 64, 1, 2),
                                               ("c4", 128, 1, 2)])
@pytest.mark.parametrize("fin,sab", [(False, False), (True, False), (False, True), (True, True)])
def test_batched_decode_split_k_parity(L, M, cfg_name, B, T, n_dec, fin, sab):
    """Decode batches above the GEMV limit: per BitLinear a split-K tcgen05 GEMM (int32
    slices) and a row-wise finalize that applies the epilogue and quantizes the row for the
    next BitLinear (k_fin.cu); short prefills take quant + GEMM + split-K epilogue.
    Free-running against the oracle, bit-exact."""
    cfg = synth.CONFIGS[cfg_name]
    st, ob = _blocks(cfg, M, 1, 0, gen_device="cuda")
    x = synth.hidden((B, T + n_dec, cfg.d), synth.generator(cfg.seed + 77), cfg.dtype)
    xd = x.cuda()
    states = st.new_state(B)
    old, old_sab = L.tern_get_batched_fin(), L.tern_get_gemm_sab()
    try:
        L.tern_set_batched_fin(fin)
        L.tern_set_gemm_sab(sab)   # swap-AB small-M kernel (k_gemm_sab.cu, opt-in)
        ys = [st.prefill(xd[:, :T].contiguous(), states)]
        for t in range(T, T + n_dec):
            ys.append(st.decode(xd[:, t].contiguous(), states).unsqueeze(1))
        torch.cuda.synchronize()
    finally:
        L.tern_set_batched_fin(old)
        L.tern_set_gemm_sab(old_sab)
    yg = f32np(torch.cat(ys, 1))
    bf = cfg.dtype == "bf16"
    H = [np.zeros((B, cfg.d), np.float32)]
    xo = f32np(x)
    y0, H = O.stack(ob, xo[:, :T], H, bf16=bf)
    outs = [y0]
    for t in range(T, T + n_dec):
        yt, H = O.stack(ob, xo[:, t:t + 1], H, bf16=bf)
        outs.append(yt)
    yo = np.concatenate(outs, 1)
    close(yg, yo, 2e-2 if bf else 1e-4, cfg_name)
    assert np.array_equal(yg, yo)
    assert np.array_equal(states[0].cpu().numpy(), H[0])


# ------------------------------------------------------------------------ full size, bench launch config
@pytest.mark.parametrize("cfg_name,n_tok", [("c2", 24), ("c3", 8), ("c4", 8)])
def test_full_size_prefill_sampled_prefixes(L, M, cfg_name, n_tok):
    """The bench workload at full size and in bench.py's launch configuration (all blocks,
    B x T prefill, fused f|c|g+scan, tcgen05 GEMMs): the MLGRU is causal, so the first
    n_tok outputs of a sequence depend only on its first n_tok inputs -- the oracle computes
    those prefixes through the whole stack and they must match bit for bit (sampled
    sequences: first, a middle one, last)."""
    cfg = synth.CONFIGS[cfg_name]
    st = M.Stack.random(cfg, device="cuda", gen_device="cuda", keep_latents=cfg.L)
    B, T = cfg.prefill_B, cfg.prefill_T
    x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 7919), cfg.dtype).cuda()
    states = st.new_state(B)
    y = st.prefill(x, states)
    torch.cuda.synchronize()
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in st.latents]
    bf = cfg.dtype == "bf16"
    for b in (0, B // 2, B - 1):
        xo = f32np(x[b:b + 1, :n_tok])
        Hs = [np.zeros((1, cfg.d), np.float32) for _ in ob]
        yo, _ = O.stack(ob, xo, Hs, bf16=bf)
        yg = f32np(y[b:b + 1, :n_tok])
        close(yg, yo, 2e-2 if bf else 1e-4, f"{cfg_name} seq {b}")
        assert np.array_equal(yg, yo), f"{cfg_name} sequence {b}"


# ------------------------------------------------------------------------ edge cases
def test_zero_rows_and_empty_calls(L, M):
    """Degenerate inputs (C7): an all-zero activation row quantizes to q = 0 and yields the
    bias exactly on both contraction paths; empty batches are no-ops."""
    n, k = 256, 512
    W = latents(n, k, 71)
    pw = M.PackedWeight([W.cuda()])
    bias = torch.randn(n, generator=synth.generator(72))
    for m, force_gemm in ((3, False), (40, True)):
        x = acts((m, k), 73)
        x[1] = 0.0
        y = torch.empty((m, n), device="cuda")
        old = L.tern_get_gemv_max_m()
        try:
            if force_gemm:
                L.tern_set_gemv_max_m(0)
            L.bitlinear_fwd(x.cuda(), pw.struct, y, bias=bias.cuda())
            torch.cuda.synchronize()
        finally:
            L.tern_set_gemv_max_m(old)
        assert torch.equal(y[1].cpu(), bias), "zero row must give the bias"
        t, mw = O.ternarize(W.numpy())
        assert np.array_equal(f32np(y), O.bitlinear(f32np(x), t, mw, bias=bias.numpy()))
    # empty batches: nothing launched, nothing written, OK status
    cfg = synth.Config("e", 1, 128, 256, "f32", 74, 1, 4, 1, 0)
    st = M.Stack.random(cfg, gen_device="cpu")
    x0 = torch.empty((0, 4, 128), device="cuda")
    h0 = st.new_state(0)
    y0 = st.prefill(x0, h0)
    assert y0.shape == (0, 4, 128)


@pytest.mark.parametrize("cfg_name,n_tok", [("c2", 300), ("c3", 260)])
def test_full_size_fused_scan_crosses_time_tiles(L, M, cfg_name, n_tok):
    """k_fcgscan at the bench's launch configuration (full B x T prefill, full width d, the
    fused f|c|g GEMM + scan path, asserted from the launch records) through 2 blocks,
    against the oracle on the first n_tok > 256 tokens of sampled sequences: the prefix
    crosses two 128-token time tiles, so the carry hand-off between tiles (mbarriers, the
    h carried in registers) is checked against the definition, not against CUDA."""
    cfg = synth.CONFIGS[cfg_name]
    st = M.Stack.random(cfg, device="cuda", gen_device="cuda", keep_latents=2, n_blocks=2)
    B, T = cfg.prefill_B, cfg.prefill_T
    x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 7919), cfg.dtype).cuda()
    states = st.new_state(B)
    L.tern_profile_enable(True)
    try:
        y = st.prefill(x, states)
        torch.cuda.synchronize()
    finally:
        L.tern_profile_enable(False)
    kernels = {r["kernel"] for r in L.tern_profile_collect()}
    assert "fcgscan" in kernels, f"fused scan not launched: {kernels}"
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in st.latents]
    bf = cfg.dtype == "bf16"
    for b in (0, B - 1):
        xo = f32np(x[b:b + 1, :n_tok])
        Hs = [np.zeros((1, cfg.d), np.float32) for _ in ob]
        yo, Hs = O.stack(ob, xo, Hs, bf16=bf)
        yg = f32np(y[b:b + 1, :n_tok])
        close(yg, yo, 2e-2 if bf else 1e-4, f"{cfg_name} seq {b}")
        assert np.array_equal(yg, yo), f"{cfg_name} sequence {b}"


def test_c2_decode_through_all_blocks(L, M):
    """8 decode steps of the c2 stack (all 24 blocks, B = 1, the GEMV path in the
    bench's CUDA graph) after a short prefill, free-running against the oracle; the
    per-block states after the last step too."""
    cfg = synth.CONFIGS["c2"]
    st = M.Stack.random(cfg, device="cuda", gen_device="cuda", keep_latents=cfg.L)
    T, n_dec = 4, 8
    x = synth.hidden((1, T + n_dec, cfg.d), synth.generator(cfg.seed + 31), cfg.dtype)
    xd = x.cuda()
    states = st.new_state(1)
    st.prefill(xd[:, :T].contiguous(), states)
    g, xin, yout = st.capture_decode(1, states)
    ys = []
    for t in range(T, T + n_dec):
        xin.copy_(xd[:, t])
        g.replay()
        ys.append(yout.clone().unsqueeze(1))
    torch.cuda.synchronize()
    yg = f32np(torch.cat(ys, 1))
    ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l) for lat in st.latents]
    Hs = [np.zeros((1, cfg.d), np.float32) for _ in ob]
    xo = f32np(x)
    _, Hs = O.stack(ob, xo[:, :T], Hs)
    outs = []
    for t in range(T, T + n_dec):
        yt, Hs = O.stack(ob, xo[:, t:t + 1], Hs)
        outs.append(yt)
    yo = np.concatenate(outs, 1)
    close(yg, yo, 1e-4, "c2 decode")
    assert np.array_equal(yg, yo)
    for i in range(cfg.L):
        assert np.array_equal(states[i].cpu().numpy(), Hs[i]), f"block {i} state"


@pytest.mark.parametrize("m,k,n,dtype", [(300, 2048, 192, "f32"), (1000, 2304, 1088, "bf16"),
                                         (257, 4096, 256, "f32")])
def test_two_sm_gemm_parity(L, M, m, k, n, dtype):
    """The CTA-pair GEMM (k_gemm_2sm: tcgen05.mma.cta_group::2, 256 x 256 tiles, both CTAs'
    TMA loads completing on the leader's barrier, multicast commits) against the oracle,
    with ragged M (not a multiple of 256), N below / not a multiple of 256 (the second CTA's
    B half partly or wholly beyond the matrix) and K of 16..32 k-blocks."""
    old = L.tern_get_gemm_2sm()
    L.tern_set_gemm_2sm(True)
    try:
        W = latents(n, k, m)
        pw = M.PackedWeight([W.cuda()])
        t, mw = O.ternarize(W.numpy())
        x = acts((m, k), m + 1, dtype)
        y = torch.empty((m, n), dtype=synth.torch_dtype(dtype), device="cuda")
        L.bitlinear_fwd(x.cuda(), pw.struct, y)
        torch.cuda.synchronize()
        assert np.array_equal(f32np(y), O.bitlinear(f32np(x), t, mw, bf16=dtype == "bf16"))
    finally:
        L.tern_set_gemm_2sm(old)


@pytest.mark.parametrize("dtype,B,T,d,l", [("f32", 3, 200, 512, 2176), ("bf16", 2, 300, 2048, 704)])
def test_two_sm_gemm_block_epilogues(L, M, dtype, B, T, d, l):
    """The CTA-pair GEMM's residual (down, K = l > 2048) and SwiGLU (gate|up, K = d = 2048)
    epilogues inside a block prefill, free-running against the oracle block."""
    old = L.tern_get_gemm_2sm()
    L.tern_set_gemm_2sm(True)
    try:
        cfg = synth.Config("p2", 1, d, l, dtype, 19, B, T, B, 0)
        st = M.Stack.random(cfg, gen_device="cpu", keep_latents=1)
        x = synth.hidden((B, T, d), synth.generator(d + l), dtype)
        h = st.new_state(B)
        y = st.prefill(x.cuda(), h)
        torch.cuda.synchronize()
        ob = O.OracleBlock({kk: v.numpy() for kk, v in st.latents[0].items()}, d, l)
        yo, ho = O.block(ob, f32np(x), np.zeros((B, d), np.float32), bf16=dtype == "bf16")
        assert np.array_equal(f32np(y), yo)
        assert np.array_equal(h[0].cpu().numpy(), ho)
    finally:
        L.tern_set_gemm_2sm(old)


# ------------------------------------------------------------------------ f3: fused quantization
@pytest.mark.parametrize("dtype,B,T,d,l", [("f32", 3, 200, 512, 2176), ("bf16", 2, 300, 2048, 704),
                                           ("f32", 1, 1000, 1024, 2816)])
def test_qfuse_block_prefill(L, M, dtype, B, T, d, l):
    """SURVEY 8(f) f3, the a2 RMSNorm + quantization fused into the o, gate|up and down GEMMs
    (tern_set_qfuse; k_gemm.cu "fused quantization"): a block prefill with ragged M (not a
    multiple of 128), 1-CTA and CTA-pair GEMMs, fp32 and bf16, free-running against the oracle
    block, bit for bit."""
    old = L.tern_get_qfuse()
    L.tern_set_qfuse(True)
    try:
        cfg = synth.Config("qf", 1, d, l, dtype, 23, B, T, B, 0)
        st = M.Stack.random(cfg, gen_device="cpu", keep_latents=1)
        x = synth.hidden((B, T, d), synth.generator(d + l + 1), dtype)
        h = st.new_state(B)
        y = st.prefill(x.cuda(), h)
        torch.cuda.synchronize()
        ob = O.OracleBlock({kk: v.numpy() for kk, v in st.latents[0].items()}, d, l)
        yo, ho = O.block(ob, f32np(x), np.zeros((B, d), np.float32), bf16=dtype == "bf16")
        close(f32np(y), yo, 2e-2 if dtype == "bf16" else 1e-4, "qfuse block")
        assert np.array_equal(f32np(y), yo)
        assert np.array_equal(h[0].cpu().numpy(), ho)
    finally:
        L.tern_set_qfuse(old)


@pytest.mark.parametrize("cfg_name,n_tok", [("c2", 24), ("c3", 8)])
def test_qfuse_full_size_prefixes(L, M, cfg_name, n_tok):
    """The fused quantization at the bench workload's full size (all blocks, B x T), sampled
    sequence prefixes through the whole stack against the oracle."""
    old = L.tern_get_qfuse()
    L.tern_set_qfuse(True)
    try:
        cfg = synth.CONFIGS[cfg_name]
        st = M.Stack.random(cfg, device="cuda", gen_device="cuda", keep_latents=cfg.L)
        B, T = cfg.prefill_B, cfg.prefill_T
        x = synth.hidden((B, T, cfg.d), synth.generator(cfg.seed + 7919), cfg.dtype).cuda()
        states = st.new_state(B)
        y = st.prefill(x, states)
        torch.cuda.synchronize()
        ob = [O.OracleBlock({k: v.numpy() for k, v in lat.items()}, cfg.d, cfg.l)
              for lat in st.latents]
        bf = cfg.dtype == "bf16"
        for b in (0, B - 1):
            xo = f32np(x[b:b + 1, :n_tok])
            Hs = [np.zeros((1, cfg.d), np.float32) for _ in ob]
            yo, _ = O.stack(ob, xo, Hs, bf16=bf)
            yg = f32np(y[b:b + 1, :n_tok])
            assert np.array_equal(yg, yo), f"{cfg_name} sequence {b}"
    finally:
        L.tern_set_qfuse(old)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_qfuse_with_gains_and_biases(L, M, dtype):
    """QFuse with per-feature norm gains (the fused quantizer's max|x r w| pass) and biases,
    1 block of 2 x 300 tokens, against the oracle block."""
    d, l, B, T = 512, 1408, 2, 300
    g = synth.generator(77)
    lat = synth.latent_block(d, l, g)
    gg = synth.generator(78)
    gains = {k: (1.0 + 0.25 * torch.randn(n, generator=gg)).cuda()
             for k, n in (("x", d), ("o", d), ("x1", d), ("p", l))}
    biases = {k: (0.05 * torch.randn(d, generator=gg)).cuda() for k in ("f", "c", "g", "o")}
    blk = M.Block(lat, d, l, gains=gains, biases=biases)
    st = M.Stack([blk], d, l, synth.torch_dtype(dtype))
    ob = O.OracleBlock({k: v.numpy() for k, v in lat.items()}, d, l,
                       gains={k: v.cpu().numpy() for k, v in gains.items()},
                       biases={k: v.cpu().numpy() for k, v in biases.items()})
    x = synth.hidden((B, T, d), synth.generator(79), dtype)
    old = L.tern_get_qfuse()
    L.tern_set_qfuse(True)
    try:
        h = st.new_state(B)
        y = st.prefill(x.cuda(), h)
        torch.cuda.synchronize()
    finally:
        L.tern_set_qfuse(old)
    yo, ho = O.block(ob, f32np(x), np.zeros((B, d), np.float32), bf16=dtype == "bf16")
    close(f32np(y), yo, 2e-2 if dtype == "bf16" else 1e-4, "qfuse gains")
    assert np.array_equal(f32np(y), yo)


@pytest.mark.parametrize("l", [1408, 2176])
def test_inplace_channel_residual(L, M, l):
    """fp32 block prefill with more than 256 tokens writes x1 into y and adds the down
    projection onto it in place (EPI_RESID_RED, TMA reduce-add): the 1-CTA GEMM (l = 1408 <
    2048) and the CTA-pair GEMM (l = 2176), ragged M = 3 x 230, against the oracle block."""
    d, B, T = 512, 3, 230
    cfg = synth.Config("red", 1, d, l, "f32", 29, B, T, B, 0)
    st = M.Stack.random(cfg, gen_device="cpu", keep_latents=1)
    x = synth.hidden((B, T, d), synth.generator(d + l + 7), "f32")
    h = st.new_state(B)
    y = st.prefill(x.cuda(), h)
    torch.cuda.synchronize()
    ob = O.OracleBlock({kk: v.numpy() for kk, v in st.latents[0].items()}, d, l)
    yo, ho = O.block(ob, f32np(x), np.zeros((B, d), np.float32))
    assert np.array_equal(f32np(y), yo)
    assert np.array_equal(h[0].cpu().numpy(), ho)
