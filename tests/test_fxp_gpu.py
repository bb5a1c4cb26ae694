"""Fixed-point W8A16 numerics (readings
F1-F5 in DESIGN.md §3b) through the C ABI, element by element against the oracle
(tests/test_fxp_oracle.py pins the oracle).  Everything is integer: bit-exact is the bar.
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


@pytest.mark.parametrize("n", [1, 7, 256, 1000, 6912])
@pytest.mark.parametrize("scale", [1e-3, 0.02, 1.0, 300.0])
@pytest.mark.parametrize("shift", [0, 6])
def test_scales(L, n, scale, shift):
    w = scale * (1.0 + 0.3 * torch.randn(n, generator=synth.generator(n + shift)))
    wq, e = L.tern_fxp_scales(w.cuda(), shift)
    wq_o, e_o = O.fxp_scales(w.numpy(), shift)
    assert e == e_o and np.array_equal(wq.cpu().numpy(), wq_o)


def test_scales_degenerate(L):
    with pytest.raises(L.TernError) as ei:
        L.tern_fxp_scales(torch.zeros(9, device="cuda"))
    assert ei.value.status == L.TERN_ERR_DEGENERATE


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape,scale", [((1,), 1.0), ((3, 5), 1e-4), ((37, 1000), 3e3),
                                         ((16384, 1024), 1.0)])
def test_quant_act(L, dtype, shape, scale):
    x = synth.hidden(shape, synth.generator(len(shape) * 31 + shape[-1]), "f32") * scale
    xt = x.to(torch.bfloat16) if dtype == "bf16" else x
    q = torch.full(shape, 77, dtype=torch.int16, device="cuda")
    e = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    L.tern_fxp_quant_act(xt.cuda(), q, e)
    q_o, e_o = O.fxp_quant_act(xt.float().numpy())
    assert int(e.item()) == e_o
    assert np.array_equal(q.cpu().numpy(), q_o)


def test_quant_act_zero_and_exact(L):
    for x in (torch.zeros(10), torch.tensor([32767.0, -1.0, 0.4, 0.5, -0.5, 1.5])):
        q = torch.empty(x.shape, dtype=torch.int16, device="cuda")
        e = torch.empty(1, dtype=torch.int32, device="cuda")
        L.tern_fxp_quant_act(x.cuda(), q, e)
        q_o, e_o = O.fxp_quant_act(x.numpy())
        assert int(e.item()) == e_o and np.array_equal(q.cpu().numpy(), q_o)


def test_sigmoid_exhaustive(L):
    """Every Q6 input in [-2^20, 2^20] plus the int32 extremes, a ragged length."""
    x = np.concatenate([np.arange(-(1 << 20), (1 << 20) + 1, dtype=np.int64),
                        [-(1 << 31), -(1 << 31) + 1, (1 << 31) - 1, 511, 512, 513, -512]])
    x = x.astype(np.int32)
    xt = torch.from_numpy(x).cuda()
    y = torch.empty_like(xt)
    L.tern_fxp_sigmoid(xt, y)
    assert np.array_equal(y.cpu().numpy(), O.fxp_sigmoid(x))
    assert y[(1 << 20)].item() == 1 << 14        # sigma_fxp(0) = 2^(y_exp - 1)


def test_inv_sqrt(L):
    rng = np.random.default_rng(11)
    v = np.concatenate([np.arange(1, 20001, dtype=np.uint64),
                        rng.integers(1, np.iinfo(np.uint64).max, 200001, dtype=np.uint64,
                                     endpoint=True),
                        (np.uint64(1) << np.arange(64, dtype=np.uint64)),
                        np.array([np.iinfo(np.uint64).max], np.uint64)])
    e = rng.integers(-100, 100, v.size).astype(np.int32)
    vt = torch.from_numpy(v.view(np.int64)).cuda()
    et = torch.from_numpy(e).cuda()
    y = torch.empty(v.size, dtype=torch.int32, device="cuda")
    ey = torch.empty(v.size, dtype=torch.int32, device="cuda")
    L.tern_fxp_inv_sqrt(vt, et, y, ey)
    y_o, ey_o = O.fxp_inv_sqrt(v, e)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), y_o)
    assert np.array_equal(ey.cpu().numpy(), ey_o)


def test_inv_sqrt_zero_is_defined(L):
    vt = torch.tensor([0, 4], dtype=torch.int64, device="cuda")
    et = torch.zeros(2, dtype=torch.int32, device="cuda")
    y = torch.full((2,), 5, dtype=torch.int32, device="cuda")
    ey = torch.full((2,), 5, dtype=torch.int32, device="cuda")
    L.tern_fxp_inv_sqrt(vt, et, y, ey)
    assert y[0].item() == 0 and ey[0].item() == 0
    assert y[1].item() * 2.0 ** ey[1].item() == pytest.approx(0.5, rel=2 ** -29)


@pytest.mark.parametrize("rows,d", [(1, 64), (9, 1000), (33, 1024), (5, 2560), (17, 2816),
                                    (3, 6912), (2, 65536), (16384, 1024)])
def test_rmsnorm(L, rows, d):
    """Rows spanning 1e-2..1e2 of the tensor's scale (one exponent for the tensor), zero rows,
    non-unit gains; the c2-sized case [16384][1024] in full."""
    g = synth.generator(rows * 7 + d)
    x = synth.hidden((rows, d), g, "f32") * torch.logspace(-2, 2, rows)[:, None]
    if rows > 2:
        x[1] = 0.0
    w = 1.0 + 0.25 * torch.randn(d, generator=g)
    xq = torch.empty((rows, d), dtype=torch.int16, device="cuda")
    ex = torch.empty(1, dtype=torch.int32, device="cuda")
    L.tern_fxp_quant_act(x.cuda(), xq, ex)
    wq, ew = L.tern_fxp_scales(w.cuda())
    out = torch.full((rows, d), 123, dtype=torch.int16, device="cuda")
    eo = torch.full((rows,), 99, dtype=torch.int32, device="cuda")
    L.tern_fxp_rmsnorm(xq, ex, wq, ew, out, eo)
    xq_o, ex_o = O.fxp_quant_act(x.numpy())
    wq_o, ew_o = O.fxp_scales(w.numpy())
    assert int(ex.item()) == ex_o and ew == ew_o
    assert np.array_equal(xq.cpu().numpy(), xq_o) and np.array_equal(wq.cpu().numpy(), wq_o)
    out_o, eo_o = O.fxp_rmsnorm(xq_o, ex_o, wq_o, ew_o)
    assert np.array_equal(eo.cpu().numpy(), eo_o)
    assert np.array_equal(out.cpu().numpy(), out_o)


@pytest.mark.parametrize("eps", [1e-6, 1e-3])
def test_rmsnorm_eps_underflow(L, eps):
    """with large activations eps_q underflows to 0 at eps = 1e-6; an all-zero row then
    yields zeros with exponent 0 (no division by zero); 1e-3 keeps eps_q > 0 at ex = 0."""
    d = 512
    xq = torch.zeros((2, d), dtype=torch.int16, device="cuda")
    xq[1, :] = 1000
    ex = torch.tensor([0], dtype=torch.int32, device="cuda")
    wq = torch.full((d,), 64, dtype=torch.int8, device="cuda")
    out = torch.empty((2, d), dtype=torch.int16, device="cuda")
    eo = torch.empty(2, dtype=torch.int32, device="cuda")
    L.tern_fxp_rmsnorm(xq, ex, wq, -6, out, eo, eps=eps)
    out_o, eo_o = O.fxp_rmsnorm(xq.cpu().numpy(), 0, wq.cpu().numpy(), -6, eps=eps)
    assert np.array_equal(out.cpu().numpy(), out_o) and np.array_equal(eo.cpu().numpy(), eo_o)
    assert not out[0].any()


@pytest.mark.parametrize("scale,d", [(1e-9, 1024), (1e-12, 2560), (1e-12, 64)])
def test_rmsnorm_tiny_activations(L, scale, d):
    """Reading F5b: tiny activations put eps_q above 2^60, so both sides form the sum on the
    coarser even grid; both warp-per-row (d <= 3072, multiple of 256) and CTA-per-row kernels."""
    g = synth.generator(d + 5)
    x = synth.hidden((6, d), g, "f32") * scale
    w = 1.0 + 0.25 * torch.randn(d, generator=g)
    xq = torch.empty((6, d), dtype=torch.int16, device="cuda")
    ex = torch.empty(1, dtype=torch.int32, device="cuda")
    L.tern_fxp_quant_act(x.cuda(), xq, ex)
    wq, ew = L.tern_fxp_scales(w.cuda())
    out = torch.empty((6, d), dtype=torch.int16, device="cuda")
    eo = torch.empty(6, dtype=torch.int32, device="cuda")
    L.tern_fxp_rmsnorm(xq, ex, wq, ew, out, eo)
    xq_o, ex_o = O.fxp_quant_act(x.numpy())
    wq_o, ew_o = O.fxp_scales(w.numpy())
    assert round(d * 1e-3 * 2.0 ** (-2 * ex_o)) > 2.0 ** 60
    out_o, eo_o = O.fxp_rmsnorm(xq_o, ex_o, wq_o, ew_o)
    assert np.array_equal(eo.cpu().numpy(), eo_o)
    assert np.array_equal(out.cpu().numpy(), out_o)


@pytest.fixture(scope="module")
def M():
    from paper_2406_02528_b200 import model
    return model


@pytest.mark.parametrize("m,k,n", [(1, 64, 16), (1, 1024, 1024), (4, 1000, 300), (7, 688, 256),
                                   (130, 1024, 640), (300, 2816, 1024), (2048, 1024, 3072)])
def test_bitlinear_w8a16(L, M, m, k, n):
    """F6 through the C ABI: F5 norm, the int16 x ternary contraction as two s8 digit planes on
    the tcgen05 GEMM plus the ternary row sums, the pow2 int8 beta, per-row requantization --
    bit-exact against the oracle over ragged m / k / n (k not a multiple of 128, n not a
    multiple of the GEMM tile); rows span 1e-2..1e2 of the tensor scale, one zero row."""
    g = synth.generator(m * 13 + k + n)
    W = synth.latent_matrix(n, k, g)
    pw = M.PackedWeight([W.cuda()])
    t, beta = O.ternarize(W.numpy())
    x = synth.hidden((m, k), g, "f32") * torch.logspace(-2, 2, m)[:, None]
    if m > 2:
        x[2] = 0.0
    gain = 1.0 + 0.25 * torch.randn(k, generator=g)
    xq = torch.empty((m, k), dtype=torch.int16, device="cuda")
    ex = torch.empty(1, dtype=torch.int32, device="cuda")
    L.tern_fxp_quant_act(x.cuda(), xq, ex)
    gq, eg = L.tern_fxp_scales(gain.cuda())
    y = torch.full((m, n), 321, dtype=torch.int16, device="cuda")
    ey = torch.full((m,), 99, dtype=torch.int32, device="cuda")
    L.tern_fxp_bitlinear(xq, ex, gq, eg, pw.struct, y, ey)
    torch.cuda.synchronize()
    y_o, ey_o = O.fxp_bitlinear(xq.cpu().numpy(), int(ex.item()), gq.cpu().numpy(), eg, t, beta)
    assert np.array_equal(ey.cpu().numpy(), ey_o)
    assert np.array_equal(y.cpu().numpy(), y_o)


def test_bitlinear_w8a16_extreme_digits(L, M):
    """Inputs at the int16 extremes (-32768, 32767, -1, 255, 256): the normalised rows reach
    +-32767, exercising the digit split's ends (hi = -128 / 127, lo' = -128 / 127) and the
    128 sum_k t correction."""
    k, n, m = 256, 128, 3
    W = synth.latent_matrix(n, k, synth.generator(77))
    pw = M.PackedWeight([W.cuda()])
    t, beta = O.ternarize(W.numpy())
    vals = np.array([-32768, 32767, -1, 255, 256, -256, 0, 128], np.int16)
    xq_np = np.resize(vals, (m, k)).astype(np.int16)
    xq_np[1] = np.roll(xq_np[1], 3)
    xq = torch.from_numpy(xq_np).cuda()
    ex = torch.tensor([-12], dtype=torch.int32, device="cuda")
    gq = torch.full((k,), 64, dtype=torch.int8, device="cuda")
    y = torch.empty((m, n), dtype=torch.int16, device="cuda")
    ey = torch.empty((m,), dtype=torch.int32, device="cuda")
    L.tern_fxp_bitlinear(xq, ex, gq, -6, pw.struct, y, ey)
    y_o, ey_o = O.fxp_bitlinear(xq_np, -12, np.full(k, 64, np.int8), -6, t, beta)
    assert np.array_equal(y.cpu().numpy(), y_o) and np.array_equal(ey.cpu().numpy(), ey_o)
