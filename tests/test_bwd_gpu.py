"""GPU-vs-oracle parity of the Alg. 1 BackwardPass (
readings B1-B6), through the C ABI (bitlinear_bwd).

Tolerance: the GPU computes in fp32 with fp32 accumulation, the oracle in
fp64 on the same fp32 inputs.  A sum of N random-sign fp32 terms carries an absolute error
of about u sqrt(N/2) rms(result) (u = 2^-24) whatever the size of the particular element, so
the floor is the row's rms: |g - o| <= 1e-4 * max(|o|, rms(o_row)) elementwise (about 30x
the expected error at N = 16384)."""
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


def close(g, o, tol, what):
    g = np.asarray(g, np.float64)
    o = np.asarray(o, np.float64)
    o2 = o.reshape(-1, o.shape[-1]) if o.ndim > 1 else o.reshape(1, -1)
    rms = np.sqrt(np.mean(o2 ** 2, axis=1, keepdims=True)).repeat(o2.shape[1], 1).reshape(o.shape)
    lim = tol * np.maximum(np.abs(o), rms) + 1e-30
    bad = np.abs(g - o) > lim
    assert not bad.any(), f"{what}: {bad.sum()} / {bad.size} outside tol {tol}; " \
                          f"max abs err {np.max(np.abs(g - o)):.3e}"


@pytest.mark.parametrize("tc", [True, False])
@pytest.mark.parametrize("m,k,n,norm", [(37, 64, 48, 0), (37, 64, 48, 1), (300, 1024, 1000, 0),
                                        (513, 2816, 1024, 1), (2048, 1024, 1024, 0),
                                        (1000, 2048, 200, 0)])
def test_bwd_parity(L, M, m, k, n, norm, tc):
    """dX, dW and db against the oracle: ragged m and n (not tile multiples), both norms,
    contractions spanning several 128-wide tiles and k-blocks; the tensor-core path (bf16
    hi + lo split, B7, with split-K slices for dW) and the fp32 CUDA-core path."""
    old = L.tern_get_bwd_tc()
    L.tern_set_bwd_tc(tc)
    try:
        _bwd_case(L, M, m, k, n, norm)
    finally:
        L.tern_set_bwd_tc(old)


@pytest.mark.parametrize("m,k,n,norm", [(300, 2048, 1000, 0), (513, 5632, 2048, 1)])
def test_bwd_parity_bf16(L, M, m, k, n, norm):
    """bf16 inputs (the c3 / c4 activation dtype, widened exactly for the oracle) on the
    tensor-core path; the CUDA-core path rejects them."""
    _bwd_case(L, M, m, k, n, norm, "bf16")


def _bwd_case(L, M, m, k, n, norm, dtype="f32"):
    g = synth.generator(m + k + n + norm)
    W = synth.latent_matrix(n, k, g)
    x = synth.hidden((m, k), g, "f32") * 1.3 + 0.2
    dO = synth.hidden((m, n), g, "f32")
    if dtype == "bf16":
        x = x.to(torch.bfloat16).float()   # values exactly representable in both
        dO = dO.to(torch.bfloat16).float()
    pw = M.PackedWeight([W.cuda()])
    t, mw = O.ternarize(W.numpy())
    xd, dOd = x.cuda(), dO.cuda()
    if dtype == "bf16":
        xd, dOd = xd.to(torch.bfloat16), dOd.to(torch.bfloat16)
    dX = torch.empty((m, k), device="cuda")
    dW = torch.empty((n, k), device="cuda")
    db = torch.empty(n, device="cuda")
    L.bitlinear_bwd(xd, pw.struct, dOd, dX, dW, db, norm=norm)
    torch.cuda.synchronize()
    oX, oW, ob = O.bitlinear_bwd(x.numpy(), t, mw, dO.numpy(), norm=norm)
    close(dX.cpu().numpy(), oX, 1e-4, "dX")
    close(dW.cpu().numpy(), oW, 1e-4, "dW")
    close(db.cpu().numpy(), ob, 1e-4, "db")


def test_bwd_edge_cases(L, M):
    """No tokens: dW = 0 and db = 0; a weight without the u8 copy and a bad norm are
    rejected before any launch."""
    k, n = 128, 64
    W = synth.latent_matrix(n, k, synth.generator(5))
    pw = M.PackedWeight([W.cuda()])
    dW = torch.full((n, k), 7.0, device="cuda")
    db = torch.full((n,), 7.0, device="cuda")
    x = torch.empty((0, k), device="cuda")
    L.bitlinear_bwd(x, pw.struct, torch.empty((0, n), device="cuda"), torch.empty((0, k),
                    device="cuda"), dW, db)
    torch.cuda.synchronize()
    assert not dW.any() and not db.any()
    pw2 = M.PackedWeight([W.cuda()], expand=False)
    x = torch.randn(4, k, device="cuda")
    with pytest.raises(L.TernError):
        L.bitlinear_bwd(x, pw2.struct, torch.randn(4, n, device="cuda"),
                        torch.empty_like(x), dW, db)
    with pytest.raises(L.TernError):
        L.bitlinear_bwd(x, pw.struct, torch.randn(4, n, device="cuda"),
                        torch.empty_like(x), dW, db, norm=5)
    old = L.tern_get_bwd_tc()
    L.tern_set_bwd_tc(False)
    try:
        with pytest.raises(L.TernError):   # bf16 only on the tensor-core path
            L.bitlinear_bwd(x.to(torch.bfloat16), pw.struct,
                            torch.randn(4, n, device="cuda").to(torch.bfloat16),
                            torch.empty_like(x), dW, db)
    finally:
        L.tern_set_bwd_tc(old)
