"""Pins of the oracle's Alg. 1 BackwardPass (readings B1-B6 in DESIGN.md 3c)
against mathematics that does not go through the oracle's own backward code:

- dX equals central finite differences of the straight-through forward loss
  L(X) = sum dO * (norm(X) W~^T) (activation quantization passed straight through, B1),
  with the norm written from its textbook definition in float64 (both norm modes);
- dW and db equal finite differences of L = sum dO * (Y~ W~^T + b) in W~ and b, with
  Y~ = q deq from the (separately pinned) forward quantizer;
- the norm's invariances: the centred norm's output is unchanged by a shift of x, so
  sum_j dX_j = 0, and (eps -> 0) by a scaling of x, so sum_j dX_j (x_j - mu) = 0; the
  RMSNorm is scale-invariant, so sum_j dX_j x_j = 0.
Shapes are non-square so a transposed operand fails."""
import numpy as np
import pytest

import oracle as O


def _setup(M=3, K=12, N=5, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((M, K)).astype(np.float32) * 1.7 + 0.3
    W = (rng.standard_normal((N, K)) * 0.05).astype(np.float32)
    t, m = O.ternarize(W)
    dO = rng.standard_normal((M, N)).astype(np.float32)
    return X, t, np.float32(m), dO


def _norm64(x, centred, eps):
    x = x.astype(np.float64)
    mu = x.mean(axis=-1, keepdims=True) if centred else 0.0
    var = ((x - mu) ** 2).mean(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + eps)


@pytest.mark.parametrize("norm", [0, 1])
def test_dx_finite_differences(norm):
    X, t, m, dO = _setup(seed=1 + norm)
    eps = 1e-6
    Wt = t.astype(np.float64) * float(m)
    dX, _, _ = O.bitlinear_bwd(X, t, m, dO, eps=eps, norm=norm)

    def loss(x):
        return float(np.sum(dO.astype(np.float64) * (_norm64(x, norm == 1, eps) @ Wt.T)))

    fd = np.zeros_like(dX)
    h = 1e-5
    X64 = X.astype(np.float64)
    for i in range(X.shape[0]):
        for j in range(X.shape[1]):
            xp = X64.copy(); xp[i, j] += h
            xm = X64.copy(); xm[i, j] -= h
            fd[i, j] = (loss(xp) - loss(xm)) / (2 * h)
    # the oracle uses the forward's binary32 mu and r (B3): ~1e-7 relative
    np.testing.assert_allclose(dX, fd, rtol=0, atol=2e-5 * np.abs(fd).max())


def test_dw_db_finite_differences():
    X, t, m, dO = _setup(M=4, K=10, N=6, seed=7)
    _, dW, db = O.bitlinear_bwd(X, t, m, dO)
    q, deq, _, _ = O.quant_rows(X)
    Yt = q.astype(np.float64) * deq.astype(np.float64)[:, None]
    Wt = t.astype(np.float64) * float(m)
    b = np.zeros(t.shape[0])
    d64 = dO.astype(np.float64)

    def loss(Wv, bv):
        return float(np.sum(d64 * (Yt @ Wv.T + bv)))

    h = 1e-3
    fdW = np.zeros_like(Wt)
    for n in range(Wt.shape[0]):
        for j in range(Wt.shape[1]):
            wp = Wt.copy(); wp[n, j] += h
            wm = Wt.copy(); wm[n, j] -= h
            fdW[n, j] = (loss(wp, b) - loss(wm, b)) / (2 * h)
    fdb = np.zeros_like(b)
    for n in range(b.size):
        bp = b.copy(); bp[n] += h
        bm = b.copy(); bm[n] -= h
        fdb[n] = (loss(Wt, bp) - loss(Wt, bm)) / (2 * h)
    np.testing.assert_allclose(dW, fdW, rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(db, fdb, rtol=1e-9, atol=1e-9)


def test_norm_invariances():
    X, t, m, dO = _setup(M=5, K=64, N=9, seed=11)
    # centred: shift invariance (exact in real arithmetic) and scale invariance (eps -> 0)
    dX, _, _ = O.bitlinear_bwd(X, t, m, dO, eps=1e-12, norm=1)
    mu = X.astype(np.float64).mean(axis=1, keepdims=True)
    scale = np.abs(dX).sum(axis=1)
    assert np.all(np.abs(dX.sum(axis=1)) <= 1e-6 * scale)
    assert np.all(np.abs((dX * (X - mu)).sum(axis=1)) <= 1e-5 * scale * np.abs(X).max())
    # RMSNorm: scale invariance only
    dX0, _, _ = O.bitlinear_bwd(X, t, m, dO, eps=1e-12, norm=0)
    scale0 = np.abs(dX0).sum(axis=1)
    assert np.all(np.abs((dX0 * X).sum(axis=1)) <= 1e-5 * scale0 * np.abs(X).max())
    assert np.any(np.abs(dX0.sum(axis=1)) > 1e-3 * scale0)   # no shift invariance there


def test_zero_upstream_gradient():
    X, t, m, dO = _setup(seed=3)
    dX, dW, db = O.bitlinear_bwd(X, t, m, np.zeros_like(dO), norm=1)
    assert not dX.any() and not dW.any() and not db.any()
