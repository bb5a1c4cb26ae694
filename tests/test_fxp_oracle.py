"""Pins of the fixed-point W8A16 oracle (
readings F1-F5 in DESIGN.md) against what the paper and the mathematics fix -- worked examples
of the scale formula, sigma(0) = 2^(y_exp-1), the symmetry identity, monotonicity, the
interpolation error bound of a piecewise-linear sigma, exact powers of four for the inverse
square root, Newton's error bound, and Eq. 1 evaluated in binary64 within one output step.
"""
import math

import numpy as np
import pytest

import oracle as O


# ------------------------------------------------------------------ F1 norm-scale quantization
def test_scales_literal_examples():
    """P:506 with shift 0 (the literal s_w = 2^round(log2 max|w|)): worked examples."""
    assert O.fxp_scales([1.0, 0.5], 0)[0].tolist() == [1, 1] and O.fxp_scales([1.0, 0.5], 0)[1] == 0
    assert O.fxp_scales([4.0], 0) [0].tolist() == [1] and O.fxp_scales([4.0], 0)[1] == 2
    wq, e = O.fxp_scales([0.3], 0)     # log2 0.3 = -1.74 -> -2: s_w = 0.25, 0.3/0.25 = 1.2 -> 1
    assert e == -2 and wq.tolist() == [1]
    wq, e = O.fxp_scales([-3.0, 0.1], 0)   # log2 3 = 1.58 -> 2: 3/4 = 0.75 -> -1; 0.025 -> 0
    assert e == 2 and wq.tolist() == [-1, 0]


def test_scales_int8_range_and_error():
    rng = np.random.default_rng(1)
    for scale in (1e-3, 0.02, 1.0, 37.0):
        w = (scale * (1 + 0.3 * rng.standard_normal(777))).astype(np.float32)
        wq, e = O.fxp_scales(w, 6)
        assert e == round(math.log2(np.abs(w).max())) - 6
        assert np.abs(wq).max() <= 91          # max|w|/2^e < 2^6.5
        assert np.abs(wq).max() >= 45          # > 2^5.5
        err = np.abs(w.astype(np.float64) - wq * 2.0 ** e)
        assert err.max() <= 2.0 ** (e - 1)     # round to nearest


def test_scales_degenerate():
    with pytest.raises(RuntimeError):
        O.fxp_scales(np.zeros(4, np.float32))


# ------------------------------------------------------------------ F2 activation quantization
def test_quant_act_minimal_exponent():
    rng = np.random.default_rng(2)
    for s in (1e-4, 1.0, 3e3):
        x = (s * rng.standard_normal(1000)).astype(np.float32)
        q, e = O.fxp_quant_act(x)
        mx = float(np.abs(x).max())
        assert np.abs(q).max() <= 32767
        assert round(mx / 2.0 ** (e - 1)) > 32767          # e - 1 would overflow
        assert np.abs(x - q * 2.0 ** e).max() <= 2.0 ** (e - 1)
    x = np.array([32767.0, -1.0, 0.4], np.float32)            # fits exactly at e = 0
    q, e = O.fxp_quant_act(x)
    assert e == 0 and q.tolist() == [32767, -1, 0]
    q, e = O.fxp_quant_act(np.zeros(5, np.float32))
    assert e == 0 and not q.any()


# ------------------------------------------------------------------ F3 sigmoid LUT
X = np.arange(-1200, 1201, dtype=np.int32)


def test_sigmoid_zero_and_symmetry():
    """sigma_fxp(0) = 2^(y_exp-1); sigma(-x) = 1 - sigma(x) exactly."""
    assert O.fxp_sigmoid([0])[0] == 2 ** (O.FXP_YEXP - 1)
    y = O.fxp_sigmoid(X)
    assert np.array_equal(y + y[::-1], np.full(X.size, 2 ** O.FXP_YEXP))


def test_sigmoid_monotone_and_breakpoints():
    y = O.fxp_sigmoid(X)
    assert np.all(np.diff(y) >= 0)
    # at the LUT points x = i (i = 0..8) the value is floor(sigma(i) 2^15);
    # sigma(1) = 0.7310585786300049 -> 23955.2 -> 23955; sigma(8) = 0.9996646498695336 -> 32757.0
    assert O.fxp_sigmoid([64])[0] == 23955
    assert O.fxp_sigmoid([512])[0] == 32757 and O.fxp_sigmoid([10 ** 6])[0] == 32757
    # worked example x = 1.5 (x_fxp = 96): 23955 + floor((26428 - 23955) * 32 / 64)
    y2 = O.fxp_sigmoid([128])[0]
    assert O.fxp_sigmoid([96])[0] == 23955 + ((y2 - 23955) * 32) // 64


def test_sigmoid_error_bound():
    """|sigma_fxp - sigma| <= h^2/8 max|sigma''| + floors: h = 1, max|sigma''| = 1/(6 sqrt 3),
    plus 2 ulps (2^-15) for the LUT and interpolation floors; beyond x = 8: 1 - sigma(8)."""
    x = np.arange(-(1 << 11), (1 << 11) + 1, dtype=np.int32)
    y = O.fxp_sigmoid(x) / 2.0 ** 15
    ref = 1.0 / (1.0 + np.exp(-x / 64.0))
    bound = 1.0 / 8.0 / (6.0 * math.sqrt(3.0)) + 2.0 ** -14
    assert np.abs(y - ref).max() <= bound
    assert np.abs(y - ref).max() > 1e-3      # the LUT really is coarse (8 entries)


# ------------------------------------------------------------------ F4 inverse square root
def test_inv_sqrt_powers_of_four():
    v = np.array([1, 4, 16, 1 << 20, 1 << 40, 1 << 62], np.uint64)
    y, ey = O.fxp_inv_sqrt(v, 0)
    val = y * 2.0 ** ey.astype(np.float64)
    ref = 1.0 / np.sqrt(v.astype(np.float64))
    assert np.all(np.abs(val / ref - 1.0) <= 2.0 ** -29)
    y, ey = O.fxp_inv_sqrt(np.array([1, 1], np.uint64), np.array([2, -2], np.int32))
    assert np.allclose(y * 2.0 ** ey.astype(np.float64), [0.5, 2.0], rtol=2.0 ** -29)


def test_inv_sqrt_relative_error_sweep():
    """Five Newton steps from a 24-entry LUT (initial error <= 3.2 %): e_{k+1} <= 1.5 e_k^2 +
    truncation -> below 2^-28 relative; spec examples 1.0 -> 1.0 and 4.0 -> 0.5 within 1e-3."""
    rng = np.random.default_rng(3)
    v = np.concatenate([np.arange(1, 5000, dtype=np.uint64),
                        rng.integers(1, 1 << 62, 20000, dtype=np.uint64)])
    e = rng.integers(-40, 40, v.size).astype(np.int32)
    y, ey = O.fxp_inv_sqrt(v, e)
    val = y.astype(np.float64) * 2.0 ** ey.astype(np.float64)
    ref = 1.0 / np.sqrt(v.astype(np.float64) * 2.0 ** e.astype(np.float64))
    # low bits of v beyond 31 significant bits are dropped (F4): relative input error <= 2^-30
    assert np.abs(val / ref - 1.0).max() <= 2.0 ** -28


def test_inv_sqrt_non_increasing():
    v = np.sort(np.random.default_rng(4).integers(1, 1 << 50, 50000, dtype=np.uint64))
    y, ey = O.fxp_inv_sqrt(v, 0)
    val = y.astype(np.float64) * 2.0 ** ey.astype(np.float64)
    assert np.all(np.diff(val) <= 0)


def test_inv_sqrt_rejects_zero():
    with pytest.raises(RuntimeError):
        O.fxp_inv_sqrt(np.array([0], np.uint64), 0)


# ------------------------------------------------------------------ F5 RMSNorm (Eq. 1)
def _eq1(x, w, eps):
    x = x.astype(np.float64)
    return x / np.sqrt(eps + (x * x).mean(1, keepdims=True)) * w


@pytest.mark.parametrize("d", [64, 1000, 1024, 2560])
def test_rmsnorm_matches_eq1(d):
    rng = np.random.default_rng(d)
    x = (rng.standard_normal((9, d)) * np.logspace(-2, 2, 9)[:, None]).astype(np.float32)
    w = (1.0 + 0.25 * rng.standard_normal(d)).astype(np.float32)
    xq, ex = O.fxp_quant_act(x)
    wq, ew = O.fxp_scales(w)
    out, eo = O.fxp_rmsnorm(xq, ex, wq, ew)
    got = out * 2.0 ** eo[:, None].astype(np.float64)
    # the exact Eq. 1 of the quantized operands, with eps on the grid of the integer sum of
    # squares (F5: eps_q = round(d eps 2^(-2 ex))); error <= half an output step + 5e-7
    # relative (sqrt(d) held in Q16: <= 2^-17/sqrt(d) <= 2.4e-7; inverse sqrt <= 2^-28)
    eps_eff = round(d * 1e-3 * 2.0 ** (-2 * ex)) * 2.0 ** (2 * ex) / d
    ref = _eq1(xq * 2.0 ** ex, wq * 2.0 ** ew, eps_eff)
    tol = 0.5 * 2.0 ** eo[:, None].astype(np.float64) + 5e-7 * np.abs(ref).max(1, keepdims=True)
    assert np.all(np.abs(got - ref) <= tol)
    big = np.abs(out).max(1) > 16383                     # the smallest fitting exponent ...
    assert np.all(big | (eo == eo.min()))                 # ... unless s = 0 already
    # and the float RMSNorm of the float operands within the quantization of x and w, on the
    # rows the per-tensor exponent resolves to >= 10 bits (rows 0-3 are 1e-2..1e0 of row 8)
    fl = _eq1(x, w, 1e-3)
    assert np.abs(got - fl)[4:].max() <= 0.02 * np.abs(fl[4:]).max()


@pytest.mark.parametrize("scale", [1e-3, 1e-6, 1e-9, 1e-12])
def test_rmsnorm_tiny_activations_keep_eq1(scale):
    """Reading F5b: when round(d eps 2^(-2 ex)) would exceed 2^60 (tiny activations) the sum
    S + eps_q is formed on a coarser even grid 2^(2k) and handed to F4 with that exponent, so
    the output is still Eq. 1 with eps = 1e-3 -- pinned here against the
    float definition.  (A clamp of eps_q at 2^60 would make the norm too large by
    sqrt(eps_q / 2^60): 2^25 at scale 1e-12.)"""
    rng = np.random.default_rng(11)
    d = 1024
    x = (rng.standard_normal((4, d)) * scale).astype(np.float32)
    w = (1.0 + 0.25 * rng.standard_normal(d)).astype(np.float32)
    xq, ex = O.fxp_quant_act(x)
    wq, ew = O.fxp_scales(w)
    if scale < 1e-5:
        assert round(d * 1e-3 * 2.0 ** (-2 * ex)) > 2.0 ** 60   # the coarse-grid regime
    out, eo = O.fxp_rmsnorm(xq, ex, wq, ew)
    got = out * 2.0 ** eo[:, None].astype(np.float64)
    ref = _eq1(xq * 2.0 ** ex, wq * 2.0 ** ew, 1e-3)
    tol = 0.5 * 2.0 ** eo[:, None].astype(np.float64) + 5e-7 * np.abs(ref).max(1, keepdims=True)
    assert np.all(np.abs(got - ref) <= tol)
    assert np.abs(out).max() > 16383          # the output still uses the int16 range


def test_rmsnorm_one_hot_and_zero():
    d = 256
    x = np.zeros((3, d), np.int16)
    x[0, 7] = 1000                  # one-hot: y_7 = k 2^ex / sqrt(eps + k^2 2^(2ex)/d) w_7
    x[1, :] = 0                     # zero row with eps_q > 0: exact zeros
    x[2, 5] = -3
    wq, ew = np.full(d, 64, np.int8), -6          # w = 1
    ex = -8
    out, eo = O.fxp_rmsnorm(x, ex, wq, ew)
    k = 1000 * 2.0 ** ex
    ref = k / math.sqrt(1e-3 + k * k / d)
    assert abs(out[0, 7] * 2.0 ** eo[0] - ref) <= 0.5 * 2.0 ** eo[0] + 1e-7 * ref
    assert np.count_nonzero(out[0]) == 1 and not out[1].any() and out[2, 5] < 0
    # eps underflow: with eps = 1e-6 and large activations eps_q = 0; a zero row then
    # has S + eps_q = 0 and outputs zeros with exponent 0 instead of dividing by zero
    out, eo = O.fxp_rmsnorm(np.zeros((1, d), np.int16), 12, wq, ew, eps=1e-6)
    assert not out.any() and eo[0] == 0


def test_rmsnorm_zero_gain_and_scale_covariance():
    rng = np.random.default_rng(7)
    d = 512
    x = rng.integers(-3000, 3000, (4, d)).astype(np.int16)
    out, eo = O.fxp_rmsnorm(x, -10, np.zeros(d, np.int8), 0)
    assert not out.any()
    wq = rng.integers(-90, 90, d).astype(np.int8)
    a, ea = O.fxp_rmsnorm(x, -10, wq, -6)
    b, eb = O.fxp_rmsnorm(x, -9, wq, -6)       # doubling x: output changes by < 0.1 %
    va, vb = a * 2.0 ** ea[:, None], b * 2.0 ** eb[:, None]
    assert np.abs(va - vb).max() <= 1e-3 * np.abs(va).max()


# ------------------------------------------------------------------ F6 W8A16 BitLinear
def _f6_case(M, K, N, seed):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((M, K)) * 3.0).astype(np.float32)
    g = (1.0 + 0.2 * rng.standard_normal(K)).astype(np.float32)
    W = (0.02 * rng.standard_normal((N, K))).astype(np.float32)
    t, beta = O.ternarize(W)
    xq, ex = O.fxp_quant_act(x)
    gq, eg = O.fxp_scales(g)
    return x, g, t, beta, xq, ex, gq, eg


@pytest.mark.parametrize("M,K,N", [(1, 64, 16), (5, 1000, 300), (3, 1024, 1024)])
def test_bitlinear_w8a16_vs_float(M, K, N):
    """(a) Against the float BitLinear (Eq. 1 RMSNorm with eps = 1e-3, the ternary product,
    the scale) of the QUANTIZED operands x_q 2^ex, g_q 2^eg, b_q 2^eb: within the int16
    roundings, 1e-4 of the row's largest output plus one output step.  (b) Against the float
    operands within the gains' and beta's int8 quantization errors, bounded term by term."""
    x, g, t, beta, xq, ex, gq, eg = _f6_case(M, K, N, K + N)
    y, ey = O.fxp_bitlinear(xq, ex, gq, eg, t, beta)
    got = y * 2.0 ** ey[:, None].astype(np.float64)
    step = 2.0 ** ey[:, None].astype(np.float64)
    bq, eb = O.fxp_scales(np.array([beta], np.float32))
    bqv = float(bq[0]) * 2.0 ** eb
    gqv = gq * 2.0 ** eg
    ref_q = _eq1(xq * 2.0 ** ex, gqv, 1e-3) @ t.T.astype(np.float64) * bqv
    scale = np.abs(ref_q).max(1, keepdims=True)
    assert np.all(np.abs(got - ref_q) <= 1e-4 * scale + step)
    assert np.all(np.abs(y).max(1) > 16383)      # the smallest fitting output exponent
    xn1 = _eq1(x, np.ones(K), 1e-3)              # x / rms(x)
    ref = xn1 * g @ t.T.astype(np.float64) * beta
    bound = (np.abs(xn1) * np.abs(g - gqv)) @ np.abs(t.T).astype(np.float64) * abs(bqv) \
        + np.abs(ref) * abs(bqv / beta - 1.0) + 2e-3 * scale + step
    assert np.all(np.abs(got - ref) <= bound)


def test_bitlinear_w8a16_identity_and_zero():
    """t = I: the output is F5's normalised row times beta's int8 value, exactly rescaled;
    a zero row stays zero."""
    K = 128
    rng = np.random.default_rng(9)
    xq = rng.integers(-20000, 20000, (2, K)).astype(np.int16)
    xq[1] = 0
    gq, eg = np.full(K, 64, np.int8), -6
    t = np.eye(K, dtype=np.int8)
    beta = 0.75                                  # log2 0.75 -> 0: e = -6, bq = 48 exactly
    y, ey = O.fxp_bitlinear(xq, -4, gq, eg, t, beta)
    yn, en = O.fxp_rmsnorm(xq, -4, gq, eg)
    p = yn[0].astype(np.int64) * 48
    s = 0
    while np.abs(np.where(p < 0, -((-p + (1 << s >> 1)) >> s), (p + (1 << s >> 1)) >> s)).max() > 32767:
        s += 1
    assert ey[0] == s + en[0] - 6
    assert np.allclose(y[0] * 2.0 ** ey[0], yn[0] * 2.0 ** en[0] * 0.75, atol=2.0 ** ey[0])
    assert not y[1].any()
