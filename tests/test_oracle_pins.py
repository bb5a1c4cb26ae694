"""Pins of the CPU oracle against values the paper / mathematics fix (not GPU).

Every test here checks ``oracle/`` against something other than itself:
worked examples (tests/golden/pins.json, each cited), closed forms,
invariants, textbook/library routines and brute force.  A plausible mistake in
the oracle (dropped term, wrong sign or index, transposed operand, wrong
rounding mode, sum-vs-mean norm) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pins.json")))
rng = np.random.default_rng(12345)


def f32(x):
    return np.asarray(x, dtype=np.float32)


# ------------------------------------------------------------------ exp / sigmoid (C12)
def _ulp_err(a, ref):
    ref32 = ref.astype(np.float32)
    spacing = np.spacing(np.abs(ref32)).astype(np.float64)
    return np.abs(a.astype(np.float64) - ref) / spacing


def test_exp_c_within_2ulp_of_libm_double():
    x = np.linspace(-87.3, 88.7, 2_000_001, dtype=np.float32)
    x = np.concatenate([x, f32([-1e-30, 0.0, 1e-30, 0.5, -0.5, 1.0, -1.0, 10.0, -10.0])])
    y = O.exp_c(x)
    ref = np.exp(x.astype(np.float64))
    assert np.max(_ulp_err(y, ref)) <= 2.0


def test_exp_c_special_values():
    y = O.exp_c(f32([0.0, 100.0, -100.0, np.inf, -np.inf, np.nan]))
    assert y[0] == 1.0 and y[1] == np.inf and y[2] == 0.0 and y[3] == np.inf and y[4] == 0.0
    assert np.isnan(y[5])


def test_sigmoid_c_pins():
    assert O.sigmoid_c(f32([0.0]))[0] == np.float32(0.5)
    x = np.linspace(-40, 40, 400_001, dtype=np.float32)
    s = O.sigmoid_c(x)
    assert np.all(np.diff(s.astype(np.float64)) >= 0), "sigmoid must be monotone"
    ref = 1.0 / (1.0 + np.exp(-x.astype(np.float64)))
    big = ref > 1e-30
    assert np.max(_ulp_err(s[big], ref[big])) <= 3.0
    # sigma(x) + sigma(-x) = 1 within one ulp of 1
    tot = s.astype(np.float64) + O.sigmoid_c(-x).astype(np.float64)
    assert np.max(np.abs(tot - 1.0)) <= 2 * np.spacing(np.float32(1.0))


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = (rng.standard_normal(200_000) * 10.0 ** rng.integers(-8, 8, 200_000)).astype(np.float32)
    x = np.concatenate([x, f32([0.0, -0.0, np.inf, -np.inf, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8])])
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert np.array_equal(O.bf16_round(x), ref)


# ------------------------------------------------------------------ a1 weight_quant
@pytest.mark.parametrize("key", ["weight_quant_W1", "weight_quant_unit", "weight_quant_W2_rounding"])
def test_weight_quant_examples(key):
    g = GOLD[key]
    t, m = O.ternarize(f32(g["W"]))
    assert np.array_equal(t, np.array(g["codes"], np.int8))
    assert abs(float(m) - g["scale"]) <= 1e-7 * max(1.0, g["scale"])


def test_weight_quant_degenerate():
    with pytest.raises(O.OracleError):
        O.absmean(np.zeros((4, 4), np.float32))
    with pytest.raises(O.OracleError):
        O.absmean(f32([[1.0, np.nan]]))


def test_zero_fraction_closed_form():
    # erf(1/(2 sqrt(pi))) = 0.3100643; +-5 sigma binomial bound on 1M weights = 0.0023
    val = GOLD["zero_fraction_gaussian"]["value"]
    assert abs(math.erf(1 / (2 * math.sqrt(math.pi))) - val) < 1e-7
    W = (rng.standard_normal((1000, 1000)) * 0.02).astype(np.float32)
    t, m = O.ternarize(W)
    zf = O.zero_fraction(t)
    assert abs(zf - val) < 0.0023
    # ternary set, and +1 / -1 balanced within binomial noise
    assert set(np.unique(t)) <= {-1, 0, 1}
    p, n = np.mean(t == 1), np.mean(t == -1)
    assert abs(p - n) < 5 * math.sqrt(0.35 / t.size) * 2


def test_weight_quant_matches_scalar_formula():
    # dequantized matrix = clamp(round(W / mean|W|), -1, 1) * mean|W| (fp64 reference)
    W = (rng.standard_normal((8, 8)) * 0.3).astype(np.float32)
    t, m = O.ternarize(W)
    mean64 = np.mean(np.abs(W.astype(np.float64)))
    assert abs(float(m) - mean64) <= 1e-7 * mean64
    v = W.astype(np.float64) / mean64
    # away from exact .5 ties the fp32 and fp64 roundings agree
    ref = np.clip(np.sign(v) * np.floor(np.abs(v) + 0.5), -1, 1)
    safe = np.abs(np.abs(v) - 0.5) > 1e-5
    assert np.array_equal(t[safe], ref[safe].astype(np.int8))


# ------------------------------------------------------------------ packed layout decoder
def test_packed_word_example():
    g = GOLD["packed_word"]
    codes = np.zeros((1, 1, 8), np.uint32)
    codes[0, 0, 0] = int(g["word"], 16)
    t = O.unpack_segment(codes, 1, 16)
    assert t.tolist() == [g["trits"]]


def test_packed_row_interleave():
    # 3 segments interleaved in groups of 64 rows: [f0..63 | c0..63 | g0..63 | f64 ...]
    assert O.packed_row(0, 0, 3, 64) == 0
    assert O.packed_row(1, 0, 3, 64) == 64
    assert O.packed_row(2, 63, 3, 64) == 191
    assert O.packed_row(0, 64, 3, 64) == 192
    assert O.packed_row(1, 70, 3, 64) == 192 + 64 + 6


def test_unpack_rejects_reserved_field():
    codes = np.zeros((1, 1, 8), np.uint32)
    codes[0, 0, 0] = 0x3
    with pytest.raises(O.OracleError):
        O.unpack_segment(codes, 1, 16)


def test_unpack_k_block_major_layout():
    # word w of packed row r sits at ((w/8)*n_rows + r)*8 + w%8: put a +1 trit at
    # k = 128*b + 16*j + 4*f + byte for a few (b, j, f, byte, r) and read it back
    n_rows, nkb = 3, 2
    for (b, j, f, byte, r) in [(0, 0, 0, 0, 0), (1, 7, 3, 3, 2), (1, 2, 1, 2, 1), (0, 5, 2, 1, 1)]:
        codes = np.full((nkb, n_rows, 8), 0x55555555, np.uint32)      # all zero trits
        w = codes[b, r, j]
        shift = 8 * byte + 2 * f
        codes[b, r, j] = (w & ~np.uint32(3 << shift)) | np.uint32(2 << shift)   # e = 2 -> +1
        t = O.unpack_segment(codes, n_rows, 256)
        k = 128 * b + 16 * j + 4 * f + byte
        assert t[r, k] == 1 and np.count_nonzero(t) == 1


# ------------------------------------------------------------------ a2 activation quant
@pytest.mark.parametrize("key", ["act_quant_A1", "act_quant_unit", "act_quant_zero",
                                 "act_quant_A2_rounding"])
def test_act_quant_examples(key):
    g = GOLD[key]
    q, deq, a = O.act_quant(f32(g["y"]))
    assert q.tolist() == g["q"]
    assert abs(float(deq) - g["deq"]) <= 1e-7


def test_act_quant_invariants():
    for _ in range(200):
        K = int(rng.integers(1, 300))
        y = (rng.standard_normal(K) * 10 ** rng.uniform(-3, 3)).astype(np.float32)
        q, deq, a = O.act_quant(y)
        assert np.max(np.abs(q.astype(np.int32))) == 127          # C5: max|q| = 127
        assert np.all(q >= -127)
        # scaling by 2^k leaves the quantized codes unchanged (exact in fp32)
        q2, deq2, _ = O.act_quant(y * np.float32(2.0 ** int(rng.integers(-20, 20))))
        assert np.array_equal(q, q2)
        # dequantized codes approximate y within half a step
        assert np.max(np.abs(q * np.float64(deq) - y)) <= 0.5 * deq * (1 + 1e-5) + 1e-30


# ------------------------------------------------------------------ RMSNorm (C1)
def test_rmsnorm_mean_form_closed_form():
    for K in (1, 7, 256, 1000):
        x = rng.standard_normal(K).astype(np.float32) * 3
        y, r = O.rmsnorm(x, eps=1e-6)
        ms = np.mean(x.astype(np.float64) ** 2)
        # mean(y^2) * (ms + eps) / ms == 1: pins mean (not sum) and eps inside the sqrt
        assert abs(np.mean(y.astype(np.float64) ** 2) * (ms + 1e-6) / ms - 1) < 3e-6
        assert abs(float(r) - 1 / math.sqrt(ms + 1e-6)) <= 1e-7 / math.sqrt(ms)


def test_rmsnorm_constant_row_and_gain():
    x = np.full(64, 2.5, np.float32)
    y, r = O.rmsnorm(x, eps=1e-6)
    assert abs(float(r) - 1 / math.sqrt(2.5 ** 2 + 1e-6)) < 1e-7
    assert np.all(y == y[0])
    g = np.linspace(0.5, 2, 64).astype(np.float32)
    yg, _ = O.rmsnorm(x, gain=g, eps=1e-6)
    assert np.allclose(yg, y * g, rtol=1e-6)


def test_double_rmsnorm_identity():
    # App. C.3: RMSNorm(RMSNorm(x; g1); g2) = x g1 g2 / sqrt(mu (g1^2+eps) + eps^2)
    #                                                = x g_comb / sqrt(mu + eps_comb)
    eps = 1e-3
    for g1, g2 in ((1.0, 1.0), (0.7, 1.3), (2.0, 0.25)):
        x = rng.standard_normal(512).astype(np.float32) * 0.05
        y, _ = O.rmsnorm(x, gain=np.full(512, g1, np.float32), eps=eps)
        z, _ = O.rmsnorm(y, gain=np.full(512, g2, np.float32), eps=eps)
        mu = np.mean(x.astype(np.float64) ** 2)
        x64 = x.astype(np.float64)
        zc = x64 * g1 * g2 / math.sqrt(mu * (g1 ** 2 + eps) + eps ** 2)
        gcomb = g1 * g2 / math.sqrt(g1 ** 2 + eps)
        ecomb = eps ** 2 / (g1 ** 2 + eps)
        zc2 = x64 * gcomb / math.sqrt(mu + ecomb)
        assert np.allclose(z, zc, rtol=2e-6, atol=1e-9)
        assert np.allclose(zc, zc2, rtol=1e-12)


# ------------------------------------------------------------------ centred norm (Alg. 1, f4(i), C22)
def test_centred_norm_worked_example():
    """Alg. 1 rms_norm_fwd on x = [1, 2, 3, 4]: mu = 2.5 and
    sigma^2 = 1.25 exactly, Y = r (X - mu) = r [-1.5, -0.5, 0.5, 1.5]; the
    absmax quantizer then gives 127/1.5 * [-1.5, -0.5, 0.5, 1.5]
    = [-127, -42.33, 42.33, 127] -> [-127, -42, 42, 127]."""
    x = f32([1, 2, 3, 4])
    with O.norm_mode(1):
        y, r = O.rmsnorm(x, eps=1e-6)
        q, deq, rr, a = O.quant_rows(x[None])
    assert float(r) == float(np.float32(1 / math.sqrt(1.25 + 1e-6)))
    assert np.array_equal(y, f32([-1.5, -0.5, 0.5, 1.5]) * np.float32(r))
    assert q[0].tolist() == [-127, -42, 42, 127]
    assert a[0] == np.float32(np.float32(1.5) * np.float32(r))
    # the uncentred reading gives different codes on the same row
    assert O.quant_rows(x[None])[0][0].tolist() == [32, 64, 95, 127]


def test_centred_norm_shift_invariance_exact():
    """Adding a power of two c to integer rows shifts mu by exactly c, so every
    x_j - mu (and hence y, q, deq, r) is bit-identical: pins the subtraction
    of the mean (dropped or wrong-signed mu fails)."""
    for K in (8, 64, 1024):
        x = rng.integers(-50, 50, K).astype(np.float32)
        with O.norm_mode(1):
            q0, d0, r0, a0 = O.quant_rows(x[None])
            q1, d1, r1, a1 = O.quant_rows((x + np.float32(64))[None])
        assert np.array_equal(q0, q1) and d0[0] == d1[0] and r0[0] == r1[0] and a0[0] == a1[0]


def test_centred_norm_zero_mean_row_equals_rmsnorm():
    """A row of +-pairs has sum exactly 0, so mu = 0 and the variance equals
    the mean square: the centred and uncentred forms agree bit for bit."""
    h = rng.standard_normal(256).astype(np.float32)
    x = np.concatenate([h, -h])
    rng.shuffle(x)
    with O.norm_mode(1):
        yc, rc = O.rmsnorm(x, eps=1e-6)
    yu, ru = O.rmsnorm(x, eps=1e-6)
    assert rc == ru and np.array_equal(yc, yu)


def test_centred_norm_moments_closed_form():
    """mean(y) ~ 0 and mean(y^2) (sigma^2 + eps) / sigma^2 = 1 (unit gain)."""
    for K in (7, 256, 1000):
        x = (rng.standard_normal(K) * 2 + 5).astype(np.float32)
        with O.norm_mode(1):
            y, r = O.rmsnorm(x, eps=1e-6)
        x64 = x.astype(np.float64)
        var = np.var(x64)
        y64 = y.astype(np.float64)
        assert abs(np.mean(y64)) < 1e-5
        assert abs(np.mean(y64 ** 2) * (var + 1e-6) / var - 1) < 1e-5
        assert abs(float(r) - 1 / math.sqrt(var + 1e-6)) <= 2e-7 / math.sqrt(var)


def test_centred_norm_constant_row_is_degenerate():
    """A constant row has X - mu = 0: q = 0 and deq = 0 (C7)."""
    x = np.full((1, 64), 3.25, np.float32)
    with O.norm_mode(1):
        q, deq, r, a = O.quant_rows(x)
    assert np.all(q == 0) and deq[0] == 0 and a[0] == 0


def test_quant_rows_per_token():
    X = rng.standard_normal((5, 40)).astype(np.float32)
    X[2] = 0
    q, deq, r, a = O.quant_rows(X)
    for i in range(5):
        y, ri = O.rmsnorm(X[i])
        qi, di, ai = O.act_quant(y)
        assert np.array_equal(q[i], qi) and deq[i] == di and r[i] == ri and a[i] == ai
    assert np.all(q[2] == 0) and deq[2] == 0


# ------------------------------------------------------------------ a3/a4 ternary accumulation
def test_tern_dot_bruteforce():
    # every trit row for K <= 6 x 100 random int8 vectors: literal add/sub == int64 MAC
    import itertools
    for K in range(1, 7):
        rows = np.array(list(itertools.product((-1, 0, 1), repeat=K)), np.int8)
        qs = rng.integers(-128, 128, size=(100, K)).astype(np.int8)
        ref = qs.astype(np.int64) @ rows.T.astype(np.int64)
        got = O.tern_matmul(qs, rows)
        assert np.array_equal(got, ref)


def test_tern_dot_extremes():
    K = 6912
    t = np.ones(K, np.int8)
    q = np.full(K, 127, np.int8)
    assert O.tern_dot(t, q) == 127 * K
    assert O.tern_dot(-t, np.full(K, -128, np.int8)) == 128 * K


def test_bitlinear_equals_dense_fp64_product():
    # G2 / S:61,S:73: BitLinear == dense fp64 product of dequantized operands (+b), 1e-6
    for M, K, N in ((1, 64, 32), (7, 96, 50), (16, 256, 64)):
        X = rng.standard_normal((M, K)).astype(np.float32)
        W = (rng.standard_normal((N, K)) * 0.02).astype(np.float32)
        b = rng.standard_normal(N).astype(np.float32)
        t, m = O.ternarize(W)
        out, tp = O.bitlinear(X, t, m, bias=b, taps=True)
        deq = tp["deq"].astype(np.float64)
        Yd = tp["q"].astype(np.float64) * deq[:, None]          # dequantized activations
        Wd = t.astype(np.float64) * float(m)                      # dequantized weights
        ref = Yd @ Wd.T + b
        scale = np.abs(Yd) @ np.abs(Wd).T + np.abs(b)
        assert np.all(np.abs(out - ref) <= 1e-6 * scale + 1e-7)
        # the taps are the oracle's own quantizer
        q2, d2, _, _ = O.quant_rows(X)
        assert np.array_equal(q2, tp["q"]) and np.array_equal(d2, tp["deq"])


def test_bitlinear_permutation_invariance():
    M, K, N = 4, 128, 40
    X = rng.standard_normal((M, K)).astype(np.float32)
    t, m = O.ternarize((rng.standard_normal((N, K)) * 0.02).astype(np.float32))
    out, tp = O.bitlinear(X, t, m, taps=True)
    pk = rng.permutation(K)
    pn = rng.permutation(N)
    out2, tp2 = O.bitlinear(X[:, pk], t[pn][:, pk], m, taps=True)
    assert np.array_equal(tp2["acc"], tp["acc"][:, pn])
    assert np.array_equal(out2, out[:, pn])


def test_bitlinear_zero_row_gives_bias():
    X = np.zeros((2, 32), np.float32)
    t, m = O.ternarize((rng.standard_normal((8, 32)) * 0.02).astype(np.float32))
    b = rng.standard_normal(8).astype(np.float32)
    assert np.array_equal(O.bitlinear(X, t, m, bias=b), np.stack([b, b]))


# ------------------------------------------------------------------ a6 MLGRU scan
def test_scan_closed_form_exact():
    # S2: f = 1/2, c = 1 => h_t = 1 - 2^-t exactly in fp32 under any association (t <= 24)
    T = 24
    f = np.full(T, 0.5, np.float32)
    c = np.ones(T, np.float32)
    ref = f32([1 - 2.0 ** -(t + 1) for t in range(T)])
    assert np.array_equal(O.scan_seq(f, c), ref)
    for chunk in (1, 3, 5, 8, 24):
        assert np.array_equal(O.scan_chunked(f, c, chunk), ref)


def test_scan_chunked_vs_sequential():
    # S4: chunked (associative) scan == sequential within 1e-5 relative
    for T in (1, 2, 17, 64, 257):
        for _ in range(8):
            f = O.sigmoid_c(rng.standard_normal(T).astype(np.float32) * 2)
            c = rng.standard_normal(T).astype(np.float32)
            h0 = float(rng.standard_normal())
            hs = O.scan_seq(f, c, h0)
            for chunk in (1, 4, 16):
                hc = O.scan_chunked(f, c, chunk, h0)
                assert np.allclose(hc, hs, rtol=1e-5, atol=1e-6)


def test_scan_convexity():
    # S3: h is a convex combination, so h stays within [min, max] of {h0, c_t}
    T = 500
    f = O.sigmoid_c(rng.standard_normal(T).astype(np.float32) * 3)
    c = rng.uniform(-2, 3, T).astype(np.float32)
    h = O.scan_seq(f, c, 0.5)
    lo, hi = min(0.5, c.min()), max(0.5, c.max())
    assert np.all(h >= lo) and np.all(h <= hi)


def test_mlgru_scan_gate_saturation():
    # fhat=-30 -> h ~ c ; fhat=+30 -> h frozen ; fhat=0, chat=0 -> h = h/2
    B, T, d = 1, 1, 16
    H = rng.standard_normal((B, d)).astype(np.float32)
    ch = rng.standard_normal((B, T, d)).astype(np.float32)
    g = rng.standard_normal((B, T, d)).astype(np.float32)
    _, H1 = O.mlgru_scan(np.full((B, T, d), -30, np.float32), ch, g, H)
    c = ch * O.sigmoid_c(ch)
    assert np.allclose(H1, c[:, 0], atol=1e-12 + 1e-12 * np.abs(H).max() + 1e-5 * 0)
    _, H2 = O.mlgru_scan(np.full((B, T, d), 30, np.float32), ch, g, H)
    assert np.array_equal(H2, H)
    _, H3 = O.mlgru_scan(np.zeros((B, T, d), np.float32), np.zeros((B, T, d), np.float32), g, H)
    assert np.array_equal(H3, H * np.float32(0.5))


def test_mlgru_scan_output_gate_modes():
    B, T, d = 2, 5, 8
    fh, chh, gh = (rng.standard_normal((B, T, d)).astype(np.float32) for _ in range(3))
    H0 = np.zeros((B, d), np.float32)
    o0, _ = O.mlgru_scan(fh, chh, gh, H0, gate_mode=0)
    o1, _ = O.mlgru_scan(fh, chh, gh, H0, gate_mode=1)
    # reconstruct h_t from the raw recurrence and check o' = g*sigma(h) / g*h (C8)
    for b in range(B):
        for ch in range(d):
            h = O.scan_seq(O.sigmoid_c(fh[b, :, ch]), chh[b, :, ch] * O.sigmoid_c(chh[b, :, ch]))
            assert np.array_equal(o0[b, :, ch], gh[b, :, ch] * O.sigmoid_c(h))
            assert np.array_equal(o1[b, :, ch], gh[b, :, ch] * h)


# ------------------------------------------------------------------ composition
def _blk(d, l, seed):
    r = np.random.default_rng(seed)
    lat = {k: (r.standard_normal(s) * 0.02).astype(np.float32) for k, s in
           {"f": (d, d), "c": (d, d), "g": (d, d), "o": (d, d), "gate": (l, d), "up": (l, d),
            "down": (d, l)}.items()}
    return O.OracleBlock(lat, d, l), lat


def test_mlgru_composition():
    d = 32
    blk, lat = _blk(d, 48, 1)
    X = rng.standard_normal((2, 6, d)).astype(np.float32)
    out, H, tp = O.mlgru(blk, X, np.zeros((2, d), np.float32), taps=True)
    Xf = X.reshape(-1, d)
    for name, key in (("f", "fhat"), ("c", "chat"), ("g", "ghat")):
        assert np.array_equal(tp[key].reshape(-1, d), O.bitlinear(Xf, blk.t[name], blk.m[name]))
    op, H2 = O.mlgru_scan(tp["fhat"], tp["chat"], tp["ghat"], np.zeros((2, d), np.float32))
    assert np.array_equal(op, tp["oprime"]) and np.array_equal(H, H2)
    assert np.array_equal(out.reshape(-1, d), O.bitlinear(op.reshape(-1, d), blk.t["o"], blk.m["o"]))


def test_glu_zero_up_and_zero_input():
    d, l = 16, 40
    blk, lat = _blk(d, l, 2)
    blk.t["up"][:] = 0            # u-path zeroed -> out = 0 (no biases in the GLU)
    X = rng.standard_normal((3, d)).astype(np.float32)
    out, tp = O.glu(blk, X, taps=True)
    assert np.all(tp["p"] == 0) and np.all(out == 0)
    blk2, _ = _blk(d, l, 3)
    assert np.all(O.glu(blk2, np.zeros((2, d), np.float32)) == 0)


def test_glu_composition():
    d, l = 24, 64
    blk, _ = _blk(d, l, 4)
    X = rng.standard_normal((5, d)).astype(np.float32)
    out, tp = O.glu(blk, X, taps=True)
    g = O.bitlinear(X, blk.t["gate"], blk.m["gate"])
    u = O.bitlinear(X, blk.t["up"], blk.m["up"])
    p = (g * O.sigmoid_c(g)) * u
    assert np.array_equal(tp["p"], p)
    assert np.array_equal(out, O.bitlinear(p, blk.t["down"], blk.m["down"]))


def test_block_prefill_then_decode_equals_longer_prefill():
    # S5: prefill(T) then decode(n) == prefill(T+n), exact in the oracle
    d, l = 32, 64
    blk, _ = _blk(d, l, 5)
    B, T, n = 2, 9, 4
    X = rng.standard_normal((B, T + n, d)).astype(np.float32)
    for bf16 in (False, True):
        Xb = O.bf16_round(X) if bf16 else X
        Yfull, Hfull = O.block(blk, Xb, np.zeros((B, d), np.float32), bf16=bf16)
        Y1, H = O.block(blk, Xb[:, :T], np.zeros((B, d), np.float32), bf16=bf16)
        ys = [Y1]
        for t in range(T, T + n):
            yt, H = O.block(blk, Xb[:, t:t + 1], H, bf16=bf16)
            ys.append(yt)
        assert np.array_equal(np.concatenate(ys, 1), Yfull)
        assert np.array_equal(H, Hfull)


def test_block_residual_structure():
    d, l = 16, 32
    blk, _ = _blk(d, l, 6)
    X = rng.standard_normal((1, 3, d)).astype(np.float32)
    Y, H, x1 = O.block(blk, X, np.zeros((1, d), np.float32), taps=True)
    o, H2 = O.mlgru(blk, X, np.zeros((1, d), np.float32))
    assert np.array_equal(x1, X + o) and np.array_equal(H, H2)
    assert np.array_equal(Y.reshape(-1, d), (x1.reshape(-1, d) + O.glu(blk, x1.reshape(-1, d))))


def test_state_is_constant_size():
    # M1: the recurrent state is B*d floats regardless of the number of decode steps
    d, l = 16, 32
    blk, _ = _blk(d, l, 7)
    H = np.zeros((1, d), np.float32)
    for _ in range(20):
        _, H = O.block(blk, rng.standard_normal((1, 1, d)).astype(np.float32), H)
        assert H.shape == (1, d) and H.nbytes == d * 4


# ---------------------------------------------------------------- sequence-parallel scan (C23)
def test_scan_seqpar_single_slice_is_sequential():
    f = O.sigmoid_c(rng.standard_normal(300).astype(np.float32))
    c = rng.standard_normal(300).astype(np.float32)
    h, hf = O.scan_seqpar(f, c, 1, 0.3)
    hs = O.scan_seq(f, c, 0.3)
    assert np.array_equal(h, hs) and hf == hs[-1]


def test_scan_seqpar_closed_form_exact():
    # S2 (f = 1/2, c = 1): h_t = 1 - 2^-t is exact in fp32 under any association (t <= 24),
    # so every slicing reproduces it bit for bit, final state included
    T = 24
    f, c = np.full(T, 0.5, np.float32), np.ones(T, np.float32)
    ref = (1.0 - 0.5 ** np.arange(1, T + 1)).astype(np.float32)
    for W in (1, 2, 3, 4, 8, 24):
        h, hf = O.scan_seqpar(f, c, W)
        assert np.array_equal(h, ref) and hf == ref[-1], W


def test_scan_seqpar_vs_sequential():
    # only the boundary states are reassociated: the first slice is bit-identical to the
    # sequential scan, the rest agree within the chunked-scan tolerance (S4)
    for T, W in ((17, 2), (256, 4), (1000, 8), (5, 8)):
        f = O.sigmoid_c(rng.standard_normal(T).astype(np.float32) * 2)
        c = rng.standard_normal(T).astype(np.float32)
        h, hf = O.scan_seqpar(f, c, W, -0.7)
        hs = O.scan_seq(f, c, -0.7)
        s1 = T // W
        assert np.array_equal(h[:s1], hs[:s1])
        assert np.allclose(h, hs, rtol=1e-5, atol=1e-6)
        assert abs(hf - hs[-1]) <= 1e-5 * max(1.0, abs(hs[-1]))


def test_mlgru_scan_slices_mode():
    B, T, d = 2, 40, 8
    fh, ch, gh = (rng.standard_normal((B, T, d)).astype(np.float32) for _ in range(3))
    H = rng.standard_normal((B, d)).astype(np.float32)
    o1, H1 = O.mlgru_scan(fh, ch, gh, H)
    with O.scan_slices(4):
        o4, H4 = O.mlgru_scan(fh, ch, gh, H)
    assert np.array_equal(o4[:, :10], o1[:, :10])          # slice 0 starts from the true state
    assert np.allclose(o4, o1, rtol=1e-5, atol=1e-6)
    assert np.allclose(H4, H1, rtol=1e-5, atol=1e-6)
    with O.scan_slices(8):                                  # tern_mlgru.num_chunks = 8
        o8, H8 = O.mlgru_scan(fh, ch, gh, H)
    assert np.array_equal(o8[:, :5], o1[:, :5])
    assert np.allclose(o8, o1, rtol=1e-5, atol=1e-6)
    assert np.allclose(H8, H1, rtol=1e-5, atol=1e-6)
    with O.scan_slices(1):
        assert np.array_equal(O.mlgru_scan(fh, ch, gh, H)[0], o1)


# ------------------------------------------------------------------ bf16 rounding points (C13)
# Reading C13: in bf16 mode values are rounded to bf16 (RNE) at R0 (block inputs /
# outputs), R1 (every BitLinear output), R2 (o' and p before their quantizer) and R3 (the
# residual stream), and NOWHERE else: h and every scale stay fp32.  These pins check the bf16
# mode of each oracle function against its fp32 mode plus a bf16 rounding done by torch (an
# independent implementation of RNE to bf16), so a missing, misplaced or extra rounding fails.
def _bf(x):
    torch = pytest.importorskip("torch")
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def _is_bf16(x):
    return np.array_equal(_bf(x), x)


def test_bf16_R1_bitlinear_output_only():
    # R1: the BitLinear output is rounded; its norm, quantizer and accumulator are not touched
    d, n = 48, 40
    r = np.random.default_rng(21)
    t, m = O.ternarize((r.standard_normal((n, d)) * 0.02).astype(np.float32))
    X = _bf(r.standard_normal((7, d)))                          # R0: bf16 input
    bias = r.standard_normal(n).astype(np.float32) * 0.1
    y32, tp32 = O.bitlinear(X, t, m, bias=bias, taps=True)
    y16, tp16 = O.bitlinear(X, t, m, bias=bias, bf16=True, taps=True)
    assert not _is_bf16(y32)                                    # the pin is not vacuous
    assert np.array_equal(y16, _bf(y32))
    for k in ("q", "acc", "deq"):
        assert np.array_equal(tp16[k], tp32[k])


def test_bf16_R2_scan_rounds_oprime_not_h():
    # R2 on o' only; the state h is fp32 (C13), identical in both modes
    B, T, d = 2, 33, 24
    r = np.random.default_rng(22)
    fh, ch, gh = (_bf(r.standard_normal((B, T, d)) * 2) for _ in range(3))
    H0 = r.standard_normal((B, d)).astype(np.float32)
    for gate in (0, 1):
        o32, H32 = O.mlgru_scan(fh, ch, gh, H0, gate_mode=gate)
        o16, H16 = O.mlgru_scan(fh, ch, gh, H0, gate_mode=gate, bf16=True)
        assert np.array_equal(H16, H32)
        assert not _is_bf16(H32)                                # h really is not rounded
        assert np.array_equal(o16, _bf(o32)) and not _is_bf16(o32)


def test_bf16_mlgru_rounding_points():
    # f̂ĉĝ (R1) are the rounded fp32-mode BitLinear outputs; the scan sees the rounded values;
    # o' (R2) and o (R1) are rounded; H is the fp32 recurrence of the rounded gates
    d = 32
    blk, _ = _blk(d, 48, 23)
    r = np.random.default_rng(23)
    X = _bf(r.standard_normal((2, 5, d)))
    H0 = np.zeros((2, d), np.float32)
    out, H, tp = O.mlgru(blk, X, H0, bf16=True, taps=True)
    Xf = X.reshape(-1, d)
    taps = {}
    for name, key in (("f", "fhat"), ("c", "chat"), ("g", "ghat")):
        taps[key] = _bf(O.bitlinear(Xf, blk.t[name], blk.m[name])).reshape(X.shape)
        assert np.array_equal(tp[key], taps[key])
    o32, Hs = O.mlgru_scan(taps["fhat"], taps["chat"], taps["ghat"], H0)
    assert np.array_equal(H, Hs) and not _is_bf16(H)
    assert np.array_equal(tp["oprime"], _bf(o32))
    assert np.array_equal(out.reshape(-1, d),
                          _bf(O.bitlinear(_bf(o32).reshape(-1, d), blk.t["o"], blk.m["o"])))


def test_bf16_glu_rounding_points():
    d, l = 24, 64
    blk, _ = _blk(d, l, 24)
    X = _bf(np.random.default_rng(24).standard_normal((5, d)))
    out, tp = O.glu(blk, X, bf16=True, taps=True)
    g = _bf(O.bitlinear(X, blk.t["gate"], blk.m["gate"]))      # R1
    u = _bf(O.bitlinear(X, blk.t["up"], blk.m["up"]))          # R1
    assert np.array_equal(tp["ghat"], g) and np.array_equal(tp["uhat"], u)
    p32 = (g * O.sigmoid_c(g)) * u
    assert not _is_bf16(p32)
    assert np.array_equal(tp["p"], _bf(p32))                    # R2
    assert np.array_equal(out, _bf(O.bitlinear(_bf(p32), blk.t["down"], blk.m["down"])))


def test_bf16_R3_block_residuals():
    # x1 = bf16(x + o), y = bf16(x1 + dn) (R3), o and dn themselves bf16 (R1); H unrounded
    d, l = 32, 64
    blk, _ = _blk(d, l, 25)
    X = _bf(np.random.default_rng(25).standard_normal((2, 6, d)))
    H0 = np.zeros((2, d), np.float32)
    Y, H, x1 = O.block(blk, X, H0, bf16=True, taps=True)
    o, Hm = O.mlgru(blk, X, H0, bf16=True)
    assert np.array_equal(H, Hm)
    assert not _is_bf16(X + o)
    assert np.array_equal(x1, _bf(X + o))
    dn = O.glu(blk, x1.reshape(-1, d), bf16=True)
    assert np.array_equal(Y.reshape(-1, d), _bf(x1.reshape(-1, d) + dn))
    assert _is_bf16(Y) and _is_bf16(x1)
