"""Plain CPU oracle of the MatMul-free LM block forward (arxiv 2406.02528).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with the CUDA path (``paper_2406_02528_b200``)
and never imports it; the product path never imports this package.

This module is a thin ctypes/numpy wrapper around ``oracle/oracle.c``; every
piece of arithmetic lives in that C file, which cites the paper line by line.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, no fp contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")


class MlgruW(C.Structure):
    _fields_ = [("tf", C.c_void_p), ("tc", C.c_void_p), ("tg", C.c_void_p), ("to", C.c_void_p),
                ("mf", C.c_float), ("mc", C.c_float), ("mg", C.c_float), ("mo", C.c_float),
                ("bf", C.c_void_p), ("bc", C.c_void_p), ("bg", C.c_void_p), ("bo", C.c_void_p),
                ("gain_x", C.c_void_p), ("gain_o", C.c_void_p)]


class GluW(C.Structure):
    _fields_ = [("tg", C.c_void_p), ("tu", C.c_void_p), ("td", C.c_void_p),
                ("mg", C.c_float), ("mu", C.c_float), ("md", C.c_float),
                ("gain_x", C.c_void_p), ("gain_p", C.c_void_p)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            L.orc_exp.restype = C.c_float
            L.orc_exp.argtypes = [C.c_float]
            L.orc_sigmoid.restype = C.c_float
            L.orc_sigmoid.argtypes = [C.c_float]
            L.orc_bf16.restype = C.c_float
            L.orc_bf16.argtypes = [C.c_float]
            for fn in ("orc_exp_arr", "orc_sigmoid_arr", "orc_bf16_arr"):
                getattr(L, fn).argtypes = [f32p, f32p, C.c_int64]
            L.orc_absmean.argtypes = [f32p, C.c_int64, C.POINTER(C.c_float)]
            L.orc_ternarize.argtypes = [f32p, C.c_int64, C.c_float, i8p]
            L.orc_zero_fraction.restype = C.c_double
            L.orc_zero_fraction.argtypes = [i8p, C.c_int64]
            L.orc_packed_row.restype = C.c_int64
            L.orc_packed_row.argtypes = [C.c_int64] * 4
            L.orc_unpack_segment.argtypes = [u32p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                             C.c_int, i8p]
            L.orc_set_norm_mode.argtypes = [C.c_int]
            L.orc_set_norm_mode.restype = None
            L.orc_get_norm_mode.restype = C.c_int
            L.orc_rmsnorm.restype = C.c_float
            L.orc_rmsnorm.argtypes = [f32p, C.c_int, C.c_void_p, C.c_float, f32p]
            L.orc_act_quant.restype = C.c_float
            L.orc_act_quant.argtypes = [f32p, C.c_int, i8p, C.POINTER(C.c_float)]
            L.orc_quant_rows.argtypes = [f32p, C.c_int, C.c_int, C.c_void_p, C.c_float, i8p, f32p,
                                         f32p, f32p]
            L.orc_tern_dot.restype = C.c_int64
            L.orc_tern_dot.argtypes = [i8p, i8p, C.c_int]
            L.orc_tern_matmul.argtypes = [i8p, C.c_int, C.c_int, i8p, C.c_int, i32p]
            L.orc_bitlinear.argtypes = [f32p, C.c_int, C.c_int, C.c_void_p, C.c_float, i8p, C.c_int,
                                        C.c_float, C.c_void_p, C.c_int, f32p, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
            L.orc_scan_seq.argtypes = [f32p, f32p, C.c_int, C.c_float, f32p]
            L.orc_scan_chunked.argtypes = [f32p, f32p, C.c_int, C.c_int, C.c_float, f32p]
            L.orc_mlgru_scan.argtypes = [f32p, f32p, f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                         C.c_int, f32p, f32p]
            L.orc_mlgru.argtypes = [C.POINTER(MlgruW), f32p, C.c_int, C.c_int, C.c_int, C.c_float,
                                    C.c_int, C.c_int, f32p, f32p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
            L.orc_glu.argtypes = [C.POINTER(GluW), f32p, C.c_int, C.c_int, C.c_int, C.c_float,
                                  C.c_int, f32p, C.c_void_p, C.c_void_p, C.c_void_p]
            L.orc_block.argtypes = [C.POINTER(MlgruW), C.POINTER(GluW), f32p, C.c_int, C.c_int,
                                    C.c_int, C.c_int, C.c_float, C.c_int, C.c_int, f32p, f32p,
                                    C.c_void_p]
            L.orc_swiglu_arr.argtypes = [f32p, f32p, C.c_int64, C.c_int, f32p]
            i16p = np.ctypeslib.ndpointer(np.int16, flags="C_CONTIGUOUS")
            u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
            L.orc_fxp_scales.argtypes = [f32p, C.c_int, C.c_int, i8p, C.POINTER(C.c_int)]
            L.orc_fxp_quant_act.argtypes = [f32p, C.c_int64, i16p, C.POINTER(C.c_int)]
            L.orc_fxp_sigmoid.restype = C.c_int32
            L.orc_fxp_sigmoid.argtypes = [C.c_int32]
            L.orc_fxp_sigmoid_arr.argtypes = [i32p, i32p, C.c_int64]
            L.orc_fxp_inv_sqrt_arr.argtypes = [u64p, i32p, C.c_int64, u32p, i32p]
            L.orc_fxp_rmsnorm.argtypes = [i16p, C.c_int, i8p, C.c_int, C.c_int, C.c_int,
                                          C.c_double, i16p, i32p]
            L.orc_fxp_bitlinear.argtypes = [i16p, C.c_int, i8p, C.c_int, C.c_double, i8p,
                                             C.c_float, C.c_int, C.c_int, C.c_int, i16p, i32p]
            L.orc_set_scan_slices.argtypes = [C.c_int]
            L.orc_set_scan_slices.restype = None
            L.orc_get_scan_slices.restype = C.c_int
            L.orc_scan_seqpar.argtypes = [f32p, f32p, C.c_int, C.c_int, C.c_float, f32p,
                                          C.POINTER(C.c_float)]
            f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
            L.orc_bitlinear_bwd.argtypes = [f32p, C.c_int, C.c_int, i8p, C.c_int, C.c_float,
                                            C.c_float, C.c_int, f32p, f64p, f64p, C.c_void_p]
            L.orc_set_threads.argtypes = [C.c_int]
            L.orc_get_threads.restype = C.c_int
            _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc:
        raise OracleError(f"{what}: oracle status {rc}")


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


# ---------------------------------------------------------------- scalars
def exp_c(x):
    x = _f32(x)
    y = np.empty_like(x)
    lib().orc_exp_arr(x.ravel(), y.ravel(), x.size)
    return y


def sigmoid_c(x):
    x = _f32(x)
    y = np.empty_like(x)
    lib().orc_sigmoid_arr(x.ravel(), y.ravel(), x.size)
    return y


def bf16_round(x):
    x = _f32(x)
    y = np.empty_like(x)
    lib().orc_bf16_arr(x.ravel(), y.ravel(), x.size)
    return y


# ---------------------------------------------------------------- a1
def absmean(W) -> float:
    W = _f32(W)
    m = C.c_float()
    _check(lib().orc_absmean(W.ravel(), W.size, C.byref(m)), "absmean")
    return float(np.float32(m.value))


def ternarize(W, m: float | None = None):
    """Return (t int8 same shape as W, m float32 scale)."""
    W = _f32(W)
    if m is None:
        m = absmean(W)
    t = np.empty(W.shape, dtype=np.int8)
    lib().orc_ternarize(W.ravel(), W.size, C.c_float(m), t.reshape(-1))
    return t, np.float32(m)


def zero_fraction(t) -> float:
    t = np.ascontiguousarray(t, dtype=np.int8)
    return float(lib().orc_zero_fraction(t.ravel(), t.size))


def packed_row(s, r, n_seg, seg_rows) -> int:
    return int(lib().orc_packed_row(s, r, n_seg, seg_rows))


def unpack_segment(codes, n, k, n_seg=1, s=0, seg_rows=64):
    """Decode segment ``s`` (n rows of k trits) of a packed uint32 array in the
    K-block-major layout [Kp/128][n_rows][8]."""
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    if codes.ndim == 2:                    # a single K-block [n_rows][8]
        codes = codes.reshape(1, *codes.shape)
    if codes.shape[-1] != 8 or codes.shape[0] * 128 < k:
        raise OracleError("unpack: codes must be [Kp/128][n_rows][8] covering k")
    t = np.empty((n, k), dtype=np.int8)
    _check(lib().orc_unpack_segment(codes.reshape(-1), codes.shape[1], n, k, n_seg, s, seg_rows,
                                    t.reshape(-1)), "unpack")
    return t


# ---------------------------------------------------------------- a2
class norm_mode:
    """Context manager: the oracle's norm variant, 0 = RMSNorm (C1), 1 = the
    centred form of Alg. 1 (reading C22)."""

    def __init__(self, mode: int):
        self.mode = int(mode)

    def __enter__(self):
        self.old = lib().orc_get_norm_mode()
        lib().orc_set_norm_mode(self.mode)
        return self

    def __exit__(self, *exc):
        lib().orc_set_norm_mode(self.old)
        return False


def rmsnorm(x, gain=None, eps=1e-6):
    x = _f32(x)
    y = np.empty_like(x)
    g = None if gain is None else _f32(gain)
    r = lib().orc_rmsnorm(x, x.size, _ptr(g), C.c_float(eps), y)
    return y, np.float32(r)


def act_quant(y):
    y = _f32(y)
    q = np.empty(y.shape, dtype=np.int8)
    deq = C.c_float()
    a = lib().orc_act_quant(y, y.size, q, C.byref(deq))
    return q, np.float32(deq.value), np.float32(a)


def quant_rows(X, gain=None, eps=1e-6):
    """Return q int8 [M][K], deq, inv_rms, absmax float32 [M]."""
    X = _f32(X)
    M, K = X.shape
    q = np.empty((M, K), dtype=np.int8)
    deq = np.empty(M, np.float32)
    r = np.empty(M, np.float32)
    a = np.empty(M, np.float32)
    g = None if gain is None else _f32(gain)
    _check(lib().orc_quant_rows(X, M, K, _ptr(g), C.c_float(eps), q, deq, r, a), "quant_rows")
    return q, deq, r, a


# ---------------------------------------------------------------- a3/a4
def tern_dot(t, q) -> int:
    t = np.ascontiguousarray(t, np.int8)
    q = np.ascontiguousarray(q, np.int8)
    return int(lib().orc_tern_dot(t, q, t.size))


def tern_matmul(q, t):
    q = np.ascontiguousarray(q, np.int8)
    t = np.ascontiguousarray(t, np.int8)
    M, K = q.shape
    N = t.shape[0]
    acc = np.empty((M, N), np.int32)
    _check(lib().orc_tern_matmul(q, M, K, t, N, acc), "tern_matmul")
    return acc


def bitlinear(X, t, m, gain=None, bias=None, eps=1e-6, bf16=False, taps=False):
    X = _f32(X)
    t = np.ascontiguousarray(t, np.int8)
    M, K = X.shape
    N = t.shape[0]
    O = np.empty((M, N), np.float32)
    g = None if gain is None else _f32(gain)
    b = None if bias is None else _f32(bias)
    q = np.empty((M, K), np.int8) if taps else None
    acc = np.empty((M, N), np.int32) if taps else None
    deq = np.empty(M, np.float32) if taps else None
    _check(lib().orc_bitlinear(X, M, K, _ptr(g), C.c_float(eps), t, N, C.c_float(m), _ptr(b),
                               int(bf16), O, _ptr(q), _ptr(acc), _ptr(deq)), "bitlinear")
    if taps:
        return O, dict(q=q, acc=acc, deq=deq)
    return O


def bitlinear_bwd(X, t, m, dO, eps=1e-6, norm=0):
    """Alg. 1 BackwardPass with the straight-through estimator (readings
    B1-B6): returns dX [M][K], dW [N][K], db [N] in float64.
    norm: 0 = RMSNorm (C1), 1 = Alg. 1's centred norm (C22)."""
    X = _f32(X)
    t = np.ascontiguousarray(t, np.int8)
    dO = _f32(dO)
    M, K = X.shape
    N = t.shape[0]
    dX = np.empty((M, K), np.float64)
    dW = np.empty((N, K), np.float64)
    db = np.empty(N, np.float64)
    _check(lib().orc_bitlinear_bwd(X, M, K, t, N, C.c_float(m), C.c_float(eps), int(norm), dO,
                                   dX, dW, _ptr(db)), "bitlinear_bwd")
    return dX, dW, db


# ---------------------------------------------------------------- a6
def scan_seq(f, c, h0=0.0):
    f = _f32(f)
    c = _f32(c)
    h = np.empty_like(f)
    lib().orc_scan_seq(f, c, f.size, C.c_float(h0), h)
    return h


def scan_chunked(f, c, chunk, h0=0.0):
    f = _f32(f)
    c = _f32(c)
    h = np.empty_like(f)
    lib().orc_scan_chunked(f, c, f.size, int(chunk), C.c_float(h0), h)
    return h


def mlgru_scan(fhat, chat, ghat, H, gate_mode=0, bf16=False):
    """fhat/chat/ghat [B][T][d]; H [B][d] (copied, returned updated). -> (oprime, H)."""
    fhat, chat, ghat = _f32(fhat), _f32(chat), _f32(ghat)
    B, T, d = fhat.shape
    H = _f32(H).copy()
    o = np.empty_like(fhat)
    _check(lib().orc_mlgru_scan(fhat, chat, ghat, B, T, d, int(gate_mode), int(bf16), H, o),
           "mlgru_scan")
    return o, H


def silu_mul(g, u, bf16=False):
    """GLU gating p = SiLU(g) * u, elementwise."""
    g, u = _f32(g), _f32(u)
    p = np.empty_like(g)
    lib().orc_swiglu_arr(g.ravel(), u.ravel(), g.size, int(bf16), p.ravel())
    return p


# ---------------------------------------------------------------- weights
class OracleBlock:
    """Ternarized weights of one block, built by the oracle from latent fp32
    weights (never from the GPU's packed codes)."""

    def __init__(self, latent: dict, d: int, l: int, biases: dict | None = None,
                 gains: dict | None = None, scales: dict | None = None):
        self.d, self.l = d, l
        self.t, self.m = {}, {}
        for name in ("f", "c", "g", "o", "gate", "up", "down"):
            t, m = ternarize(latent[name], None if scales is None else scales.get(name))
            self.t[name], self.m[name] = t, m
        biases = biases or {}
        gains = gains or {}
        self._keep = []
        keep = self._keep

        def P(a):
            if a is None:
                return None
            a = _f32(a)
            keep.append(a)
            return a.ctypes.data_as(C.c_void_p)

        tp = {k: v.ctypes.data_as(C.c_void_p) for k, v in self.t.items()}
        self.mw = MlgruW(tp["f"], tp["c"], tp["g"], tp["o"], self.m["f"], self.m["c"], self.m["g"],
                         self.m["o"], P(biases.get("f")), P(biases.get("c")), P(biases.get("g")),
                         P(biases.get("o")), P(gains.get("x")), P(gains.get("o")))
        self.gw = GluW(tp["gate"], tp["up"], tp["down"], self.m["gate"], self.m["up"],
                       self.m["down"], P(gains.get("x1")), P(gains.get("p")))


def mlgru(blk: OracleBlock, X, H, eps=1e-6, gate_mode=0, bf16=False, taps=False):
    X = _f32(X)
    B, T, d = X.shape
    H = _f32(H).copy()
    O = np.empty_like(X)
    tp = {k: np.empty_like(X) for k in ("fhat", "chat", "ghat", "oprime")} if taps else {}
    _check(lib().orc_mlgru(C.byref(blk.mw), X, B, T, d, C.c_float(eps), int(gate_mode), int(bf16),
                           H, O, _ptr(tp.get("fhat")), _ptr(tp.get("chat")),
                           _ptr(tp.get("ghat")), _ptr(tp.get("oprime"))), "mlgru")
    return (O, H, tp) if taps else (O, H)


def glu(blk: OracleBlock, X, eps=1e-6, bf16=False, taps=False):
    X = _f32(X)
    M, d = X.shape
    l = blk.l
    O = np.empty_like(X)
    tp = {k: np.empty((M, l), np.float32) for k in ("ghat", "uhat", "p")} if taps else {}
    _check(lib().orc_glu(C.byref(blk.gw), X, M, d, l, C.c_float(eps), int(bf16), O,
                         _ptr(tp.get("ghat")), _ptr(tp.get("uhat")), _ptr(tp.get("p"))), "glu")
    return (O, tp) if taps else O


def block(blk: OracleBlock, X, H, eps=1e-6, gate_mode=0, bf16=False, taps=False):
    """x1 = x + MLGRU(x); y = x1 + GLU(x1).  X [B][T][d]; H [B][d] -> (Y, H[, x1])."""
    X = _f32(X)
    B, T, d = X.shape
    H = _f32(H).copy()
    Y = np.empty_like(X)
    x1 = np.empty_like(X) if taps else None
    _check(lib().orc_block(C.byref(blk.mw), C.byref(blk.gw), X, B, T, d, blk.l, C.c_float(eps),
                           int(gate_mode), int(bf16), H, Y, _ptr(x1)), "block")
    return (Y, H, x1) if taps else (Y, H)


def stack(blocks, X, Hs, **kw):
    """Run blocks in order; Hs is a list of [B][d] states (returned updated)."""
    Hs = [np.array(h, np.float32, copy=True) for h in Hs]
    for i, blk in enumerate(blocks):
        X, Hs[i] = block(blk, X, Hs[i], **kw)
    return X, Hs


# ---------------------------------------------------------------- fixed-point W8A16 (f4(ii))
# PAPER.md P:499-518; readings F1-F5 in DESIGN.md.  Integer in, integer out.
FXP_XEXP, FXP_YEXP, FXP_NSIG = 6, 15, 8


def fxp_scales(w, shift=6):
    """F1: (w_q int8, e) with w ~ w_q 2^e, 2^e = 2^(round(log2 max|w|) - shift)."""
    w = _f32(w)
    wq = np.zeros(w.size, np.int8)
    e = C.c_int(0)
    _check(lib().orc_fxp_scales(w, w.size, int(shift), wq, C.byref(e)), "orc_fxp_scales")
    return wq, e.value


def fxp_quant_act(x):
    """F2: (q int16, e) with x ~ q 2^e, e the smallest fitting power of two."""
    x = _f32(x)
    q = np.zeros(x.shape, np.int16)
    e = C.c_int(0)
    _check(lib().orc_fxp_quant_act(x.reshape(-1), x.size, q.reshape(-1), C.byref(e)),
           "orc_fxp_quant_act")
    return q, e.value


def fxp_sigmoid(x):
    """F3: Q6 int32 inputs -> Q15 int32 sigma."""
    x = np.ascontiguousarray(x, dtype=np.int32)
    y = np.zeros(x.shape, np.int32)
    lib().orc_fxp_sigmoid_arr(x.reshape(-1), y.reshape(-1), x.size)
    return y


def fxp_inv_sqrt(v, e):
    """F4: 1/sqrt(v 2^e) ~ y 2^ey; returns (y uint32, ey int32)."""
    v = np.ascontiguousarray(v, dtype=np.uint64)
    e = np.ascontiguousarray(np.broadcast_to(np.asarray(e, np.int32), v.shape), dtype=np.int32)
    y = np.zeros(v.shape, np.uint32)
    ey = np.zeros(v.shape, np.int32)
    _check(lib().orc_fxp_inv_sqrt_arr(v.reshape(-1), e.reshape(-1), v.size, y.reshape(-1),
                                      ey.reshape(-1)), "orc_fxp_inv_sqrt")
    return y, ey


def fxp_rmsnorm(xq, ex, wq, ew, eps=1e-3):
    """F5 (Eq. 1, eps = 1e-3 P:510): int16 rows -> (int16 rows, per-row exponent)."""
    xq = np.ascontiguousarray(xq, dtype=np.int16)
    rows, d = xq.shape
    wq = np.ascontiguousarray(wq, dtype=np.int8)
    out = np.zeros((rows, d), np.int16)
    eo = np.zeros(rows, np.int32)
    _check(lib().orc_fxp_rmsnorm(xq, int(ex), wq, int(ew), rows, d, float(eps), out, eo),
           "orc_fxp_rmsnorm")
    return out, eo


def fxp_bitlinear(xq, ex, gq, eg, t, beta, eps=1e-3):
    """F6: W8A16 BitLinear, int16 rows [M][K] -> (int16 [M][N], exponent per row)."""
    xq = np.ascontiguousarray(xq, dtype=np.int16)
    M, K = xq.shape
    t = np.ascontiguousarray(t, dtype=np.int8)
    N = t.shape[0]
    y = np.zeros((M, N), np.int16)
    ey = np.zeros(M, np.int32)
    _check(lib().orc_fxp_bitlinear(xq, int(ex), np.ascontiguousarray(gq, dtype=np.int8), int(eg),
                                   float(eps), t, C.c_float(beta), M, K, N, y, ey),
           "orc_fxp_bitlinear")
    return y, ey


# ---------------------------------------------------------------- sequence-parallel scan (f3)
def scan_seqpar(f, c, W, h0=0.0):
    """Reading C23: W contiguous slices, slice aggregates composed in order, each slice
    scanned sequentially from its boundary state.  -> (h [T], final state)."""
    f, c = _f32(f), _f32(c)
    h = np.empty_like(f)
    hf = C.c_float(0.0)
    lib().orc_scan_seqpar(f, c, f.size, int(W), C.c_float(h0), h, C.byref(hf))
    return h, np.float32(hf.value)


class scan_slices:
    """Context manager: orc_mlgru_scan (and so mlgru / block / stack) uses the W-slice
    sequence-parallel scan of reading C23 while active."""

    def __init__(self, w: int):
        self.w = int(w)

    def __enter__(self):
        self.old = lib().orc_get_scan_slices()
        lib().orc_set_scan_slices(self.w)

    def __exit__(self, *exc):
        lib().orc_set_scan_slices(self.old)
