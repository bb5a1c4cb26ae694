"""ctypes binding of libtern.so (include/tern.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  Function names match the C ABI.  There is no fallback: if the
shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TERN_LIB", os.path.join(_HERE, "libtern.so"))

TERN_OK, TERN_ERR_INVALID_ARG, TERN_ERR_DEGENERATE, TERN_ERR_UNSUPPORTED, TERN_ERR_CUDA = range(5)
TERN_F32, TERN_BF16 = 0, 1
TERN_GATE_SIGMOID_H, TERN_GATE_LINEAR_H = 0, 1
TERN_NORM_RMS, TERN_NORM_CENTERED = 0, 1


class TernError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[tern status {status}] {msg}")
        self.status = status


class tern_weight(C.Structure):
    _fields_ = [("codes", C.c_void_p), ("scales", C.c_void_p), ("n_out", C.c_int32),
                ("k", C.c_int32), ("ldw", C.c_int32), ("n_seg", C.c_int32),
                ("n_rows", C.c_int32), ("e8", C.c_void_p)]


class tern_bl_taps(C.Structure):
    _fields_ = [("q", C.c_void_p), ("ldq", C.c_int32), ("acc", C.c_void_p), ("ldacc", C.c_int32),
                ("deq", C.c_void_p), ("inv_rms", C.c_void_p), ("absmax", C.c_void_p)]


class tern_mlgru(C.Structure):
    _fields_ = [("fcg", tern_weight), ("o", tern_weight), ("gain_x", C.c_void_p),
                ("gain_o", C.c_void_p), ("bias_fcg", C.c_void_p), ("bias_o", C.c_void_p),
                ("gate", C.c_int), ("eps", C.c_float), ("norm", C.c_int),
                ("num_chunks", C.c_int32)]


class tern_glu(C.Structure):
    _fields_ = [("gu", tern_weight), ("down", tern_weight), ("gain_x", C.c_void_p),
                ("gain_p", C.c_void_p), ("eps", C.c_float), ("norm", C.c_int)]


# int ag(void* ctx, const void* send, void* recv, size_t bytes_per_rank, cudaStream_t stream)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


# int ar(void* ctx, const int32_t* send, int32_t* recv, size_t count, cudaStream_t stream)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)


class tern_shard(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("ag", ALLGATHER_FN),
                ("ctx", C.c_void_p), ("gather_q", C.c_int32), ("megatron", C.c_int32),
                ("ar", ALLREDUCE_FN)]


class tern_seqpar(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("ag", ALLGATHER_FN),
                ("ctx", C.c_void_p)]


class tern_block(C.Structure):
    _fields_ = [("mix", tern_mlgru), ("ch", tern_glu), ("d", C.c_int32), ("l", C.c_int32),
                ("shard", tern_shard), ("next_block", C.c_void_p)]


class tern_block_taps(C.Structure):
    _fields_ = [("fcg", C.c_size_t), ("oprime", C.c_size_t), ("x1", C.c_size_t),
                ("p", C.c_size_t)]


class tern_prof_rec(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("epi", C.c_int32), ("m", C.c_int32), ("n", C.c_int32),
                ("k", C.c_int32), ("n_seg", C.c_int32), ("dtype", C.c_int32), ("ms", C.c_float)]


KERNEL_NAMES = {0: "quant", 1: "gemv", 2: "gemm_tc", 3: "scan", 4: "fcgscan", 5: "stack", 6: "fin", 7: "gemm_qf"}

P = C.c_void_p
I32 = C.c_int32
SZ = C.c_size_t
F = C.c_float
_SIGS = {
    "tern_abi_version": (C.c_int, []),
    "tern_last_error": (C.c_char_p, []),
    "tern_packed_rows": (I32, [I32, I32]),
    "tern_packed_ldw": (I32, [I32]),
    "tern_codes_init": (C.c_int, [P, I32, I32, P]),
    "tern_pack_workspace": (SZ, [I32, I32]),
    "tern_pack": (C.c_int, [P, I32, I32, P, I32, I32, P, I32, P, P, SZ, P]),
    "tern_expand": (C.c_int, [C.POINTER(tern_weight), P, P]),
    "tern_quant": (C.c_int, [P, C.c_int, I32, I32, I32, P, F, P, I32, P, P, P, P, P]),
    "tern_bitlinear_workspace": (SZ, [I32, I32]),
    "bitlinear_fwd": (C.c_int, [P, C.c_int, I32, I32, I32, P, F, C.POINTER(tern_weight), P, P,
                                C.c_int, I32, C.POINTER(tern_bl_taps), P, SZ, P]),
    "tern_contract": (C.c_int, [P, I32, I32, P, C.POINTER(tern_weight), P, I32, P]),
    "bitlinear_bwd_workspace": (SZ, [I32, I32, I32]),
    "bitlinear_bwd": (C.c_int, [P, C.c_int, I32, I32, C.POINTER(tern_weight), F, I32, P, P, P, P,
                                P, SZ, P]),
    "tern_mlgru_scan": (C.c_int, [P, C.c_int, I32, I32, I32, C.c_int, P, P, P]),
    "tern_mlgru_workspace": (SZ, [C.POINTER(tern_mlgru), I32, I32, I32, C.c_int]),
    "tern_mlgru_chunks": (I32, [C.POINTER(tern_mlgru), I32, I32, I32]),
    "tern_glu_workspace": (SZ, [C.POINTER(tern_glu), I32, I32, I32, C.c_int]),
    "tern_block_workspace": (SZ, [C.POINTER(tern_block), I32, I32, C.c_int]),
    "tern_block_ws_layout": (C.c_int, [C.POINTER(tern_block), I32, I32, C.c_int,
                                       C.POINTER(tern_block_taps)]),
    "mlgru_fwd": (C.c_int, [C.POINTER(tern_mlgru), P, P, C.c_int, I32, I32, I32, P, P, SZ, P]),
    "glu_fwd": (C.c_int, [C.POINTER(tern_glu), P, P, C.c_int, I32, I32, I32, P, SZ, P]),
    "block_prefill": (C.c_int, [C.POINTER(tern_block), P, P, C.c_int, I32, I32, P, P, SZ, P]),
    "block_decode": (C.c_int, [C.POINTER(tern_block), P, P, C.c_int, I32, P, P, SZ, P]),
    "tern_stack_decode_workspace": (SZ, [C.POINTER(tern_block), I32, I32, C.c_int]),
    "stack_decode": (C.c_int, [C.POINTER(tern_block), I32, P, P, C.c_int, I32,
                               C.POINTER(C.c_void_p), P, SZ, P]),
    "tern_profile_enable": (None, [I32]),
    "tern_trace_enable": (None, [I32]),
    "tern_trace_collect": (I32, [C.c_void_p, I32]),
    "tern_profile_collect": (I32, [C.POINTER(tern_prof_rec), I32]),
    "tern_selftest": (C.c_int, [I32, P, C.POINTER(C.c_uint64)]),
    "tern_set_gemv_max_m": (None, [I32]),
    "tern_get_gemv_max_m": (I32, []),
    "tern_set_fused_scan": (None, [I32]),
    "tern_get_fused_scan": (I32, []),
    "tern_set_batched_fin": (None, [I32]),
    "tern_set_gemm_sab": (None, [I32]),
    "tern_set_gemm_2sm": (None, [I32]),
    "tern_set_qfuse": (None, [I32]),
    "tern_set_bwd_tc": (None, [I32]),
    "tern_get_bwd_tc": (I32, []),
    "tern_get_qfuse": (I32, []),
    "tern_get_gemm_2sm": (I32, []),
    "tern_get_gemm_sab": (I32, []),
    "tern_set_norm_mode": (None, [C.c_int]),
    "tern_get_norm_mode": (C.c_int, []),
    "tern_get_batched_fin": (I32, []),
    "tern_block_prefill_sp_workspace": (SZ, [C.POINTER(tern_block), I32, I32, C.c_int, I32]),
    "block_prefill_sp": (C.c_int, [C.POINTER(tern_block), P, P, C.c_int, I32, I32, P,
                                   C.POINTER(tern_seqpar), P, SZ, P]),
    "tern_fxp_scales": (C.c_int, [P, I32, I32, P, C.POINTER(I32), P, P]),
    "tern_fxp_quant_act": (C.c_int, [P, C.c_int, C.c_int64, P, P, P, P]),
    "tern_fxp_sigmoid": (C.c_int, [P, C.c_int64, P, P]),
    "tern_fxp_inv_sqrt": (C.c_int, [P, P, C.c_int64, P, P, P]),
    "tern_fxp_rmsnorm": (C.c_int, [P, P, P, I32, C.c_double, I32, I32, P, P, P]),
    "tern_fxp_bitlinear_workspace": (SZ, [I32, I32, I32]),
    "tern_fxp_bitlinear": (C.c_int, [P, P, I32, I32, P, I32, C.c_double, C.POINTER(tern_weight),
                                     P, I32, P, P, SZ, P]),
}
EXPORTS = tuple(_SIGS)

_lib = None


def load():
    """Load libtern.so (raises OSError if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"libtern.so not found at {LIB_PATH}; run "
                          f"`python -m paper_2406_02528_b200.build` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != TERN_OK:
        msg = load().tern_last_error()
        raise TernError(st, f"{what}: {msg.decode() if msg else ''}")


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float32:
        return TERN_F32
    if dt == torch.bfloat16:
        return TERN_BF16
    raise TypeError(f"unsupported activation dtype {dt}")


def stream_handle(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


# ------------------------------------------------------------------ wrappers with C names
def tern_packed_rows(n_out: int, n_seg: int) -> int:
    return int(load().tern_packed_rows(n_out, n_seg))


def tern_packed_ldw(k: int) -> int:
    return int(load().tern_packed_ldw(k))


def tern_codes_init(codes: torch.Tensor, stream=None):
    """codes: int32 [Kp/128][n_rows][8] (K-block-major packed layout)."""
    nkb, n_rows, _ = codes.shape
    _check(load().tern_codes_init(ptr(codes), n_rows, nkb * 8, stream_handle(stream)),
           "tern_codes_init")


def tern_pack(W: torch.Tensor, codes: torch.Tensor, scale_out: torch.Tensor, n_seg=1, seg_idx=0,
              scale_in: torch.Tensor | None = None, stream=None):
    """Ternarize + pack fp32 W [n][k] (device) into segment seg_idx of codes."""
    assert W.is_cuda and W.dtype == torch.float32 and W.is_contiguous()
    n, k = W.shape
    L = load()
    wsb = int(L.tern_pack_workspace(n, k))
    ws = torch.empty(wsb, dtype=torch.uint8, device=W.device)
    _check(L.tern_pack(ptr(W), n, k, ptr(scale_in), n_seg, seg_idx, ptr(codes), codes.shape[1],
                       ptr(scale_out), ptr(ws), wsb, stream_handle(stream)), "tern_pack")


def tern_expand(w: tern_weight, e8: torch.Tensor, stream=None):
    _check(load().tern_expand(C.byref(w), ptr(e8), stream_handle(stream)), "tern_expand")


def tern_quant(x: torch.Tensor, q: torch.Tensor, deq: torch.Tensor, qsum: torch.Tensor,
               gain=None, eps=1e-6, inv_rms=None, absmax=None, stream=None):
    m, k = x.shape
    _check(load().tern_quant(ptr(x), dtype_code(x.dtype), m, k, x.stride(0), ptr(gain), eps,
                             ptr(q), q.stride(0), ptr(deq), ptr(qsum), ptr(inv_rms), ptr(absmax),
                             stream_handle(stream)), "tern_quant")


def bitlinear_fwd(x, w: tern_weight, y, gain=None, bias=None, eps=1e-6, taps=None, ws=None,
                  stream=None):
    m, k = x.shape
    L = load()
    need = int(L.tern_bitlinear_workspace(m, k))
    if ws is None:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    tp = None
    if taps is not None:
        tp = tern_bl_taps(ptr(taps.get("q")), taps["q"].stride(0) if taps.get("q") is not None else 0,
                          ptr(taps.get("acc")),
                          taps["acc"].stride(0) if taps.get("acc") is not None else 0,
                          ptr(taps.get("deq")), ptr(taps.get("inv_rms")), ptr(taps.get("absmax")))
    _check(L.bitlinear_fwd(ptr(x), dtype_code(x.dtype), m, k, x.stride(0), ptr(gain), eps,
                           C.byref(w), ptr(bias), ptr(y), dtype_code(y.dtype), y.stride(0),
                           C.byref(tp) if tp is not None else None, ptr(ws), ws.numel(),
                           stream_handle(stream)), "bitlinear_fwd")


def bitlinear_bwd(x, w: tern_weight, dO, dX, dW, db=None, eps=1e-6, norm=TERN_NORM_RMS,
                  ws=None, stream=None):
    """Alg. 1 BackwardPass of one BitLinear (include/tern.h): x and dO fp32 or
    bf16 (same dtype), fp32 dX, dW, db."""
    m, k = x.shape
    L = load()
    need = int(L.bitlinear_bwd_workspace(m, k, w.n_out))
    if ws is None:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=x.device)
    _check(L.bitlinear_bwd(ptr(x), dtype_code(x.dtype), m, k, C.byref(w), eps, int(norm), ptr(dO),
                           ptr(dX), ptr(dW), ptr(db), ptr(ws), ws.numel(), stream_handle(stream)),
           "bitlinear_bwd")


def tern_contract(q, qsum, w: tern_weight, acc, stream=None):
    m = q.shape[0]
    _check(load().tern_contract(ptr(q), m, q.stride(0), ptr(qsum), C.byref(w), ptr(acc),
                                acc.stride(0), stream_handle(stream)), "tern_contract")


def tern_mlgru_scan(fcg, B, T, d, h, oprime, gate=TERN_GATE_SIGMOID_H, stream=None):
    _check(load().tern_mlgru_scan(ptr(fcg), dtype_code(fcg.dtype), B, T, d, gate, ptr(h),
                                  ptr(oprime), stream_handle(stream)), "tern_mlgru_scan")


def mlgru_fwd(p: tern_mlgru, x, out, h, ws, stream=None):
    B, T, d = x.shape
    _check(load().mlgru_fwd(C.byref(p), ptr(x), ptr(out), dtype_code(x.dtype), B, T, d, ptr(h),
                            ptr(ws), ws.numel(), stream_handle(stream)), "mlgru_fwd")


def glu_fwd(p: tern_glu, x, out, l, ws, stream=None):
    m, d = x.shape
    _check(load().glu_fwd(C.byref(p), ptr(x), ptr(out), dtype_code(x.dtype), m, d, l, ptr(ws),
                          ws.numel(), stream_handle(stream)), "glu_fwd")


def block_prefill(b: tern_block, x, y, h, ws, stream=None):
    B, T, d = x.shape
    _check(load().block_prefill(C.byref(b), ptr(x), ptr(y), dtype_code(x.dtype), B, T, ptr(h),
                                ptr(ws), ws.numel(), stream_handle(stream)), "block_prefill")


def block_decode(b: tern_block, x, y, h, ws, stream=None):
    B = x.shape[0]
    _check(load().block_decode(C.byref(b), ptr(x), ptr(y), dtype_code(x.dtype), B, ptr(h),
                               ptr(ws), ws.numel(), stream_handle(stream)), "block_decode")


def tern_stack_decode_workspace(blocks, B: int, dt: torch.dtype) -> int:
    """blocks: ctypes array of tern_block."""
    return int(load().tern_stack_decode_workspace(blocks, len(blocks), B, dtype_code(dt)))


def stack_decode(blocks, x, y, hs, ws, stream=None, allow_unsupported=False) -> int:
    """One decode step through the whole stack in one launch (tern.h stack_decode).
    blocks: ctypes array of tern_block; hs: list of per-block fp32 states.
    With allow_unsupported, TERN_ERR_UNSUPPORTED is returned instead of raised."""
    B = x.shape[0]
    harr = (C.c_void_p * len(hs))(*[h.data_ptr() for h in hs])
    st = load().stack_decode(blocks, len(blocks), ptr(x), ptr(y), dtype_code(x.dtype), B, harr,
                             ptr(ws), ws.numel(), stream_handle(stream))
    if st == TERN_ERR_UNSUPPORTED and allow_unsupported:
        load().tern_last_error()
        return st
    _check(st, "stack_decode")
    return st


def tern_set_gemv_max_m(m: int):
    load().tern_set_gemv_max_m(int(m))


def tern_set_fused_scan(mode):
    """True / 2: always the fused f|c|g+scan kernel; False / 0: never; 1: by grid size (default)."""
    if isinstance(mode, bool):
        mode = 2 if mode else 0
    load().tern_set_fused_scan(int(mode))


def tern_set_norm_mode(mode: int):
    """Norm variant of tern_quant / bitlinear_fwd (0 RMSNorm, 1 centred, Alg. 1)."""
    load().tern_set_norm_mode(int(mode))


def tern_get_norm_mode() -> int:
    return int(load().tern_get_norm_mode())


def tern_set_batched_fin(on: bool):
    load().tern_set_batched_fin(1 if on else 0)


def tern_set_gemm_sab(on: bool):
    load().tern_set_gemm_sab(1 if on else 0)


def tern_set_gemm_2sm(on: bool):
    load().tern_set_gemm_2sm(1 if on else 0)


def tern_set_qfuse(on: bool):
    """f3: the a2 quantization fused into the prefill GEMMs (opt-in, include/tern.h)."""
    load().tern_set_qfuse(1 if on else 0)


def tern_get_qfuse() -> bool:
    return bool(load().tern_get_qfuse())


def tern_set_bwd_tc(on: bool):
    """Backward contractions on the tensor cores (default) or fp32 CUDA cores."""
    load().tern_set_bwd_tc(1 if on else 0)


def tern_get_bwd_tc() -> bool:
    return bool(load().tern_get_bwd_tc())


def tern_get_gemm_2sm() -> bool:
    return bool(load().tern_get_gemm_2sm())


def tern_get_gemm_sab() -> bool:
    return bool(load().tern_get_gemm_sab())


def tern_get_batched_fin() -> bool:
    return bool(load().tern_get_batched_fin())


def tern_get_fused_scan() -> int:
    return int(load().tern_get_fused_scan())


def tern_get_gemv_max_m() -> int:
    return int(load().tern_get_gemv_max_m())


def tern_trace_enable(on: bool):
    load().tern_trace_enable(1 if on else 0)


def tern_trace_collect(with_kind=False):
    """-> list of (ctas, array[ctas][16]: start, released, end, ...), or with_kind
    (kind, ctas, array) with kind a tern_kernel_id (+16: split-K epilogue)."""
    import numpy as np
    Lb = load()
    n = int(Lb.tern_trace_collect(None, 0))
    rec = 1 + 1024 * 16
    buf = np.zeros(n * rec, dtype=np.uint64)
    n = int(Lb.tern_trace_collect(buf.ctypes.data_as(C.c_void_p), n))
    out = []
    for i in range(n):
        r = buf[i * rec:(i + 1) * rec]
        u, kind = int(r[0]) & 0xFFFFF, int(r[0]) >> 20
        arr = r[1:1 + 16 * u].reshape(u, 16).astype(np.int64)
        out.append((kind, u, arr) if with_kind else (u, arr))
    return out


def tern_profile_enable(on: bool):
    load().tern_profile_enable(1 if on else 0)


def tern_profile_collect() -> list:
    """Per-launch records [(kernel name, dict(meta), ms)] of the library's kernels."""
    Lb = load()
    n = int(Lb.tern_profile_collect(None, 0))
    arr = (tern_prof_rec * max(n, 1))()
    n = int(Lb.tern_profile_collect(arr, n))
    out = []
    for r in arr[:n]:
        out.append({"kernel": KERNEL_NAMES.get(r.kernel, str(r.kernel)), "epi": r.epi, "m": r.m,
                    "n": r.n, "k": r.k, "n_seg": r.n_seg, "dtype": r.dtype, "ms": float(r.ms)})
    return out


# ---------------------------------------------------------------- sequence-parallel prefill (f3)
def block_prefill_sp(blk, x, y, h, sp: tern_seqpar, ws, B: int, T_local: int, dt,
                     stream=None):
    """One block over this rank's token slice x [B][T_local][d] (tern.h block_prefill_sp)."""
    _check(load().block_prefill_sp(C.byref(blk), ptr(x), ptr(y), dtype_code(dt), B, T_local,
                                   ptr(h), C.byref(sp), ptr(ws), ws.numel(),
                                   stream_handle(stream)), "block_prefill_sp")


# ---------------------------------------------------------------- fixed point W8A16 (f4(ii))
def tern_fxp_scales(w: torch.Tensor, shift: int = 6, stream=None):
    """F1: fp32 gains [n] (device) -> (int8 wq [n] device tensor, exponent e)."""
    wq = torch.empty(w.numel(), dtype=torch.int8, device=w.device)
    ws = torch.zeros(16, dtype=torch.uint8, device=w.device)
    e = I32(0)
    _check(load().tern_fxp_scales(ptr(w), w.numel(), int(shift), ptr(wq), C.byref(e), ptr(ws),
                                  stream_handle(stream)), "tern_fxp_scales")
    return wq, int(e.value)


def tern_fxp_quant_act(x: torch.Tensor, q: torch.Tensor, e: torch.Tensor, ws=None, stream=None):
    """F2: x (fp32/bf16) -> q int16 (same numel), e int32 [1] (device)."""
    if ws is None:
        ws = torch.empty(16, dtype=torch.uint8, device=x.device)
    _check(load().tern_fxp_quant_act(ptr(x), dtype_code(x.dtype), x.numel(), ptr(q), ptr(e),
                                     ptr(ws), stream_handle(stream)), "tern_fxp_quant_act")


def tern_fxp_sigmoid(x: torch.Tensor, y: torch.Tensor, stream=None):
    """F3: int32 Q6 -> int32 Q15."""
    _check(load().tern_fxp_sigmoid(ptr(x), x.numel(), ptr(y), stream_handle(stream)),
           "tern_fxp_sigmoid")


def tern_fxp_inv_sqrt(v: torch.Tensor, e: torch.Tensor, y: torch.Tensor, ey: torch.Tensor,
                      stream=None):
    """F4: v (uint64 as int64 storage) and e int32 -> y (uint32 as int32 storage), ey int32."""
    _check(load().tern_fxp_inv_sqrt(ptr(v), ptr(e), v.numel(), ptr(y), ptr(ey),
                                    stream_handle(stream)), "tern_fxp_inv_sqrt")


def tern_fxp_rmsnorm(xq: torch.Tensor, ex: torch.Tensor, wq: torch.Tensor, ew: int,
                     out: torch.Tensor, eo: torch.Tensor, eps: float = 1e-3, stream=None):
    """F5: int16 rows [rows][d] (exponent ex: device int32 [1]) -> int16 rows, int32 [rows]."""
    rows, d = xq.shape
    _check(load().tern_fxp_rmsnorm(ptr(xq), ptr(ex), ptr(wq), int(ew), float(eps), rows, d,
                                   ptr(out), ptr(eo), stream_handle(stream)), "tern_fxp_rmsnorm")


def tern_fxp_bitlinear(xq: torch.Tensor, ex: torch.Tensor, gq: torch.Tensor, eg: int,
                       w: tern_weight, y: torch.Tensor, ey: torch.Tensor, eps: float = 1e-3,
                       ws=None, stream=None):
    """F6: W8A16 BitLinear, int16 [m][k] -> int16 [m][n_out] + int32 exponents [m]."""
    m, k = xq.shape
    L = load()
    need = int(L.tern_fxp_bitlinear_workspace(m, k, w.n_rows))
    if ws is None:
        ws = torch.empty(max(need, 16), dtype=torch.uint8, device=xq.device)
    _check(L.tern_fxp_bitlinear(ptr(xq), ptr(ex), m, k, ptr(gq), int(eg), float(eps), C.byref(w),
                                ptr(y), y.stride(0), ptr(ey), ptr(ws), ws.numel(),
                                stream_handle(stream)), "tern_fxp_bitlinear")


def tern_selftest(which: int) -> int:
    ws = torch.zeros(128, dtype=torch.uint8, device="cuda")
    out = C.c_uint64(0)
    _check(load().tern_selftest(int(which), ptr(ws), C.byref(out)), "tern_selftest")
    return int(out.value)
