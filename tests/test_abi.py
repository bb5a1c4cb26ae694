"""The C-ABI library builds, loads and exports every symbol include/tern.h
declares; argument validation rejects bad calls before touching the GPU.
(CPU only: no compute calls.)"""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "tern.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?!typedef)(?:const\s+)?[a-z_0-9]+\s*\**\s+\**([a-z_0-9]+)\s*\(", src,
                       flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_02528_b200 import _lib, build
    build.build()
    return _lib.load()


def test_header_declares_the_north_star_entry_points():
    names = header_functions()
    for n in ("tern_pack", "bitlinear_fwd", "mlgru_fwd", "glu_fwd", "block_prefill", "block_decode"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    for n in header_functions():
        assert hasattr(lib, n), f"{n} declared in tern.h but not exported"


def test_binding_covers_every_symbol():
    from paper_2406_02528_b200 import _lib
    assert set(header_functions()) == set(_lib.EXPORTS)


def test_abi_version_and_host_helpers(lib):
    assert lib.tern_abi_version() == 1
    assert lib.tern_packed_rows(688, 2) == 2 * 704
    assert lib.tern_packed_rows(1024, 3) == 3072
    assert lib.tern_packed_rows(1000, 1) == 1000
    assert lib.tern_packed_ldw(688) == 48
    assert lib.tern_packed_ldw(1024) == 64


def test_validation_rejects_before_launch(lib):
    from paper_2406_02528_b200 import _lib as L
    st = lib.tern_quant(None, 0, 4, 256, 256, None, 1e-6, None, 256, None, None, None, None, None)
    assert st == L.TERN_ERR_INVALID_ARG
    assert b"null" in lib.tern_last_error()
    fake = C.c_void_p(0x1000)
    # K not a multiple of 16
    st = lib.tern_quant(fake, 0, 4, 250, 256, None, 1e-6, fake, 256, fake, fake, None, None, None)
    assert st == L.TERN_ERR_INVALID_ARG
    # misaligned pointer
    st = lib.tern_quant(C.c_void_p(0x1004), 0, 4, 256, 256, None, 1e-6, fake, 256, fake, fake,
                        None, None, None)
    assert st == L.TERN_ERR_INVALID_ARG
    # bad weight struct
    w = L.tern_weight(0x1000, 0x2000, 64, 128, 8, 1, 65)   # n_rows inconsistent
    y = C.c_void_p(0x3000)
    st = lib.bitlinear_fwd(fake, 0, 1, 128, 128, None, 1e-6, C.byref(w), None, y, 0, 64, None,
                           None, 0, None)
    assert st == L.TERN_ERR_INVALID_ARG and b"n_rows" in lib.tern_last_error()
    st = lib.tern_mlgru_scan(fake, 0, 1, 1, 100, 0, fake, fake, None)   # d % 64 != 0
    assert st == L.TERN_ERR_INVALID_ARG


def test_validation_of_the_later_entry_points(lib):
    """stack_decode, the knobs and the self-test reject bad arguments up front."""
    from paper_2406_02528_b200 import _lib as L
    fake = C.c_void_p(0x1000)
    harr = (C.c_void_p * 1)(0x2000)
    st = lib.stack_decode(None, 0, fake, fake, 0, 1, harr, fake, 1 << 20, None)
    assert st == L.TERN_ERR_INVALID_ARG and b"stack_decode" in lib.tern_last_error()
    ws = C.create_string_buffer(64)
    bad = C.c_uint64(0)
    assert lib.tern_selftest(9, ws, C.byref(bad)) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_stack_decode_workspace(None, 0, 1, 0) == 0
    # a block whose norm mode is out of range is rejected by the block checks
    w3 = L.tern_weight(0x1000, 0x2000, 256, 256, 16, 3, 768)
    w1 = L.tern_weight(0x1000, 0x2000, 256, 256, 16, 1, 256)
    wgu = L.tern_weight(0x1000, 0x2000, 688, 256, 16, 2, 2 * 704)
    wdn = L.tern_weight(0x1000, 0x2000, 256, 688, 48, 1, 256)
    mix = L.tern_mlgru(w3, w1, None, None, None, None, 0, 1e-6, 7)
    ch = L.tern_glu(wgu, wdn, None, None, 1e-6, 0)
    blk = L.tern_block(mix, ch, 256, 688)
    st = lib.block_decode(C.byref(blk), fake, C.c_void_p(0x5000), 0, 1, fake, fake, 1 << 30, None)
    assert st == L.TERN_ERR_INVALID_ARG and b"norm" in lib.tern_last_error()
    # knobs are clamped, not trusted
    old = lib.tern_get_norm_mode()
    lib.tern_set_norm_mode(5)
    assert lib.tern_get_norm_mode() == 0
    lib.tern_set_norm_mode(old)


def test_validation_of_the_fixed_point_entry_points(lib):
    """tern_fxp_* (f4(ii)) reject bad arguments before touching the device; empty calls are
    no-ops; the fused-scan knob is clamped."""
    from paper_2406_02528_b200 import _lib as L
    fake = C.c_void_p(0x1000)
    odd = C.c_void_p(0x1004)
    e = C.c_int32(0)
    assert lib.tern_fxp_scales(None, 4, 6, fake, C.byref(e), fake, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_scales(fake, 4, 7, fake, C.byref(e), fake, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_scales(fake, 4, 6, fake, C.byref(e), odd, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_quant_act(fake, 5, 4, fake, fake, fake, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_quant_act(None, 0, 0, None, None, None, None) == L.TERN_OK
    assert lib.tern_fxp_sigmoid(odd, 8, fake, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_sigmoid(None, 0, None, None) == L.TERN_OK
    assert lib.tern_fxp_inv_sqrt(odd, fake, 3, fake, fake, None) == L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_rmsnorm(fake, fake, fake, 0, 1e-3, 2, 0, fake, fake, None) == \
        L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_rmsnorm(fake, fake, fake, 0, 1e-3, 2, 70000, fake, fake, None) == \
        L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_rmsnorm(odd, fake, fake, 0, 1e-3, 2, 64, fake, fake, None) == \
        L.TERN_ERR_INVALID_ARG
    assert lib.tern_fxp_rmsnorm(fake, fake, fake, 0, -1.0, 2, 64, fake, fake, None) == \
        L.TERN_ERR_INVALID_ARG
    assert b"tern_fxp_rmsnorm" in lib.tern_last_error()
    assert lib.tern_fxp_rmsnorm(None, None, None, 0, 1e-3, 0, 64, None, None, None) == L.TERN_OK
    old = lib.tern_get_fused_scan()
    lib.tern_set_fused_scan(9)
    assert lib.tern_get_fused_scan() == 2
    lib.tern_set_fused_scan(-3)
    assert lib.tern_get_fused_scan() == 0
    lib.tern_set_fused_scan(old)


def test_validation_of_the_backward_and_qfuse_knobs(lib):
    """bitlinear_bwd (f4(iii)) rejects bad arguments before any launch: k % 16, a fused
    group (n_seg != 1), a weight without its u8 copy, a bad norm, a short workspace;
    the workspace query; the f3 / backward knobs read back what was set."""
    from paper_2406_02528_b200 import _lib as L
    fake = C.c_void_p(0x1000)
    w1 = L.tern_weight(0x1000, 0x2000, 64, 128, 8, 1, 64)
    w1.e8 = 0x4000
    ws = 1 << 30
    bw = lib.bitlinear_bwd
    assert bw(fake, 0, 4, 120, C.byref(w1), 1e-6, 0, fake, fake, fake, None, fake, ws, None) == \
        L.TERN_ERR_INVALID_ARG
    w3 = L.tern_weight(0x1000, 0x2000, 64, 128, 8, 3, 192)
    w3.e8 = 0x4000
    assert bw(fake, 0, 4, 128, C.byref(w3), 1e-6, 0, fake, fake, fake, None, fake, ws, None) == \
        L.TERN_ERR_INVALID_ARG
    w0 = L.tern_weight(0x1000, 0x2000, 64, 128, 8, 1, 64)   # no e8
    assert bw(fake, 0, 4, 128, C.byref(w0), 1e-6, 0, fake, fake, fake, None, fake, ws, None) == \
        L.TERN_ERR_INVALID_ARG and b"e8" in lib.tern_last_error()
    assert bw(fake, 0, 4, 128, C.byref(w1), 1e-6, 3, fake, fake, fake, None, fake, ws, None) == \
        L.TERN_ERR_INVALID_ARG and b"norm" in lib.tern_last_error()
    need = lib.bitlinear_bwd_workspace(4, 128, 64)
    assert need > 4 * 128 * 4
    assert bw(fake, 0, 4, 128, C.byref(w1), 1e-6, 0, fake, fake, fake, None, fake, need - 16, None) \
        == L.TERN_ERR_INVALID_ARG and b"workspace" in lib.tern_last_error()
    assert lib.bitlinear_bwd_workspace(0, 128, 64) == 0
    for get, put in ((lib.tern_get_qfuse, lib.tern_set_qfuse),
                     (lib.tern_get_bwd_tc, lib.tern_set_bwd_tc)):
        old = get()
        put(7)
        assert get() == 1
        put(0)
        assert get() == 0
        put(old)


def test_product_path_has_no_fallback(tmp_path, monkeypatch):
    """The binding raises when the CUDA library is missing (no CPU fallback)."""
    import importlib
    monkeypatch.setenv("TERN_LIB", str(tmp_path / "missing.so"))
    import paper_2406_02528_b200._lib as mod
    m2 = importlib.reload(mod)
    try:
        with pytest.raises(OSError):
            m2.load()
    finally:
        monkeypatch.delenv("TERN_LIB")
        importlib.reload(mod)


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2406_02528_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "oracle.h" not in txt and "liboracle" not in txt, f
