"""The C-ABI library loads and exports exactly what include/hwb.h declares; its
argument validation (which runs before any CUDA call) maps to TfheError.
CPU only: no entry point here reaches the GPU."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_2403_20190_b200 import _lib
from paper_2403_20190_b200.params import named_params


def header_symbols():
    text = open(os.path.join(REPO, "include", "hwb.h")).read()
    return sorted(set(re.findall(r"\b(hwb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    declared = header_symbols()
    assert declared == sorted(_lib.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name
    assert L.hwb_version() == 1


def test_ggsw_words():
    cp = _lib.c_params(named_params("CFG2"))
    assert _lib.load().hwb_ggsw_ntt_words(ctypes.byref(cp)) == 6 * 2 * 2 * 1024


def _ext(cp):
    null = ctypes.c_void_p(0)
    return _lib.load().hwb_ext_product(ctypes.byref(cp), null, null, null, null, 1, null)


@pytest.mark.parametrize("field,value,msg", [
    ("q_bits", 64, "q_bits"), ("N", 512, "ring degree"), ("k", 2, "GLWE"),
    ("l", 4, "levels"), ("base_log", 12, "spans"),
])
def test_invalid_params_rejected_before_cuda(field, value, msg):
    cp = _lib.c_params(named_params("CFG2"))
    setattr(cp, field, value)
    rc = _ext(cp)
    assert rc == _lib.HWB_EINVAL
    assert msg in _lib.load().hwb_last_error().decode()
    with pytest.raises(_lib.TfheError):
        _lib.check(rc)


def test_exactness_envelope():
    # a 2 x 16-bit gadget at N = 1024 would overflow the two-prime CRT range
    cp = _lib.c_params(named_params("CFG2"))
    cp.l, cp.base_log = 2, 16
    assert _ext(cp) == _lib.HWB_EINVAL
    assert "2-prime" in _lib.load().hwb_last_error().decode()
    for name in ("CFG1", "CFG2", "CFG4", "INSECURE_1024", "INSECURE_2048"):
        cp = _lib.c_params(named_params(name))
        null = ctypes.c_void_p(0)
        # B = 0 passes validation and returns before touching the device
        assert _lib.load().hwb_ext_product(ctypes.byref(cp), null, null, null, null, 0, null) == 0


def test_keyswitch_validation():
    cp = _lib.c_params(named_params("CFG2"))
    cp.ks_l = 0
    null = ctypes.c_void_p(0)
    assert _lib.load().hwb_keyswitch(ctypes.byref(cp), null, null, null, 1, null) == _lib.HWB_EINVAL
    cp = _lib.c_params(named_params("CFG2"))
    assert _lib.load().hwb_sample_extract(ctypes.byref(cp), null, null, 1, 1024, null) == _lib.HWB_EINVAL


def test_variant_switch_validation():
    with pytest.raises(_lib.TfheError):
        _lib.set_variant(7)
    _lib.set_variant(0)


def test_tensor_core_keyswitch_sizes_and_validation():
    """hwb_ksk_tc_bytes / workspace sizes and argument checks (host-only)."""
    L = _lib.load()
    P = named_params("CFG2")                       # n = 630, N = 1024, KS 2^2 x 8
    cp = _lib.c_params(P)
    n_col_tiles, k_blocks = (P.lwe_n + 1 + 63) // 64, 1024 * 8 // 128
    assert L.hwb_ksk_tc_bytes(ctypes.byref(cp)) == n_col_tiles * k_blocks * 32768
    assert L.hwb_keyswitch_tc_workspace_bytes(ctypes.byref(cp), 129) == 256 * 1024 * 8
    ext = (4 * 129 * 1025 + 255) // 256 * 256
    assert L.hwb_pbs_tc_workspace_bytes(ctypes.byref(cp), 129) == ext + 256 * 1024 * 8
    null = ctypes.c_void_p(0)
    assert L.hwb_keyswitch_tc(ctypes.byref(cp), null, null, null, 0, null, null) == 0     # B = 0
    assert L.hwb_keyswitch_tc(ctypes.byref(cp), null, null, null, 1, null, null) == _lib.HWB_EINVAL
    assert "workspace" in L.hwb_last_error().decode()
    cp.ks_base_log, cp.ks_l = 10, 2                # digits beyond int8
    assert L.hwb_ksk_tc_bytes(ctypes.byref(cp)) == 0
    assert L.hwb_ksk_to_tc(ctypes.byref(cp), null, null, null) == _lib.HWB_EINVAL
    assert "int8" in L.hwb_last_error().decode()


def test_latency_threshold_roundtrip():
    prev = _lib.set_latency_batch(5)
    try:
        assert _lib.set_latency_batch(-2) == 5          # < -1 only queries
        assert _lib.set_latency_batch(-1) == 5          # -1 = automatic
        assert _lib.set_latency_batch(-2) == -1
    finally:
        _lib.set_latency_batch(prev)


def test_fft_ladder_knobs():
    """FFT ladder settings: validation before any CUDA call, query-only values."""
    L = _lib.load()
    assert L.hwb_set_fft_mode(len(_lib.FFT_MODES)) == _lib.HWB_EINVAL
    assert L.hwb_set_fft_mode(-1) == _lib.HWB_EINVAL
    assert "mode" in L.hwb_last_error().decode()
    assert L.hwb_set_fft_cluster_mode(2) == _lib.HWB_EINVAL
    assert L.hwb_set_fft_group(3) == _lib.HWB_EINVAL
    for setter in (L.hwb_set_fft_cluster_batch, L.hwb_set_fft_latency_batch):
        prev = setter(-2)                               # < -1 only queries
        try:
            assert setter(7) == prev
            assert setter(-2) == 7
        finally:
            setter(prev)
    cp = _lib.c_params(named_params("CFG4"))            # N = 2048: no cluster ladder
    assert L.hwb_fft_cluster_capacity(ctypes.byref(cp)) == 0
    # FFT key sizes: N = 1024 (double2 per folded point) and N = 2048 (two halves)
    for name, n_pts in (("CFG2", 512), ("CFG4", 1024)):
        P = named_params(name)
        cp = _lib.c_params(P)
        assert L.hwb_bsk_fft_bytes(ctypes.byref(cp)) == P.lwe_n * 2 * P.gadget.levels * 2 * 2 * n_pts * 16
    cp = _lib.c_params(named_params("CFG2"))
    cp.base_log, cp.l = 17, 1                           # digits wider than 16 bits
    assert L.hwb_bsk_fft_bytes(ctypes.byref(cp)) == 0
    cp.base_log, cp.l = 9, 3
    assert L.hwb_bsk_fft_bytes(ctypes.byref(cp)) > 0


def test_full_precision_gadget_routes_to_the_fft_ladders():
    """2 x 16 gadgets: rejected by the two-prime NTT, accepted by the FP64 FFT ladders
    (16-bit digit staging)."""
    from paper_2403_20190_b200 import tfhe
    for name in ("INSECURE_1024W", "INSECURE_2048W"):
        P = named_params(name)
        cp = _lib.c_params(P)
        assert not tfhe.ntt_supported(P)
        assert _lib.load().hwb_bsk_fft_bytes(ctypes.byref(cp)) == P.lwe_n * 4 * 2 * 2 * (P.n // 2) * 16
    cp = _lib.c_params(named_params("INSECURE_1024W"))
    cp.l, cp.base_log = 3, 11                      # 3 x 11 = 33 bits: no gadget
    assert _lib.load().hwb_bsk_fft_bytes(ctypes.byref(cp)) == 0
