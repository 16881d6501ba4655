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
