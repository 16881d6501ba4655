"""ctypes binding of libhwb200.so (the C ABI declared in include/hwb.h).

There is no CPU fallback: if the library or a GPU is missing, every
homomorphic entry point raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
# HWB_LIB_PATH: load another build of the library (A/B measurement of kernel
# variants, tools/ab_variants.sh); the default is the in-tree build.
LIB_PATH = os.environ.get("HWB_LIB_PATH") or os.path.join(HERE, "libhwb200.so")

HWB_OK, HWB_EINVAL, HWB_ECUDA = 0, 1, 2
FFT_MODE_DEFAULT = 5   # hwb_set_fft_mode's default (libhwb200: g_fft_mode), FFT_MODES = 0..8
FFT_MODES = tuple(range(9))

# every symbol include/hwb.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "hwb_version", "hwb_last_error", "hwb_set_variant", "hwb_probe_modmul", "hwb_ggsw_ntt_words",
    "hwb_ggsw_to_ntt", "hwb_ext_product", "hwb_cmux", "hwb_cdemux", "hwb_blind_rotate",
    "hwb_sample_extract", "hwb_keyswitch", "hwb_pbs_workspace_bytes", "hwb_pbs",
    "hwb_ivp_level", "hwb_vp_level", "hwb_monomial_gather", "hwb_accumulate",
    "hwb_poly_to_ntt", "hwb_key_mul", "hwb_rgsw_add_gadget", "hwb_pack_ks_workspace_bytes", "hwb_pack_ks",
    "hwb_accumulate_rows", "hwb_ksk_tc_bytes", "hwb_ksk_to_tc", "hwb_keyswitch_tc_workspace_bytes",
    "hwb_keyswitch_tc", "hwb_pbs_tc_workspace_bytes", "hwb_pbs_tc", "hwb_probe_i8mma",
    "hwb_set_latency_batch", "hwb_bsk_fft_bytes", "hwb_bsk_to_fft", "hwb_pbs_fft",
    "hwb_pbs_fft_workspace_bytes", "hwb_set_fft_segment", "hwb_probe_fp64",
    "hwb_ggsw_fft_bytes", "hwb_ggsw_to_fft", "hwb_blind_rotate_fft", "hwb_ivp_level_fft", "hwb_vp_level_fft",
    "hwb_set_fft_group", "hwb_set_fft_latency_batch", "hwb_set_fft_mode", "hwb_set_fft_cluster_batch",
    "hwb_fft_cluster_capacity", "hwb_set_fft_cluster_mode", "hwb_fft_margin", "hwb_lwe_lincomb",
    "hwb_gather_rows", "hwb_philox_rgsw",
)


class TfheError(ValueError):
    """Parameter, arity, range and geometry errors (reference hw/tfhe.py:25-26)."""


class EncodingError(TfheError):
    """Message coefficient outside Z_p (reference hw/tfhe.py:29-30)."""


class HwbPhilox(ctypes.Structure):
    _fields_ = [("key", ctypes.c_uint64 * 2), ("ctr", ctypes.c_uint64 * 4), ("prefix", ctypes.c_uint32 * 9),
                ("nprefix", ctypes.c_int32)]


class HwbParams(ctypes.Structure):
    _fields_ = [(name, ctypes.c_uint32) for name in
                ("q_bits", "n", "N", "k", "l", "base_log", "ks_l", "ks_base_log")]


_lib = None
_lock = threading.Lock()
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_pp = ctypes.POINTER(HwbParams)


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        _lib = _configure(ctypes.CDLL(LIB_PATH))
    return _lib


MARGIN_LIB_PATH = os.path.join(HERE, "libhwb200_margin.so")


@contextlib.contextmanager
def using_library(path: str):
    """Route every call of this module through another build of the library (the
    rounding-margin instrumented build in tests and bench; not thread-safe)."""
    global _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing (build it with paper_2403_20190_b200.build)")
    other = _configure(ctypes.CDLL(path))
    prev = load()
    _lib = other
    try:
        yield other
    finally:
        _lib = prev


def _configure(L: ctypes.CDLL) -> ctypes.CDLL:
    L.hwb_version.restype = ctypes.c_int
    L.hwb_last_error.restype = ctypes.c_char_p
    L.hwb_set_variant.argtypes = [ctypes.c_int]
    L.hwb_probe_modmul.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, _vp]
    L.hwb_probe_modmul.restype = ctypes.c_int64
    L.hwb_probe_i8mma.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, _vp]
    L.hwb_probe_fp64.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, _vp]
    L.hwb_probe_fp64.restype = ctypes.c_int64
    L.hwb_probe_i8mma.restype = ctypes.c_int64
    L.hwb_bsk_fft_bytes.argtypes = [_pp]
    L.hwb_bsk_to_fft.argtypes = [_pp, _vp, _vp, _vp]
    L.hwb_pbs_fft.argtypes = [_pp, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _i64, _vp, _vp]
    L.hwb_pbs_fft_workspace_bytes.argtypes = [_pp, _i64, ctypes.c_int]
    L.hwb_set_fft_segment.argtypes = [ctypes.c_int]
    L.hwb_set_fft_group.argtypes = [ctypes.c_int]
    L.hwb_set_fft_latency_batch.argtypes = [_i64]
    L.hwb_set_fft_mode.argtypes = [ctypes.c_int]
    L.hwb_set_fft_cluster_batch.argtypes = [_i64]
    L.hwb_set_fft_cluster_batch.restype = ctypes.c_int64
    L.hwb_fft_cluster_capacity.argtypes = [ctypes.POINTER(HwbParams)]
    L.hwb_fft_cluster_capacity.restype = ctypes.c_int64
    L.hwb_set_fft_cluster_mode.argtypes = [ctypes.c_int]
    L.hwb_set_fft_latency_batch.restype = ctypes.c_int64
    L.hwb_ggsw_fft_bytes.argtypes = [_pp]
    L.hwb_ggsw_to_fft.argtypes = [_pp, _vp, _vp, _i64, _vp]
    L.hwb_blind_rotate_fft.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_ivp_level_fft.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_vp_level_fft.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_set_latency_batch.argtypes = [_i64]
    L.hwb_set_latency_batch.restype = ctypes.c_int64
    L.hwb_ggsw_ntt_words.argtypes = [_pp]
    L.hwb_ggsw_ntt_words.restype = ctypes.c_size_t
    L.hwb_ggsw_to_ntt.argtypes = [_pp, _vp, _vp, _i64, _vp]
    L.hwb_ext_product.argtypes = [_pp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_cmux.argtypes = [_pp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_cdemux.argtypes = [_pp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_blind_rotate.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_sample_extract.argtypes = [_pp, _vp, _vp, _i64, ctypes.c_int32, _vp]
    L.hwb_keyswitch.argtypes = [_pp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_pbs_workspace_bytes.argtypes = [_pp, _i64]
    L.hwb_pbs_workspace_bytes.restype = ctypes.c_size_t
    L.hwb_pbs.argtypes = [_pp, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _i64, _vp, _vp]
    L.hwb_ivp_level.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_vp_level.argtypes = [_pp, _vp, _vp, _vp, _vp, ctypes.c_int32, _i64, _vp]
    L.hwb_monomial_gather.argtypes = [_pp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_accumulate.argtypes = [_vp, _vp, _i64, _i64, ctypes.c_int, _vp]
    L.hwb_accumulate_rows.argtypes = [_vp, _vp, _i64, ctypes.c_int32, _vp]
    L.hwb_poly_to_ntt.argtypes = [_pp, _vp, _vp, _i64, _vp]
    L.hwb_key_mul.argtypes = [_pp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.hwb_rgsw_add_gadget.argtypes = [_pp, _vp, _vp, _i64, _vp]
    L.hwb_pack_ks_workspace_bytes.argtypes = [_pp, _i64]
    L.hwb_pack_ks_workspace_bytes.restype = ctypes.c_size_t
    L.hwb_pack_ks.argtypes = [_pp, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, _vp, _i64, _vp, _vp]
    L.hwb_ksk_tc_bytes.argtypes = [_pp]
    L.hwb_ksk_to_tc.argtypes = [_pp, _vp, _vp, _vp]
    L.hwb_keyswitch_tc_workspace_bytes.argtypes = [_pp, _i64]
    L.hwb_keyswitch_tc.argtypes = [_pp, _vp, _vp, _vp, _i64, _vp, _vp]
    L.hwb_pbs_tc_workspace_bytes.argtypes = [_pp, _i64]
    L.hwb_pbs_tc.argtypes = [_pp, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _i64, _vp, _vp]
    sizes = ("hwb_ggsw_ntt_words", "hwb_pbs_workspace_bytes", "hwb_pack_ks_workspace_bytes",
             "hwb_ksk_tc_bytes", "hwb_keyswitch_tc_workspace_bytes", "hwb_pbs_tc_workspace_bytes",
             "hwb_bsk_fft_bytes", "hwb_pbs_fft_workspace_bytes", "hwb_ggsw_fft_bytes")
    for name in sizes:
        getattr(L, name).restype = ctypes.c_size_t
    for name in EXPORTS:
        if name not in ("hwb_version", "hwb_last_error", "hwb_probe_modmul", "hwb_probe_i8mma", "hwb_probe_fp64",
                        "hwb_set_latency_batch", "hwb_set_fft_latency_batch", "hwb_set_fft_cluster_batch",
                        "hwb_fft_cluster_capacity", *sizes):
            getattr(L, name).restype = ctypes.c_int
    L.hwb_fft_margin.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    L.hwb_lwe_lincomb.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, ctypes.c_int32, ctypes.c_int32, _vp]
    L.hwb_gather_rows.argtypes = [_vp, _vp, _vp, _i64, ctypes.c_int32, _vp]
    L.hwb_philox_rgsw.argtypes = [ctypes.POINTER(HwbPhilox), _vp, _vp, ctypes.c_int32, _vp, _i64, ctypes.c_int32,
                                  ctypes.c_int32, _vp]
    return L


def check(rc: int) -> None:
    if rc == HWB_OK:
        return
    msg = load().hwb_last_error().decode(errors="replace")
    if rc == HWB_EINVAL:
        raise TfheError(msg)
    raise RuntimeError(f"libhwb200: {msg}")


def c_params(params) -> HwbParams:
    """hwb_params from a paper_2403_20190_b200.params.HeParams."""
    return HwbParams(32, int(params.lwe_n), int(params.n), 1, int(params.gadget.levels),
                     int(params.gadget.base_log), int(params.gadget_ks.levels),
                     int(params.gadget_ks.base_log))


def set_variant(v: int) -> None:
    check(load().hwb_set_variant(int(v)))


def set_latency_batch(max_batch: int) -> int:
    """Batches of at most max_batch ciphertexts use the latency-mode ladder
    (N = 1024); returns the previous threshold."""
    return int(load().hwb_set_latency_batch(int(max_batch)))


def fft_margin(reset: bool = False) -> float:
    """Largest FFT rounding residual |y - rint(y)| recorded by the instrumented build
    (inside `using_library(MARGIN_LIB_PATH)`); TfheError on the production build."""
    v = ctypes.c_double(0.0)
    check(load().hwb_fft_margin(ctypes.byref(v), int(reset)))
    return float(v.value)
