"""ctypes bindings for the C oracle (`oracle/c/hwb_oracle.c`) -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use this.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "c", "libhwb_oracle.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "c", "hwb_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "c"), "-B" if force else "libhwb_oracle.so"],
                       check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i, i64 = ctypes.c_int, ctypes.c_int64
        L.orc_ext_product.argtypes = [i, i, i, _u32p, i, _u32p, _u32p, i64, i]
        L.orc_blind_rotate.argtypes = [i, i, i, _u32p, _i32p, _u32p, i, i64, i]
        L.orc_keyswitch.argtypes = [i, i, i, i, _u32p, _u32p, _u32p, i64, i]
        L.orc_pbs.argtypes = [i, i, i, i, i, i, _u32p, _u32p, _u32p, i, _u32p, _u32p, i64, i, i]
        L.orc_max_threads.restype = i
        L.orc_pack_ks.argtypes = [i, i, i, _u32p, _u32p, _u32p, _u32p, i64, i, i]
        _lib = L
    return _lib


def _p(a, t=_u32p):
    return a.ctypes.data_as(t)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def max_threads() -> int:
    return lib().orc_max_threads()


def ext_product_batch(rgsw, cts, levels, base_log, nthreads=0):
    rgsw, cts = _u32(rgsw), _u32(cts)
    B, _, N = cts.shape
    bcast = 1 if rgsw.ndim == 3 or rgsw.shape[0] == 1 else 0
    out = np.empty_like(cts)
    lib().orc_ext_product(N, levels, base_log, _p(rgsw), bcast, _p(cts), _p(out), B, nthreads)
    return out


def blind_rotate_batch(acc, bsk, exps, levels, base_log, nthreads=0):
    """acc (B,2,N) in, bsk (L,2l,2,N), exps (B,L) = I_i as in hw/tfhe.py:340."""
    acc = _u32(acc).copy()
    bsk = _u32(bsk)
    exps = np.ascontiguousarray(exps, dtype=np.int32)
    B, _, N = acc.shape
    lib().orc_blind_rotate(N, levels, base_log, _p(bsk), _p(exps, _i32p), _p(acc),
                           exps.shape[1], B, nthreads)
    return acc


def keyswitch(lwe, ksk, levels, base_log, nthreads=0):
    lwe, ksk = _u32(lwe), _u32(ksk)
    B = lwe.shape[0]
    N = lwe.shape[1] - 1
    n = ksk.shape[-1] - 1
    out = np.empty((B, n + 1), dtype=np.uint32)
    lib().orc_keyswitch(N, n, levels, base_log, _p(ksk), _p(lwe), _p(out), B, nthreads)
    return out


def pack_batch(a_stacks, b_polys, ksk, levels, base_log, nthreads=0):
    """hw/tfhe.py:390-420 exact: a_stacks (B, k, N), b_polys (B, N), ksk (N, l, 2, N)."""
    a_stacks, b_polys, ksk = _u32(a_stacks), _u32(b_polys), _u32(ksk)
    B, k, N = a_stacks.shape
    out = np.empty((B, 2, N), dtype=np.uint32)
    lib().orc_pack_ks(N, levels, base_log, _p(ksk), _p(a_stacks), _p(b_polys), _p(out), B, k, nthreads)
    return out


def pbs(lwe, tv, bsk, ksk, params, keyswitch=True, nthreads=0):
    lwe, tv, bsk = _u32(lwe), _u32(tv), _u32(bsk)
    ksk = _u32(ksk) if ksk is not None else np.zeros(1, dtype=np.uint32)
    B = lwe.shape[0]
    N, n = params.n, lwe.shape[1] - 1
    g, gk = params.gadget, params.gadget_ks
    width = (n + 1) if keyswitch else (N + 1)
    out = np.empty((B, width), dtype=np.uint32)
    lib().orc_pbs(N, n, g.levels, g.base_log, gk.levels, gk.base_log, _p(bsk), _p(ksk),
                  _p(tv), 1 if tv.ndim == 3 else 0, _p(lwe), _p(out), B,
                  1 if keyswitch else 0, nthreads)
    return out
