"""A/B of the FFT PBS ladder modes (hwb_set_fft_mode) on BASELINE parameter sets:
bit-identity of every mode against mode 1 (and the NTT ladder) and blind-rotation
time (CUDA events, no key switch).
Usage: python tools/ab_modes.py [B] [modes, e.g. 1,2] [sets, e.g. CFG2,CFG1] [reps]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    modes = [int(m) for m in (sys.argv[2] if len(sys.argv) > 2 else "1,2").split(",")]
    sets = (sys.argv[3] if len(sys.argv) > 3 else "CFG2").split(",")
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
    L = _lib.load()
    for name in sets:
        P = named_params(name)
        keys = tfhe.pbs_keygen(P, 1)
        bsk, _ = keys.device_keys()
        cp = _lib.c_params(P)
        nb = L.hwb_bsk_fft_bytes(ctypes.byref(cp))
        fk = torch.empty(nb, dtype=torch.uint8, device="cuda")
        _lib.check(L.hwb_bsk_to_fft(ctypes.byref(cp), tfhe._ptr(tfhe.to_device(keys.bsk)), tfhe._ptr(fk),
                                    tfhe._stream()))
        rng = tfhe.make_rng(9)
        ms = rng.integers(0, P.p, B)
        lwe = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
        tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
        ref = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="ntt") if B <= 8192 else None
        ws = torch.empty(L.hwb_pbs_fft_workspace_bytes(ctypes.byref(cp), B, 0), dtype=torch.uint8, device="cuda")
        outs = {}
        for mode in modes:
            _lib.check(L.hwb_set_fft_mode(mode))
            out = torch.zeros((B, P.n + 1), dtype=torch.int32, device="cuda")

            def fft():
                _lib.check(L.hwb_pbs_fft(ctypes.byref(cp), tfhe._ptr(fk), None, tfhe._ptr(tv), 0, tfhe._ptr(lwe),
                                         tfhe._ptr(out), B, tfhe._ptr(ws), tfhe._stream()))
            fft()
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(reps):
                fft()
            e.record()
            e.synchronize()
            ms_ = s.elapsed_time(e) / reps
            outs[mode] = out
            same_ref = None if ref is None else torch.equal(out.view(torch.int32), ref.view(torch.int32))
            same_m = torch.equal(out, outs[modes[0]])
            print(f"{name} B={B} mode {mode}: {ms_:.3f} ms  {B / ms_ * 1e3:,.0f} PBS/s  "
                  f"== mode {modes[0]}: {same_m}  == ntt: {same_ref}", flush=True)
        _lib.check(L.hwb_set_fft_mode(1))


if __name__ == "__main__":
    main()
