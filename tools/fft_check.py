"""FP64 FFT ladder vs NTT ladder: bit-exactness and speed on cfg2/cfg1 PBS batches
(blind rotation + extraction, no key switch).  Usage: python tools/fft_check.py [B] [segment] [ciphertexts/CTA] [mode: 0 registers, 1 TMEM]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def main(B=4096):
    L = _lib.load()
    for name in ("CFG2", "CFG1", "CFG4"):
        P = named_params(name)
        keys = tfhe.pbs_keygen(P, 1)
        bsk, _ = keys.device_keys()
        cp = _lib.c_params(P)
        nb = L.hwb_bsk_fft_bytes(ctypes.byref(cp))
        fk = torch.empty(nb, dtype=torch.uint8, device="cuda")
        coeff = tfhe.to_device(keys.bsk)
        _lib.check(L.hwb_bsk_to_fft(ctypes.byref(cp), tfhe._ptr(coeff), tfhe._ptr(fk), tfhe._stream()))
        rng = tfhe.make_rng(9)
        ms = rng.integers(0, P.p, B)
        lwe = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
        tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
        ref = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="ntt")
        out = torch.empty_like(ref)
        ws = torch.empty(L.hwb_pbs_fft_workspace_bytes(ctypes.byref(cp), B, 0), dtype=torch.uint8, device="cuda")
        seg = int(sys.argv[2]) if len(sys.argv) > 2 else 64
        _lib.check(L.hwb_set_fft_segment(seg))
        _lib.check(L.hwb_set_fft_group(int(sys.argv[3]) if len(sys.argv) > 3 else 1))
        _lib.check(L.hwb_set_fft_mode(int(sys.argv[4]) if len(sys.argv) > 4 else 1))

        def fft():
            _lib.check(L.hwb_pbs_fft(ctypes.byref(cp), tfhe._ptr(fk), None, tfhe._ptr(tv), 0, tfhe._ptr(lwe),
                                     tfhe._ptr(out), B, tfhe._ptr(ws), tfhe._stream()))
        fft()
        torch.cuda.synchronize()
        same = torch.equal(out, ref)
        nd = int((out != ref).sum())
        times = {}
        for label, fn in (("ntt", lambda: tfhe.pbs_batch(P, lwe, tv, bsk, None, out=ref, ladder="ntt")), ("fft", fft)):
            fn()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(3):
                fn()
            e.record()
            e.synchronize()
            times[label] = s.elapsed_time(e) / 3
        print(f"{name} B={B}: bit-identical {same} (differing words {nd}); ntt {times['ntt']:.2f} ms "
              f"({B / times['ntt'] * 1e3:.0f}/s), fft {times['fft']:.2f} ms ({B / times['fft'] * 1e3:.0f}/s)")


if __name__ == "__main__":
    main(*[int(x) for x in sys.argv[1:2]])
