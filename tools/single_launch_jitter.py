"""Per-call times of the single-launch ladder (FFT mode 5) against per-segment launches (mode 8),
alternating segment lengths: looks for outliers.  Usage: python tools/single_launch_jitter.py [SET] [B] [calls]"""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import named_params
L = _lib.load()
P = named_params(sys.argv[1] if len(sys.argv) > 1 else "CFG2")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 12
K = tfhe.pbs_keygen(P, 1)
bsk, ksk = K.device_keys()
rng = tfhe.make_rng(9)
lwe = tfhe.to_device(tfhe.enc_lwe_batch(rng.integers(0, P.p, B) * P.delta, K.lwe_key, rng))
tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
for mode in (5, 8, 5):
    _lib.check(L.hwb_set_fft_mode(mode))
    for seg in (24, 32, 25, 32, 64, 48, 32):
        _lib.check(L.hwb_set_fft_segment(seg))
        ts = []
        for _ in range(calls):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="fft")
            e.record()
            e.synchronize()
            ts.append(s.elapsed_time(e))
        print(f"mode {mode} segment {seg}: min {min(ts):.2f} median {sorted(ts)[len(ts) // 2]:.2f} max {max(ts):.2f} ms",
              flush=True)
