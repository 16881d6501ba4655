"""Smallest launches of the mbarrier / TMEM / tcgen05 kernels for compute-sanitizer
(racecheck, synccheck): cluster ladder (B = 1), TMEM ladder (B = 8 x SMs + 5,
n = 40), tcgen05 key switch (B = 129), FFT2 ladder (B = 3, n = 8), Philox RGSW
regeneration.  Usage: python tools/sanitize_case.py [case ...]"""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def run(case):
    rng = np.random.default_rng(1)
    if case == "cluster":
        P = dataclasses.replace(named_params("CFG2"), lwe_n=16)
        B = 1
    elif case == "tmem":
        P = dataclasses.replace(named_params("CFG2"), lwe_n=40)
        B = 8 * torch.cuda.get_device_properties(0).multi_processor_count + 5
    elif case == "ks":
        P = dataclasses.replace(named_params("CFG2"), lwe_n=630)
        B = 129
    elif case == "fft2":
        P = dataclasses.replace(named_params("CFG4"), lwe_n=8)
        B = 200
    else:
        raise SystemExit(f"unknown case {case}")
    K = tfhe.pbs_keygen(P, 3)
    bsk, ksk = K.device_keys()
    lwe = rng.integers(0, 1 << 32, (B, P.lwe_n + 1), dtype=np.uint64).astype(np.uint32)
    tv = tfhe.test_polynomial(np.arange(P.p // 2), P)
    if case == "ks":
        ext = rng.integers(0, 1 << 32, (B, P.n + 1), dtype=np.uint64).astype(np.uint32)
        out = tfhe.lwe_keyswitch(P, ext, ksk, engine="tc")
    else:
        out = tfhe.pbs_batch(P, lwe, tv, bsk, ksk, ladder="fft")
    torch.cuda.synchronize()
    print(case, "ok", out.shape, flush=True)


for c in sys.argv[1:] or ["cluster", "tmem", "ks", "fft2"]:
    run(c)
