"""Debug: PBS with n = N (self-bootstrapping shape) on every ladder vs the NTT ladder."""
import dataclasses
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402

for n in (630, 1024):
    P = dataclasses.replace(named_params("CFG3", 256), lwe_n=n)
    K = tfhe.pbs_keygen(P, 3)
    bsk, _ = K.device_keys()
    rng = np.random.default_rng(4)
    for B in (5, 60, 140, 300, 1200):
        lwe = rng.integers(0, 1 << 32, (B, n + 1), dtype=np.uint64).astype(np.uint32)
        tv = rng.integers(0, 1 << 32, (B, 2, P.n), dtype=np.uint64).astype(np.uint32)
        a = tfhe.pbs_batch(P, lwe, tv, bsk, None)
        b = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="ntt")
        print(n, B, "equal" if np.array_equal(a, b) else f"DIFF {np.mean(a != b):.3f}", flush=True)
