"""One cfg2 PBS batch through tfhe.pbs_batch (for ncu captures of a single launch
configuration).  Usage: python tools/run_pbs.py B [ladder] [fft_latency_batch] [reps] [fft_mode] [cluster_batch]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ladder = sys.argv[2] if len(sys.argv) > 2 else "fft"
if len(sys.argv) > 3:
    _lib.load().hwb_set_fft_latency_batch(int(sys.argv[3]))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
if len(sys.argv) > 5:
    _lib.check(_lib.load().hwb_set_fft_mode(int(sys.argv[5])))
if len(sys.argv) > 6:
    _lib.load().hwb_set_fft_cluster_batch(int(sys.argv[6]))
P = named_params("CFG2")
keys = tfhe.pbs_keygen(P, 1)
bsk, ksk = keys.device_keys()
rng = tfhe.make_rng(5)
ms = rng.integers(0, P.p, B)
lw = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
tv = tfhe.to_device(tfhe.test_polynomial(np.arange(4), P))
for _ in range(reps):
    out = tfhe.pbs_batch(P, lw, tv, bsk, ksk, ladder=ladder)
torch.cuda.synchronize()
print("ok", B, ladder)
