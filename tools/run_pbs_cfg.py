"""One PBS batch of a named parameter set through tfhe.pbs_batch (ncu captures).
Usage: python tools/run_pbs_cfg.py NAME B [ladder] [reps]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402

name = sys.argv[1]
B = int(sys.argv[2])
ladder = sys.argv[3] if len(sys.argv) > 3 else "fft"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
P = named_params(name)
keys = tfhe.pbs_keygen(P, 1)
bsk, ksk = keys.device_keys()
rng = tfhe.make_rng(5)
lw = tfhe.to_device(tfhe.enc_lwe_batch(rng.integers(0, P.p, B) * P.delta, keys.lwe_key, rng))
tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
for _ in range(reps):
    out = tfhe.pbs_batch(P, lw, tv, bsk, ksk, ladder=ladder)
torch.cuda.synchronize()
print("ok", name, B, ladder)
