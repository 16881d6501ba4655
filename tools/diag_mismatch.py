import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import named_params
import dataclasses
L = _lib.load()
for n in (1, 2, 8, 64, 65):
    P = dataclasses.replace(named_params("CFG2"), lwe_n=n)
    keys = tfhe.pbs_keygen(P, 1)
    bsk, _ = keys.device_keys()
    B = 1184
    rng = tfhe.make_rng(9)
    ms = rng.integers(0, P.p, B)
    lwe = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
    tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
    ref = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="ntt").cpu().numpy().view(np.uint32)
    _lib.check(L.hwb_set_fft_mode(5))
    out = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="fft").cpu().numpy().view(np.uint32)
    bad = out != ref
    d = (out.astype(np.int64) - ref.astype(np.int64)) & 0xFFFFFFFF
    print("n", n, "bad items", int(bad.any(axis=1).sum()), "of", B, "bad words", int(bad.sum()), "of", bad.size)
    if bad.any():
        it = np.argwhere(bad.any(axis=1))[0, 0]
        w = np.argwhere(bad[it])[:, 0]
        print(" first bad item", it, "bad word idx (first 12)", w[:12], "count", len(w))
        print(" diffs hex", [hex(int(x)) for x in d[it, w[:8]]])
