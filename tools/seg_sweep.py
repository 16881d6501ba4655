import sys, ctypes
sys.path.insert(0, '.')
import torch, numpy as np
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import named_params
L = _lib.load()
P = named_params(sys.argv[2] if len(sys.argv) > 2 else "CFG2"); B = int(sys.argv[3]) if len(sys.argv) > 3 else 4096
K = tfhe.pbs_keygen(P, 1); bsk, ksk = K.device_keys()
rng = tfhe.make_rng(9)
lwe = tfhe.to_device(tfhe.enc_lwe_batch(rng.integers(0, P.p, B) * P.delta, K.lwe_key, rng))
tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
ref = None
for seg in (tuple(int(a) for a in sys.argv[1].split(",")) if len(sys.argv) > 1 else (64, 128, 256, 630)):
    _lib.check(L.hwb_set_fft_segment(seg))
    out = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="fft"); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="fft")
    e.record(); e.synchronize()
    ms = s.elapsed_time(e) / 5
    same = True if ref is None else torch.equal(out, ref)
    ref = out if ref is None else ref
    print(f"segment {seg}: {ms:.3f} ms {B / ms * 1e3:,.0f} PBS/s same={same}", flush=True)
