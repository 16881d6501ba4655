"""FFT latency ladder vs FFT throughput ladder vs NTT latency ladder on cfg2 PBS
batches (blind rotation + extraction + tensor-core key switch, device-resident):
latency per batch and bit-identity.  Usage: python tools/fft_lat_sweep.py [B ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        out = fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / reps, out


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [1, 16, 74, 148, 296, 444]
    L = _lib.load()
    for name in ("CFG2", "CFG1"):
        P = named_params(name)
        keys = tfhe.pbs_keygen(P, 1)
        bsk, ksk = keys.device_keys()
        tv = tfhe.to_device(tfhe.test_polynomial(np.arange(P.p // 2), P))
        rng = tfhe.make_rng(5)
        for B in sizes:
            ms = rng.integers(0, P.p, B)
            lw = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
            row = {}
            outs = {}
            for mode, thr, cl, cm in (("fft_cluster", 0, 1 << 40, 0), ("fft_cluster4", 0, 1 << 40, 1),
                                      ("fft_lat", 1 << 40, 0, 0), ("fft_thr", 0, 0, 0)):
                L.hwb_set_fft_latency_batch(thr)
                L.hwb_set_fft_cluster_batch(cl)
                _lib.check(L.hwb_set_fft_cluster_mode(cm))
                t, o = timed(lambda: tfhe.pbs_batch(P, lw, tv, bsk, ksk, ladder="fft"))
                row[mode] = round(t, 3)
                outs[mode] = o.clone()
            L.hwb_set_fft_latency_batch(-1)
            L.hwb_set_fft_cluster_batch(0)
            _lib.check(L.hwb_set_fft_cluster_mode(0))
            t, o = timed(lambda: tfhe.pbs_batch(P, lw, tv, bsk, ksk, ladder="ntt"))
            row["ntt_auto"] = round(t, 3)
            row["bit_identical"] = all(bool(torch.equal(v, o)) for v in outs.values())
            print(name, B, json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
