"""Compare the throughput and latency-mode ladders on cfg2 PBS batches (device-
resident, CUDA events): PBS/s and latency per batch size, outputs compared
bit for bit between the two modes.  Usage: python tools/lat_sweep.py [B ...]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import _lib, tfhe  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def main():
    sizes = [int(x) for x in sys.argv[1:]] or [1, 2, 16, 74, 148, 296, 444, 592]
    P = named_params("CFG2")
    keys = tfhe.pbs_keygen(P, 1)
    bsk, ksk = keys.device_keys()
    tv = tfhe.to_device(tfhe.test_polynomial(np.arange(4), P))
    rng = tfhe.make_rng(5)
    res = {}
    for B in sizes:
        ms = rng.integers(0, P.p, B)
        lw = tfhe.to_device(tfhe.enc_lwe_batch(ms * P.delta, keys.lwe_key, rng))
        row, outs = {}, {}
        for mode, thr in (("throughput", 0), ("latency", 1 << 40)):
            _lib.set_latency_batch(thr)
            out = tfhe.pbs_batch(P, lw, tv, bsk, ksk)          # warm-up
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 3
            s0.record()
            for _ in range(reps):
                out = tfhe.pbs_batch(P, lw, tv, bsk, ksk)
            s1.record()
            s1.synchronize()
            t = s0.elapsed_time(s1) / reps
            row[mode] = {"latency_ms": round(t, 3), "pbs_per_s": round(B / t * 1e3, 1)}
            outs[mode] = out.clone()
        row["bit_identical"] = bool(torch.equal(outs["throughput"], outs["latency"]))
        res[B] = row
        print(B, json.dumps(row), flush=True)
    _lib.set_latency_batch(-1)


if __name__ == "__main__":
    main()
