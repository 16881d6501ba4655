#!/usr/bin/env python
"""Run one workload in isolation (for ncu launch lists / captures).

    python tools/run_workload.py pbs   [--batch 4096] [--reps 2]
    python tools/run_workload.py train [--cfg 3] [--images 32] [--reps 2]
    python tools/run_workload.py infer [--cfg 3] [--images 8] [--reps 2]

Prints per-rep wall times (CUDA-synchronised); not a benchmark (use bench.py).
"""

import argparse
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2403_20190_b200 import data, hewnn, tfhe, wnn  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["pbs", "train", "infer"])
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--images", type=int, default=32)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--ladder", default="auto", choices=["auto", "fft", "ntt"])
    a = ap.parse_args()
    if a.what == "pbs":
        P = named_params("CFG2")
        K = tfhe.pbs_keygen(P, 1)
        bsk, ksk = K.device_keys()
        rng = tfhe.make_rng(2)
        lwe = tfhe.to_device(tfhe.enc_lwe_batch(rng.integers(0, 8, a.batch) * P.delta, K.lwe_key, rng))
        tv = tfhe.to_device(tfhe.test_polynomial(np.arange(4), P))
        run = lambda: tfhe.pbs_batch(P, lwe, tv, bsk, ksk)  # noqa: E731
    else:
        (s, l, aa, r, p), pname = data.CONFIG_GEOMETRY[a.cfg]
        P = named_params(pname, p)
        geom = wnn.WisardGeometry(s, l, aa, r, p)
        key, pksk = tfhe.keygen(P, 1)
        ds = data.config_dataset(a.cfg, n=a.images)
        rng = tfhe.make_rng(2)
        lab = None if a.what == "infer" else ds.labels
        smp = [hewnn.encrypt_sample(ds.bits[i], None if lab is None else int(lab[i]), key, rng,
                                    label_bits=geom.label_bits) for i in range(a.images)]
        if a.what == "train":
            run = lambda: hewnn.he_train(smp, geom, P, batch=a.images, ladder=a.ladder)  # noqa: E731
        else:
            model = hewnn.HomWisardModel.zeros(geom, P)
            run = lambda: hewnn.he_infer_pd_batch(model, smp, pksk)  # noqa: E731
    for i in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run()
        torch.cuda.synchronize()
        print(f"{a.what} rep {i}: {time.perf_counter() - t0:.4f} s", flush=True)


if __name__ == "__main__":
    main()
