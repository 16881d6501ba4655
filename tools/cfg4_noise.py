"""cfg4 feasibility at q = 2^32: train the cfg4 geometry (a = 16, 147 RAMs, N = 2048)
on M images and measure the decrypted model's noise and counter correctness, for the
BASELINE parameter set and for variants (sigma of the client RGSWs, p).
Usage: python tools/cfg4_noise.py"""
import dataclasses
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2403_20190_b200 import data, hewnn, tfhe, wnn  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402

(s, l, a, r, _), _ = data.CONFIG_GEOMETRY[4]
for name, sigma_rel, p, M in (("CFG4 (BASELINE)", None, 4096, 4), ("CFG4 sigma 2^-32", 2.0 ** -32, 4096, 4),
                              ("CFG4 sigma 2^-32 p=256", 2.0 ** -32, 256, 16),
                              ("CFG4 sigma 2^-32 p=256", 2.0 ** -32, 256, 64),
                              ("CFG4 sigma 2^-32 p=256", 2.0 ** -32, 256, 128)):
    P = named_params("CFG4", p)
    if sigma_rel is not None:
        P = dataclasses.replace(P, sigma_rel=sigma_rel)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    key = tfhe.SecretKey(P, tfhe.make_rng(1).integers(0, 2, P.n).astype(np.uint32))
    ds = data.config_dataset(4, n=M, seed=0)
    rng = tfhe.make_rng(2)
    smp = [hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits)
           for i in range(M)]
    t0 = time.perf_counter()
    model = hewnn.he_train(smp, geom, P, batch=8)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    noise, margin = hewnn.model_noise(model, key)
    dm, _ = hewnn.decrypt_model(model, key)
    ref, _ = wnn.train_integer(ds.bits, ds.labels, geom)
    print(f"{name:28s} M={M:4d}: noise 2^{np.log2(max(noise, 1)):.2f} margin 2^{np.log2(margin):.2f} "
          f"correct {np.mean(dm.counters == ref.counters):.6f}  ({M / dt:.1f} img/s)", flush=True)
    del smp, model
