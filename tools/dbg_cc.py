import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2403_20190_b200 import data, hewnn, tfhe, wnn
from paper_2403_20190_b200.params import named_params
(s, l, a, r, _), _ = data.CONFIG_GEOMETRY[4]
P = named_params("CFG4V"); geom = wnn.WisardGeometry(s, l, a, r, P.p)
M = 256
ds = data.config_dataset(4, n=M, seed=0)
key = tfhe.SecretKey(P, tfhe.make_rng(1).integers(0, 2, P.n).astype(np.uint32))
for dn in (True, False):
    rng = tfhe.make_rng(2)
    smp = [hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, rng, label_bits=geom.label_bits, device_noise=dn) for i in range(M)]
    # RGSW noise of the first sample: rows t (gadget on b at coefficient 0)
    st = tfhe.to_host(smp[0].rgsw)            # (n_rgsw, 4, 2, N)
    ph = (st[:, :, 1].astype(np.int64) - tfhe._key_mul_host(st[:, :, 0], key.s).astype(np.int64))
    ph = ((ph + 2**31) % 2**32) - 2**31
    print("device_noise", dn, "rgsw phase (coeff>0) mean", ph[:, :, 1:].mean(), "std", ph[:, :, 1:].std())
    model = hewnn.he_train(smp, geom, P, batch=32)
    cc = tfhe.to_host(model.counts_ct)
    phc = (cc[1].astype(np.int64) - tfhe._key_mul_host(cc[0], key.s).astype(np.int64)) % 2**32
    err = ((phc + P.delta // 2) % P.delta) - P.delta // 2
    print("  counts err mean (all coeffs)", err.mean(), "at 0..l", err[:l])
    rams = tfhe.to_host(model.rams[:4])
    phr = (rams[:, :, 1].astype(np.int64) - tfhe._key_mul_host(rams[:, :, 0], key.s).astype(np.int64)) % 2**32
    er = ((phr + P.delta // 2) % P.delta) - P.delta // 2
    print("  rams err mean", er.mean(), "std", er.std(), "max", np.abs(er).max())
