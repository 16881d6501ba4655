"""IVP deposit bias at q = 2^32: the exact C-oracle restatement of the
reference label IVP (hw/hewnn.py:180-186, 4 rotation CMUXes at cfg4 gadget 2^10 x 2, sigma = 1)
over many images; prints the mean / std of the error at the deposit coefficient."""
import sys; sys.path.insert(0,'.')
import numpy as np
from oracle import tfhe32 as o, coracle
coracle.build()
N=2048; lv, w = 2, 10; p=8; D=(1<<32)//p
rng=o.make_rng(3)
s=rng.integers(0,2,N).astype(np.uint32)
errs=[]
for img in range(300):
    lab = int(rng.integers(0, 10))
    bits=[(lab>>i)&1 for i in range(4)]
    C=o.enc_rgsw_batch(bits, s, 1.0, lv, w, rng)
    acc=np.zeros((2,N),np.uint32); acc[1,0]=D
    for i,wt in enumerate([1,2,4,8]):
        c1=o.monomial_mul(acc, wt)
        acc=coracle.ext_product_batch(C[i][None], ((c1-acc).astype(np.uint32))[None], lv, w)[0]+acc
        acc=acc.astype(np.uint32)
    ph=o.phase_rlwe(acc, s).astype(np.int64)
    err=((ph + D//2) % D) - D//2
    errs.append(err[lab])
    # others
print("deposit-coefficient error per image:", np.mean(errs), np.std(errs), errs[:8])
