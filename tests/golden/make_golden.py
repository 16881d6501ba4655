"""Generate golden fixtures by running the REFERENCE on q=2^32 operands.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The reference (`hewisard`, q = 2^64) computes the q = 2^32 results bit for bit
when every operand is embedded as x << 32 and the parameter set uses the
exact (schoolbook) path: gadget digits of x << 32 with levels*base_log <= 32
are the q = 2^32 digits (hw/ring.py:136-150) and products of multiples of 2^32
stay multiples of 2^32 (SURVEY.md §0 finding 4).  Every result is checked to
have all-zero low 32 bits before being shifted back.

Functions the reference lacks (mod switch, LWE key switch, q = 2^32 key
generation) come from the oracle restatement; the fixture records which.
The fixtures are small .npz files; large keys are regenerated from their seed
in the tests and pinned here by SHA-256.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from hewisard import lut as rl  # noqa: E402
from hewisard import ring as rr  # noqa: E402
from hewisard import tfhe as rt  # noqa: E402
from hewisard.params import GadgetSpec as RGadget  # noqa: E402
from hewisard.params import HeParams as RParams  # noqa: E402

from oracle import tfhe32 as o  # noqa: E402
from paper_2403_20190_b200.params import named_params  # noqa: E402

U64 = np.uint64


def emb(x):
    return np.asarray(x, dtype=np.uint32).astype(U64) << U64(32)


def unemb(y):
    y = np.asarray(y, dtype=U64)
    assert not np.any(y & U64(0xFFFFFFFF)), "embedding broke: low 32 bits non-zero"
    return (y >> U64(32)).astype(np.uint32)


def ref_params(N_log, levels, base_log, p=8):
    return RParams(name="emb", degree_log=N_log, sigma_rel=0.0,
                   gadget=RGadget(levels, base_log), gadget_ks=RGadget(2, 32),
                   p=p, insecure=True, exact_mul=True)


def rand_u32(rng, shape):
    return rng.integers(0, 1 << 32, shape, dtype=np.uint64).astype(np.uint32)


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def gen_decompose(rng):
    out = {}
    for (lv, w) in [(3, 7), (2, 8), (2, 10), (8, 2), (7, 2), (2, 16), (1, 23), (4, 8)]:
        x = rand_u32(rng, 4096)
        x[:6] = [0, 0xFFFFFFFF, 0x80000000, 0x7FFFFFFF, 1 << (32 - lv * w) if lv * w < 32 else 1, 0x40000000]
        d = rr.gadget_decompose_raw(emb(x), RGadget(lv, w))           # hw/ring.py:126-151
        out[f"x_{lv}_{w}"] = x
        out[f"d_{lv}_{w}"] = d.astype(np.int32)
    np.savez_compressed(os.path.join(HERE, "decompose.npz"), **out)


def gen_negacyclic(rng):
    out = {}
    for N in (8, 1024, 2048):
        a = rand_u32(rng, (2, N))
        b = rand_u32(rng, (2, N))
        c = np.stack([unemb(rr.negacyclic_mul_raw(emb(a[i]), b[i].astype(U64))) for i in range(2)])
        out[f"a_{N}"], out[f"b_{N}"], out[f"c_{N}"] = a, b, c
    np.savez_compressed(os.path.join(HERE, "negacyclic.npz"), **out)


def gen_ext_product(rng):
    out = {}
    for tag, (N_log, lv, w, B) in {"cfg2": (10, 3, 7, 3), "cfg1": (10, 2, 8, 2),
                                    "cfg4": (11, 2, 10, 2), "ins": (10, 2, 16, 2)}.items():
        N = 1 << N_log
        P = ref_params(N_log, lv, w)
        G = rand_u32(rng, (B, 2 * lv, 2, N))
        cts = rand_u32(rng, (B, 2, N))
        res = unemb(rt.ext_product_batch(P, emb(G), emb(cts)))         # hw/tfhe.py:301-315
        resb = unemb(rt.ext_product_batch(P, emb(G[:1]), emb(cts)))    # broadcast GGSW
        out.update({f"{tag}_G": G, f"{tag}_cts": cts, f"{tag}_out": res, f"{tag}_out_bcast": resb})
    np.savez_compressed(os.path.join(HERE, "ext_product.npz"), **out)


def gen_blind_rotate(rng):
    out = {}
    for tag, (N_log, lv, w, L) in {"cfg2": (10, 3, 7, 5), "cfg4": (11, 2, 10, 3)}.items():
        N = 1 << N_log
        P = ref_params(N_log, lv, w)
        c = rand_u32(rng, (2, N))
        C = rand_u32(rng, (L, 2 * lv, 2, N))
        I = [int(v) for v in rng.integers(-3 * N, 3 * N, L)]
        I[0] = 0
        acc = rt.blind_rotate(rt.RlweCiphertext(P, emb(c)),
                              [rt.RgswCiphertext(P, emb(Ci)) for Ci in C], I)   # hw/tfhe.py:340-349
        res = unemb(acc.data)
        ext = rt.extract_lwe(acc, 0)                                            # hw/tfhe.py:352-361
        out.update({f"{tag}_c": c, f"{tag}_C": C, f"{tag}_I": np.array(I, dtype=np.int64),
                    f"{tag}_out": res, f"{tag}_ext_a": unemb(ext.a),
                    f"{tag}_ext_b": unemb(np.array([ext.b], dtype=U64))})
    np.savez_compressed(os.path.join(HERE, "blind_rotate.npz"), **out)


def gen_pbs(name, count, key_seed=1, enc_seed=2):
    """Full PBS: reference blind_rotate/extract on embedded keys + restated
    mod switch and key switch (NEW, oracle)."""
    P = named_params(name)
    keys = o.pbs_keygen(P, key_seed)
    N, n, g = P.n, P.lwe_n, P.gadget
    RP = ref_params(P.degree_log, g.levels, g.base_log, p=P.p)
    rng = o.make_rng(enc_seed)
    ms = rng.integers(0, P.p, count)
    lwe = o.enc_lwe_batch(ms * P.delta, keys["s0"], P.lwe_sigma, rng)
    tv = o.test_polynomial(np.arange(P.p // 2) % P.p, P.p, N)
    bsk_ref = [rt.RgswCiphertext(RP, emb(b)) for b in keys["bsk"]]
    ext_rows = []
    for row in lwe:
        msw = o.mod_switch(row, N)                                              # NEW
        acc0 = rt.RlweCiphertext(RP, rr.monomial_mul_raw(emb(tv), -int(msw[-1])))  # hw/ring.py:106
        acc = rt.blind_rotate(acc0, bsk_ref, [-int(x) for x in msw[:-1]])       # hw/tfhe.py:340
        ext = rt.extract_lwe(acc, 0)                                            # hw/tfhe.py:352
        ext_rows.append(np.concatenate([unemb(ext.a), unemb(np.array([ext.b], dtype=U64))]))
    ext_rows = np.stack(ext_rows)
    gk = P.gadget_ks
    out_rows = o.lwe_keyswitch(ext_rows, keys["ksk"], gk.levels, gk.base_log)   # NEW
    np.savez_compressed(
        os.path.join(HERE, f"pbs_{name.lower()}.npz"),
        key_seed=key_seed, enc_seed=enc_seed, ms=ms, lwe_in=lwe, tv=tv,
        extracted=ext_rows, lwe_out=out_rows,
        sha_s0=sha(keys["s0"]), sha_s1=sha(keys["s1"]), sha_bsk=sha(keys["bsk"]),
        sha_ksk=sha(keys["ksk"]))


sys.path.insert(0, HERE)
from cases import TRAIN_CASES, train_inputs  # noqa: E402


def gen_train(name):
    """Encrypted WiSARD training by the REFERENCE's he_train (hw/hewnn.py:189)
    on embedded q = 2^32 RGSW inputs."""
    from hewisard import hewnn as rh
    from hewisard import wnn as rw
    P, s1, bits, labels, stacks = train_inputs(name)
    (s, l, a, r) = TRAIN_CASES[name][2]
    g = P.gadget
    RP = ref_params(P.degree_log, g.levels, g.base_log, p=P.p)
    geom = rw.WisardGeometry(s=s, l=l, a=a, r=r, p=P.p)
    samples = [rh.EncryptedSample(RP, [rt.RgswCiphertext(RP, emb(x)) for x in st[:s]],
                                  [rt.RgswCiphertext(RP, emb(x)) for x in st[s:]]) for st in stacks]
    model = rh.he_train(samples, geom, RP)
    rams, counts = unemb(model.rams), unemb(model.counts_ct)
    # sanity: the reference's own decryption equals its plaintext trainer
    key = rt.SecretKey(RP, s1.astype(np.uint64))
    plain, cc = rh.decrypt_model(model, key)
    ref_int, ref_counts = rw.train_integer(bits, labels, geom)
    assert np.array_equal(plain.counters, ref_int.counters) and np.array_equal(cc.counts, ref_counts.counts)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), rams_head=rams[:, :2], counts_ct=counts,
                        sha_rams=sha(rams), sha_stacks=sha(*stacks), counters=ref_int.counters,
                        class_counts=ref_counts.counts, bits=bits, labels=labels)


def gen_infer():
    """Reference pack_batch (hw/tfhe.py:390) and he_infer_pd (hw/hewnn.py:278)
    on the train_tree model, embedded at q = 2^32.  The packing key comes from
    the q = 2^32 restatement of keygen (its first draw is the training key s1)."""
    from hewisard import hewnn as rh
    from hewisard import wnn as rw
    from hewisard.params import GadgetSpec as RG
    name = "train_tree"
    P, s1, bits, labels, stacks = train_inputs(name)
    (s, l, a, r) = TRAIN_CASES[name][2]
    kseed = TRAIN_CASES[name][4]
    s_pk, ksk = o.keygen_packing(P, kseed)
    assert np.array_equal(s_pk, s1)
    g, gp = P.gadget, P.gadget_pks
    RP = RParams(name="emb", degree_log=P.degree_log, sigma_rel=0.0, gadget=RG(g.levels, g.base_log),
                 gadget_ks=RG(gp.levels, gp.base_log), p=P.p, insecure=True, exact_mul=True)
    rksk = rt.PackingKeySwitchKey(RP, emb(ksk))
    # pack_batch on random LWEs
    prng = np.random.default_rng(99)
    k = 7
    a_st = rand_u32(prng, (2, k, P.n))
    b_p = np.zeros((2, P.n), dtype=np.uint32)
    b_p[:, :k] = rand_u32(prng, (2, k))
    packed = unemb(rt.pack_batch(emb(a_st), emb(b_p), rksk))
    # he_infer_pd on the trained model and a fresh (unlabelled) test sample
    geom = rw.WisardGeometry(s=s, l=l, a=a, r=r, p=P.p)
    samples = [rh.EncryptedSample(RP, [rt.RgswCiphertext(RP, emb(x)) for x in st[:s]],
                                  [rt.RgswCiphertext(RP, emb(x)) for x in st[s:]]) for st in stacks]
    model = rh.he_train(samples, geom, RP)
    test_bits = prng.integers(0, 2, s)
    test_rgsw = o.enc_rgsw_batch(test_bits, s1, P.sigma, g.levels, g.base_log, o.make_rng(13))
    tsample = rh.EncryptedSample(RP, [rt.RgswCiphertext(RP, emb(x)) for x in test_rgsw], None)
    pack = rh.he_infer_pd(model, tsample, rksk)
    fin = rh.client_finalize(pack, rt.SecretKey(RP, s1.astype(np.uint64)), rw.ActivationSpec("bin", 0))
    np.savez_compressed(os.path.join(HERE, "infer_tree.npz"), sha_ksk=sha(ksk), pack_a=a_st, pack_b=b_p,
                        pack_out=packed, test_bits=test_bits, sha_test_rgsw=sha(test_rgsw),
                        infer_packed=unemb(pack.packed), raw=fin.raw, prediction=fin.prediction)


def main():
    rng = np.random.default_rng(20240329)
    t = time.time()
    gen_decompose(rng)
    gen_negacyclic(rng)
    gen_ext_product(rng)
    gen_blind_rotate(rng)
    print(f"primitives: {time.time() - t:.1f}s", flush=True)
    for name, count in (("CFG2", 2), ("CFG1", 1), ("CFG4", 1)):
        t = time.time()
        gen_pbs(name, count)
        print(f"pbs {name}: {time.time() - t:.1f}s", flush=True)
    for name in TRAIN_CASES:
        t = time.time()
        gen_train(name)
        print(f"{name}: {time.time() - t:.1f}s", flush=True)
    t = time.time()
    gen_infer()
    print(f"infer: {time.time() - t:.1f}s", flush=True)


if __name__ == "__main__":
    main()
