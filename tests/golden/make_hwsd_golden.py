"""Generate HWSD fixtures with the REFERENCE's own writer (`hewisard.fileio`,
hw/fileio.py:66-260), for the q = 2^32 objects of `hwsd_objects()` embedded as
x << 32 -- the arrays the reference computes on.

Run in the build container, where the reference is importable:
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_hwsd_golden.py
The tests (tests/test_fileio.py) rebuild the same objects from the same seeds,
write them with `paper_2403_20190_b200.fileio` (q64=True) and compare bytes, and
read these files back with the build's reader.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "hwsd")

# tiny ring (N = 16) so the fixtures stay a few KB
PARAM_KW = dict(name="HWSD_TOY", degree_log=4, sigma_rel=2.0 ** -20, p=16)
GADGET, GADGET_PKS = (3, 7), (2, 8)
GEOM = dict(s=5, l=3, a=2, r=7, p=16)      # k0 = 3, label bits 2, selector bits 4 -> 1 RLWE per row


def hwsd_objects(seed: int = 11) -> dict:
    """The fixture content as q = 2^32 words (numpy u32), from one Philox stream."""
    rng = np.random.Generator(np.random.Philox(seed))
    N, l, lp = 1 << PARAM_KW["degree_log"], GADGET[0], GADGET_PKS[0]

    def words(*shape):
        return rng.integers(0, 1 << 32, size=shape, dtype=np.uint64).astype(np.uint32)

    k0 = -(-GEOM["s"] // GEOM["a"])
    samples = [(words(GEOM["s"], 2 * l, 2, N), words(2, 2 * l, 2, N)), (words(GEOM["s"], 2 * l, 2, N), None)]
    return {
        "s1": rng.integers(0, 2, N).astype(np.uint32),
        "pksk": words(N, lp, 2, N),
        "samples": samples,
        "rams": words(k0, 1, 2, N),
        "counts_ct": words(2, N),
        "packs": [(words(1, 2, N), words(2, N)) for _ in range(2)],
        "counters": rng.integers(0, GEOM["p"], size=(GEOM["l"], k0, 1 << GEOM["a"])).astype(np.int64),
        "class_counts": rng.integers(0, 9, size=GEOM["l"]).astype(np.int64),
        "q64_lowbits": rng.integers(0, 1 << 64, size=(2, N), dtype=np.uint64),   # genuine q = 2^64 words
    }


def main():
    from hewisard import fileio as F
    from hewisard.hewnn import EncryptedSample, HomWisardModel, ScorePack
    from hewisard.params import GadgetSpec, HeParams
    from hewisard.tfhe import PackingKeySwitchKey, RgswCiphertext, SecretKey
    from hewisard.wnn import ClassCounts, IntegerWisardModel, WisardGeometry

    os.makedirs(OUT, exist_ok=True)
    P = HeParams(gadget=GadgetSpec(*GADGET), gadget_ks=GadgetSpec(*GADGET_PKS), exact_mul=True, **PARAM_KW)
    Pin = HeParams(gadget=GadgetSpec(*GADGET), gadget_ks=GadgetSpec(*GADGET_PKS), exact_mul=True,
                   insecure=True, **{**PARAM_KW, "name": "HWSD_TOY_INSECURE"})
    geom = WisardGeometry(**GEOM)
    o = hwsd_objects()

    def emb(a):
        return a.astype(np.uint64) << np.uint64(32)

    F.save_secret_key(os.path.join(OUT, "secret_key.hwsd"), SecretKey(P, o["s1"].astype(np.uint64)))
    F.save_secret_key(os.path.join(OUT, "secret_key_insecure.hwsd"), SecretKey(Pin, o["s1"].astype(np.uint64)))
    F.save_ksk(os.path.join(OUT, "ksk.hwsd"), PackingKeySwitchKey(P, emb(o["pksk"])))
    smp = [EncryptedSample(P, [RgswCiphertext(P, c) for c in emb(d)],
                           None if lab is None else [RgswCiphertext(P, c) for c in emb(lab)])
           for d, lab in o["samples"]]
    F.write_samples(os.path.join(OUT, "samples.hwsd"), smp, P, {"source": "fixture"})
    F.save_he_model(os.path.join(OUT, "he_model.hwsd"), HomWisardModel(geom, P, emb(o["rams"]), emb(o["counts_ct"])),
                    {"images": 2})
    F.write_scorepacks(os.path.join(OUT, "scorepacks.hwsd"),
                       [ScorePack(geom, P, emb(a), emb(b)) for a, b in o["packs"]], P, geom)
    F.save_plain_model(os.path.join(OUT, "plain_model.hwsd"), IntegerWisardModel(geom, o["counters"]),
                       ClassCounts(o["class_counts"]), {"note": "fixture"})
    # a genuine q = 2^64 model (low bits set): the build's reader must refuse it
    # unless asked to modulus-switch
    F.save_he_model(os.path.join(OUT, "he_model_q64.hwsd"),
                    HomWisardModel(geom, P, np.stack([o["q64_lowbits"][None]] * 3), o["q64_lowbits"]))
    F.write_manifest(os.path.join(OUT, "manifest.txt"), {"kind": "train", "images": 2, "params": P.name})
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    sys.exit(main())
