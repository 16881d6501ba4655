"""Full-precision gadgets (2 x 16 = 32 bits), the reference's exact mode at q = 2^32
(hw/params.py:94-101: zero noise and a full-precision gadget make every external
product exact).  Beyond the two-prime NTT's range, these run on the
FP64 FFT ladders with 16-bit digits; every result is compared with the schoolbook C
oracle, and encrypted training decrypts to the plaintext counters with ZERO noise
(the reference's bit-exact test strategy, pkg/tests/test_hewnn.py:85-103)."""

import dataclasses

import numpy as np
import pytest

from conftest import assert_u32_equal
from oracle import tfhe32 as o
from paper_2403_20190_b200 import hewnn, tfhe, wnn
from paper_2403_20190_b200.params import named_params

pytestmark = pytest.mark.gpu


def _rand(rng, shape):
    return rng.integers(0, 1 << 32, shape, dtype=np.uint64).astype(np.uint32)


@pytest.mark.parametrize("name", ["INSECURE_1024W", "INSECURE_2048W"])
def test_wide_gadget_pbs_vs_oracle(coracle, name):
    P = dataclasses.replace(named_params(name), lwe_n=24)
    assert not tfhe.ntt_supported(P)
    K = tfhe.pbs_keygen(P, 3)
    bsk, _ = K.device_keys()
    assert bsk.ntt is None and bsk.fft is not None
    rng = np.random.default_rng(4)
    sms = 148
    for B in (1, 5, 200, 8 * sms + 3):                    # cluster / latency / register / TMEM ladders
        lwe = _rand(rng, (B, P.lwe_n + 1))
        tvs = _rand(rng, (B, 2, P.n))
        out = tfhe.pbs_batch(P, lwe, tvs, bsk, None)
        idx = np.unique(np.linspace(0, B - 1, min(B, 24)).astype(int))
        assert_u32_equal(out[idx], coracle.pbs(lwe[idx], tvs[idx], K.bsk, None, P, keyswitch=False))


@pytest.mark.parametrize("name", ["INSECURE_1024W", "INSECURE_2048W"])
def test_wide_gadget_single_ops_vs_oracle(name):
    P = named_params(name)
    lv, w = P.gadget.levels, P.gadget.base_log
    rng = np.random.default_rng(5)
    G = _rand(rng, (6, 2 * lv, 2, P.n))
    cts = _rand(rng, (6, 2, P.n))
    c1 = _rand(rng, (6, 2, P.n))
    want = o.ext_product_batch(G, cts, lv, w)
    assert_u32_equal(tfhe.ext_product_batch(P, G, cts), want)
    lo, hi = tfhe.cdemux_batch(P, G, cts)
    assert_u32_equal(hi, want)
    assert_u32_equal(lo, (cts - want).astype(np.uint32))
    mux = tfhe.cmux_batch(P, G, c1, cts)
    assert_u32_equal(mux, (cts + o.ext_product_batch(G, (c1 - cts).astype(np.uint32), lv, w)).astype(np.uint32))
    exps = rng.integers(0, 2 * P.n, (6, 6))
    got = tfhe.blind_rotate_batch(P, cts, G, exps)
    ref = cts.copy()
    for b in range(6):
        ref[b] = o.blind_rotate(cts[b], list(G), list(exps[b]), lv, w)
    assert_u32_equal(got, ref)


def test_exact_mode_training_zero_noise():
    """Encrypted training at the zero-noise, full-precision set: decrypted counters equal
    train_integer and the model's noise is exactly zero."""
    P = named_params("INSECURE_1024W", p=256)
    geom = wnn.WisardGeometry(40, 3, 8, 3, 256)
    key, ksk = tfhe.keygen(P, rng_seed=42)
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2, (12, geom.s)).astype(np.uint8)
    labels = rng.integers(0, 3, 12)
    erng = tfhe.make_rng(1)
    samples = [hewnn.encrypt_sample(bits[i], int(labels[i]), key, erng, label_bits=geom.label_bits)
               for i in range(10)]
    model = hewnn.he_train(samples, geom, P)
    plain, counts = wnn.train_integer(bits[:10], labels[:10], geom)
    dec, dcounts = hewnn.decrypt_model(model, key)
    assert np.array_equal(dec.counters, plain.counters)
    assert np.array_equal(dcounts.counts, counts.counts)
    noise, _ = hewnn.model_noise(model, key)
    assert noise == 0
    # PD-act inference on the exact model: predictions equal the plaintext
    test = [hewnn.encrypt_sample(bits[i], None, key, erng) for i in (10, 11)]
    packs = hewnn.he_infer_pd_batch(model, test, ksk)
    act = wnn.ActivationSpec("bin", 0)
    preds = [hewnn.client_finalize(pk, key, act).prediction for pk in packs]
    assert preds == list(wnn.evaluate_dataset(plain, bits[10:], act))
