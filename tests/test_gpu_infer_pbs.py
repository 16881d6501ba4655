"""OTF-act inference on the PBS engine (paper_2403_20190_b200.infer_pbs): bleaching
threshold, popcount and argmax on ciphertexts.

* bit-exact with the CPU restatement (oracle/infer32.py on the C oracle's PBS),
* decrypted results equal the plaintext semantics: [m > thr] for every counter
  value, the popcount of the activated RAMs, and the prediction of
  wnn.evaluate_dataset(model, bits, ActivationSpec("bin", thr)) (hw/wnn.py:86-109,
  296-309), on the BASELINE cfg3 geometry.
"""

import dataclasses

import numpy as np
import pytest
import torch

from conftest import assert_u32_equal
from oracle import infer32
from paper_2403_20190_b200 import data, hewnn, infer_pbs, tfhe, wnn
from paper_2403_20190_b200.params import named_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    P = named_params("CFG3", 256)
    key = tfhe.SecretKey(P, tfhe.make_rng(21).integers(0, 2, P.n).astype(np.uint32))
    sbk = infer_pbs.self_bootstrap_keygen(key, 22)
    return P, key, sbk


def _enc_lwe_s1(ms, P, key, rng, scale):
    """LWEs of m * scale under S1 (sample extraction of RLWE encryptions)."""
    rows = []
    for m in ms:
        mu = np.zeros(P.n, dtype=np.uint32)
        mu[0] = np.uint32((int(m) * scale) & 0xFFFFFFFF)
        ct = tfhe.enc_rlwe_raw(mu, key, rng)
        rows.append(ct.data)
    return tfhe.sample_extract_batch(P, np.stack(rows))


def test_bleach_every_counter_value(ctx, coracle):
    """Every m in Z_256 and several thresholds: decrypts to [m > thr]; a sample of the
    ciphertexts equals the oracle restatement bit for bit."""
    P, key, sbk = ctx
    rng = tfhe.make_rng(23)
    ms = np.arange(256)
    lwe = _enc_lwe_s1(ms, P, key, rng, P.delta)
    P16 = dataclasses.replace(P, p=16)
    luts = infer_pbs.Luts(P)
    for thr in (0, 1, 3, 127, 200, 254, 255, 300, -1):
        out = tfhe.to_host(infer_pbs.bleach(sbk, luts, tfhe.to_device(lwe), 256, thr))
        dec = tfhe.dec_lwe_batch(out, key, P16)
        assert np.array_equal(dec, (ms > thr).astype(np.int64)), thr
    sub = lwe[[0, 1, 77, 128, 255]]
    boot = infer32.Boot(sbk.params, sbk.bsk)
    want = infer32.bleach(boot, sub, 256, 77)
    got = tfhe.to_host(infer_pbs.bleach(sbk, luts, tfhe.to_device(sub), 256, 77))
    assert_u32_equal(got, want)


@pytest.mark.parametrize("p", [2, 8, 32])
def test_bleach_odd_counter_widths(ctx, p):
    """p = 2^K with K odd (cfg4's stated variant uses p = 8): the top digit is a single
    bit; every value and every threshold decrypts to [m > thr]."""
    P, key, sbk = ctx
    ms = np.arange(p)
    lwe = tfhe.to_device(_enc_lwe_s1(ms, P, key, tfhe.make_rng(26), (1 << 32) // p))
    P16 = dataclasses.replace(P, p=16)
    luts = infer_pbs.Luts(P)
    for thr in range(-1, p + 1):
        out = tfhe.to_host(infer_pbs.bleach(sbk, luts, lwe, p, thr))
        assert np.array_equal(tfhe.dec_lwe_batch(out, key, P16), (ms > thr).astype(np.int64)), (p, thr)


def test_popcount_and_argmax(ctx):
    """Activated-bit sums up to 196 (cfg3's k0) and first-max argmax with ties."""
    P, key, sbk = ctx
    rng = np.random.default_rng(24)
    l, k0 = 5, 196
    prob = np.array([0.1, 0.5, 0.5, 0.9, 0.3])
    bits = (rng.random((2, l, k0)) < prob[None, :, None]).astype(np.int64)
    bits[1, 2] = bits[1, 3]                                  # tie between classes 2 and 3 in sample 1
    bits[1, 3, :] = 1
    bits[1, 2, :] = 1                                        # both 196: first max (2) wins
    enc = _enc_lwe_s1(bits.reshape(-1), P, key, tfhe.make_rng(25), infer_pbs.OUT)
    luts = infer_pbs.Luts(P)
    d = tfhe.to_device(enc).reshape(2 * l, k0, -1)
    scores = infer_pbs.popcount(sbk, luts, d, k0)
    P16 = dataclasses.replace(P, p=16)
    dig = np.stack([tfhe.dec_lwe_batch(tfhe.to_host(s), key, P16) for s in scores])
    got = (dig * (4 ** np.arange(len(scores)))[:, None]).sum(axis=0).reshape(2, l)
    assert np.array_equal(got, bits.sum(axis=2))
    idx = infer_pbs.argmax(sbk, luts, scores, l)
    pred = sum(tfhe.dec_lwe_batch(tfhe.to_host(x), key, P16) << (2 * k) for k, x in enumerate(idx))
    assert np.array_equal(pred, np.argmax(bits.sum(axis=2), axis=1))


def test_infer_bin_small_geometry_vs_oracle(coracle):
    """End to end on a small geometry (3 classes, 2 RAMs, 4-bit counters): the
    encrypted class indices equal the oracle restatement bit for bit and decrypt to
    the plaintext prediction."""
    P = named_params("CFG3", 16)
    geom = wnn.WisardGeometry(8, 3, 4, 7, 16)
    key = tfhe.SecretKey(P, tfhe.make_rng(31).integers(0, 2, P.n).astype(np.uint32))
    sbk = infer_pbs.self_bootstrap_keygen(key, 32)
    rng = np.random.default_rng(33)
    bits = rng.integers(0, 2, (12, 8))
    labels = rng.integers(0, 3, 12)
    erng = tfhe.make_rng(34)
    train = [hewnn.encrypt_sample(bits[i], int(labels[i]), key, erng, label_bits=geom.label_bits)
             for i in range(10)]
    model = hewnn.he_train(train, geom, P)
    test = [hewnn.encrypt_sample(bits[i], None, key, erng) for i in (10, 11)]
    thr = 1
    lookups = hewnn.vp_lookups(model, test)
    preds = infer_pbs.he_infer_bin_batch(model, test, sbk, thr, keep_scores=True)
    boot = infer32.Boot(sbk.params, sbk.bsk)
    want_idx, want_scores = infer32.infer(boot, tfhe.to_host(lookups), 2, geom.l, geom.k0, 16, thr)
    for i in range(2):
        assert_u32_equal(preds[i].index_digits, want_idx[i])
        assert_u32_equal(preds[i].score_digits, want_scores[i])
    plain, _ = wnn.train_integer(bits[:10], labels[:10], geom)
    expect = wnn.evaluate_dataset(plain, bits[10:], wnn.ActivationSpec("bin", thr))
    assert [infer_pbs.decrypt_prediction(p, key) for p in preds] == list(expect)


def test_infer_bin_cfg3_geometry():
    """BASELINE cfg3 geometry (10 classes, 196 RAMs, 8-bit counters): predictions of
    the fully encrypted pipeline == wnn.evaluate_dataset(..., ActivationSpec("bin", thr))."""
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[3]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    key = tfhe.SecretKey(P, tfhe.make_rng(41).integers(0, 2, P.n).astype(np.uint32))
    sbk = infer_pbs.self_bootstrap_keygen(key, 42)
    ds = data.config_dataset(3, n=40, seed=3)
    erng = tfhe.make_rng(43)
    train = [hewnn.encrypt_sample(ds.bits[i], int(ds.labels[i]), key, erng, label_bits=geom.label_bits)
             for i in range(36)]
    model = hewnn.he_train(train, geom, P)
    test = [hewnn.encrypt_sample(ds.bits[i], None, key, erng) for i in range(36, 40)]
    plain, _ = wnn.train_integer(ds.bits[:36], ds.labels[:36], geom)
    for thr in (0, 2):
        preds = infer_pbs.he_infer_bin_batch(model, test, sbk, thr, keep_scores=True)
        expect = wnn.evaluate_dataset(plain, ds.bits[36:], wnn.ActivationSpec("bin", thr))
        assert [infer_pbs.decrypt_prediction(x, key) for x in preds] == list(expect)
        addr = wnn.addresses(ds.bits[36:], geom)
        lookup = plain.counters[:, np.arange(geom.k0)[None, :], addr].transpose(1, 0, 2)   # (S, l, k0)
        for x, want in zip(preds, (lookup > thr).sum(axis=2)):
            assert np.array_equal(infer_pbs.decrypt_scores(x, key), want)
