"""GPU parity for encrypted WiSARD training/LUT evaluation: the device
IVP/VP engine and he_train vs the reference-generated fixtures and the oracle."""

import hashlib
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN, assert_u32_equal, golden
from oracle import tfhe32 as o
from oracle import wnn32
from paper_2403_20190_b200 import hewnn, lut, tfhe, wnn
from paper_2403_20190_b200.params import named_params

sys.path.insert(0, GOLDEN)
from cases import TRAIN_CASES, train_inputs  # noqa: E402

pytestmark = pytest.mark.gpu


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def samples_of(name, device=True):
    P, s1, bits, labels, stacks = train_inputs(name)
    s, l, a, r = TRAIN_CASES[name][2]
    lb = max(1, (l - 1).bit_length())
    smp = [hewnn.EncryptedSample.from_stack(P, tfhe.to_device(st) if device else st, s, lb) for st in stacks]
    return P, s1, bits, labels, smp, wnn.WisardGeometry(s, l, a, r, P.p)


@pytest.mark.parametrize("name", sorted(TRAIN_CASES))
@pytest.mark.parametrize("batch", [1, 16])
@pytest.mark.parametrize("ladder", ["fft", "ntt"])
def test_he_train_matches_reference(name, batch, ladder):
    g = golden(f"{name}.npz")
    P, s1, bits, labels, smp, geom = samples_of(name)
    model = hewnn.he_train(smp, geom, P, batch=batch, ladder=ladder)
    rams = tfhe.to_host(model.rams)
    assert sha(rams) == str(g["sha_rams"])
    assert_u32_equal(rams[:, :2], g["rams_head"])
    assert_u32_equal(tfhe.to_host(model.counts_ct), g["counts_ct"])
    plain, cc = hewnn.decrypt_model(model, tfhe.SecretKey(P, s1))
    assert np.array_equal(plain.counters, g["counters"])
    assert np.array_equal(cc.counts, g["class_counts"])


@pytest.mark.parametrize("host", ["numpy", "pinned"])
def test_he_train_from_host_stacks_staged(host):
    """Host RGSW stacks go through the two-slot staging ring (chunks of 1 sample,
    so every slot is reused several times): bit-identical to device-resident input."""
    name = sorted(TRAIN_CASES)[0]
    g = golden(f"{name}.npz")
    P, s1, bits, labels, smp, geom = samples_of(name, device=False)
    if host == "pinned":
        smp = [hewnn.EncryptedSample.from_stack(P, torch.from_numpy(x.rgsw.view(np.int32)).pin_memory(), x.s, x.n_label_bits)
               for x in smp]
    for batch in (1, 2):
        model = hewnn.he_train(smp, geom, P, batch=batch)
        assert sha(tfhe.to_host(model.rams)) == str(g["sha_rams"])
        assert_u32_equal(tfhe.to_host(model.counts_ct), g["counts_ct"])


def test_continuous_training_and_merge():
    name = "train_cfg1"
    P, s1, bits, labels, smp, geom = samples_of(name)
    full = hewnn.he_train(smp, geom, P)
    part = hewnn.he_train(smp[:1], geom, P)
    cont = hewnn.he_train(smp[1:], geom, P, model=part.copy())               # hw/hewnn.py:189-202
    assert torch.equal(cont.rams, full.rams) and torch.equal(cont.counts_ct, full.counts_ct)
    other = hewnn.he_train(smp[1:], geom, P)
    merged = hewnn.he_merge(part, other)                                    # hw/hewnn.py:264-271
    assert torch.equal(merged.rams, full.rams) and torch.equal(merged.counts_ct, full.counts_ct)


def test_device_rgsw_encryption_matches_host():
    P = named_params("CFG2", 256)
    key = tfhe.SecretKey(P, tfhe.make_rng(3).integers(0, 2, P.n).astype(np.uint32))
    ms = tfhe.make_rng(4).integers(0, 2, 37)
    host = np.stack([c.data for c in tfhe.enc_rgsw_batch(ms, key, tfhe.make_rng(5))])
    dev = hewnn.enc_rgsw_batch_device(ms, key, tfhe.make_rng(5))
    assert_u32_equal(tfhe.to_host(dev), host)
    P4 = named_params("CFG4")
    key4 = tfhe.SecretKey(P4, tfhe.make_rng(3).integers(0, 2, P4.n).astype(np.uint32))
    host4 = np.stack([c.data for c in tfhe.enc_rgsw_batch(ms[:5], key4, tfhe.make_rng(6))])
    assert_u32_equal(tfhe.to_host(hewnn.enc_rgsw_batch_device(ms[:5], key4, tfhe.make_rng(6))), host4)


def test_device_key_cache_never_stale():
    """Advisor finding: the device image of a secret key must follow the key object
    (a fresh key at a reused address, or a key changed in place, is re-uploaded)."""
    P = named_params("CFG2", 256)
    ms = tfhe.make_rng(4).integers(0, 2, 9)
    for seed in (11, 12, 13):                        # keys created and dropped in sequence
        key = tfhe.SecretKey(P, tfhe.make_rng(seed).integers(0, 2, P.n).astype(np.uint32))
        host = np.stack([c.data for c in tfhe.enc_rgsw_batch(ms, key, tfhe.make_rng(5))])
        assert_u32_equal(tfhe.to_host(hewnn.enc_rgsw_batch_device(ms, key, tfhe.make_rng(5))), host)
        del key
    key = tfhe.SecretKey(P, tfhe.make_rng(14).integers(0, 2, P.n).astype(np.uint32))
    hewnn.enc_rgsw_batch_device(ms, key, tfhe.make_rng(5))
    key.s[:] = 1 - key.s                             # mutated in place
    host = np.stack([c.data for c in tfhe.enc_rgsw_batch(ms, key, tfhe.make_rng(5))])
    assert_u32_equal(tfhe.to_host(hewnn.enc_rgsw_batch_device(ms, key, tfhe.make_rng(5))), host)
    for c, m in zip(tfhe.enc_rgsw_batch(ms, key, tfhe.make_rng(6)), ms):
        assert tfhe.dec_rgsw(c, key) == m


def _random_codes(rng, B, k, R, clear_frac=0.25):
    codes = rng.integers(0, R, (B, k))
    mask = rng.random((B, k)) < clear_frac
    codes[mask] = rng.choice([lut.CLEAR0, lut.CLEAR1], size=mask.sum())
    return codes


@pytest.mark.parametrize("name,p", [("CFG2", 256), ("CFG4", 4096)])
@pytest.mark.parametrize("k", [4, 12, 13])
def test_ivp_vp_codes_vs_oracle(k, name, p):
    """Random selector matrices mixing encrypted and clear bits, tree (k > log2 N)
    and rotation-only shapes, N = 1024 and 2048, on both ladders."""
    P = named_params(name, p)
    gl, gb = P.gadget.levels, P.gadget.base_log
    rng = np.random.default_rng(k)
    R = 6
    table = rng.integers(0, 1 << 32, (R, 2 * gl, 2, P.n), dtype=np.uint64).astype(np.uint32)
    payload = rng.integers(0, 1 << 32, (2, P.n), dtype=np.uint64).astype(np.uint32)
    codes = _random_codes(rng, 5, k, R)
    want = wnn32.ivp_batch(codes, table, payload, gl, gb, P.degree_log)
    z = lut.tree_depth(k, P)
    luts = rng.integers(0, 1 << 32, (3, max(1, 1 << z), 2, P.n), dtype=np.uint64).astype(np.uint32)
    lut_idx = rng.integers(0, 3, 5)
    vcodes = _random_codes(rng, 5, k, R)
    vcodes[:, 0] = lut.CLEAR1                       # exercise the clear-prefix slicing
    vwant = wnn32.vp_batch(vcodes, table, luts[lut_idx], gl, gb, P.degree_log)
    for tab in (tfhe.rgsw_to_ntt(P, table), tfhe.rgsw_to_fft(P, table)):     # both ladders
        assert_u32_equal(tfhe.to_host(lut.ivp_codes(P, codes, tab, payload)), want)
        got = tfhe.to_host(lut.vp_codes(P, vcodes, tab, tfhe.to_device(luts), lut_idx))
        assert_u32_equal(got, vwant)


def test_lut_roundtrip_decrypts():
    """VP(IVP(payload)) exposes the payload at the selected entry (pkg/tests/test_lut.py:170-181)."""
    P = named_params("CFG2", 256)
    key = tfhe.SecretKey(P, tfhe.make_rng(8).integers(0, 2, P.n).astype(np.uint32))
    rng = tfhe.make_rng(9)
    k = 12
    for m in (0, 1, 1023, 1024, 4095):
        bits = [(m >> (k - 1 - i)) & 1 for i in range(2)] + [(m >> w) & 1 for w in range(10)]
        sel = [lut.SelectorBit.enc(c) for c in tfhe.enc_rgsw_batch(bits, key, rng)]
        assert lut.selector_index(bits, k, P) == m
        rows = lut.ivp_batch([sel], tfhe.trivial_rlwe(5, P).data, P)[0]        # (4, 2, N)
        dec = np.concatenate([tfhe.dec_rlwe(tfhe.RlweCiphertext(P, r), key) for r in rows])
        expect = np.zeros(4 * P.n, dtype=np.int64)
        expect[m] = 5
        assert np.array_equal(dec, expect)
        out = lut.vertical_packing(sel, lut.EncryptedLut([tfhe.RlweCiphertext(P, r) for r in rows], k))
        assert isinstance(out, tfhe.LweCiphertext) and tfhe.dec_lwe(out, key) == 5


def test_monomial_gather_vs_oracle():
    P = named_params("CFG2")
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 32, (6, 2, P.n), dtype=np.uint64).astype(np.uint32)
    es = np.array([0, 1, -1, 2047, 3000, -5000])
    assert_u32_equal(lut.monomial_gather(P, x, es), o.monomial_gather(x, es))


def test_pack_batch_and_he_infer_pd_match_reference():
    g = golden("infer_tree.npz")
    name = "train_tree"
    P, s1, bits, labels, smp, geom = samples_of(name)
    key, pksk = tfhe.keygen(P, TRAIN_CASES[name][4])
    assert np.array_equal(key.s, s1)
    assert_u32_equal(tfhe.pack_batch(g["pack_a"], g["pack_b"], pksk), g["pack_out"])     # hw/tfhe.py:390
    model = hewnn.he_train(smp, geom, P)
    test_rgsw = o.enc_rgsw_batch(g["test_bits"], s1, P.sigma, P.gadget.levels, P.gadget.base_log, o.make_rng(13))
    assert sha(test_rgsw) == str(g["sha_test_rgsw"])
    tsample = hewnn.EncryptedSample.from_stack(P, tfhe.to_device(test_rgsw), geom.s, 0)
    pack = hewnn.he_infer_pd(model, tsample, pksk)                                         # hw/hewnn.py:278
    assert_u32_equal(pack.packed, g["infer_packed"])
    assert_u32_equal(hewnn.he_infer_pd_batch(model, [tsample], pksk, ladder="ntt")[0].packed, g["infer_packed"])
    fin = hewnn.client_finalize(pack, key, wnn.ActivationSpec("bin", 0))
    assert np.array_equal(fin.raw, g["raw"]) and fin.prediction == int(g["prediction"])
    assert fin.noise_ok
    # batched inference over several samples equals per-sample calls
    packs = hewnn.he_infer_pd_batch(model, [tsample, smp[0], tsample], pksk)
    assert_u32_equal(packs[0].packed, g["infer_packed"])
    assert_u32_equal(packs[2].packed, g["infer_packed"])
    assert_u32_equal(packs[1].packed, hewnn.he_infer_pd(model, smp[0], pksk).packed)


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_full_geometry_training_vs_oracle(cfg):
    """BASELINE configs' real geometries (cfg4: N = 2048, a = 16, 9 tree levels,
    512 polynomials per RAM row) on one encrypted image: GPU he_train is
    bit-exact with the oracle's restatement of hw/hewnn.py:189-229, and (where
    the noise budget allows) decrypts to train_integer."""
    from paper_2403_20190_b200 import data
    (s, l, a, r, p), pname = data.CONFIG_GEOMETRY[cfg]
    P = named_params(pname, p)
    geom = wnn.WisardGeometry(s, l, a, r, p)
    ds = data.config_dataset(cfg, n=1, seed=5)
    key = tfhe.SecretKey(P, tfhe.make_rng(6).integers(0, 2, P.n).astype(np.uint32))
    smp = hewnn.encrypt_sample(ds.bits[0], int(ds.labels[0]), key, tfhe.make_rng(7), label_bits=geom.label_bits)
    model = hewnn.he_train([smp], geom, P)
    rams, counts = wnn32.he_train([tfhe.to_host(smp.rgsw)], s, l, a, r, P)
    assert_u32_equal(tfhe.to_host(model.rams), rams)
    assert_u32_equal(tfhe.to_host(model.counts_ct), counts)
    if cfg != 4:
        plain, cc = hewnn.decrypt_model(model, key)
        ref, rc = wnn.train_integer(ds.bits, ds.labels, geom)
        assert np.array_equal(plain.counters, ref.counters) and np.array_equal(cc.counts, rc.counts)


def test_he_train_multi_equals_separate_runs():
    """hw/hewnn.py:232-261: multi-seed training in one pass == per-seed he_train."""
    name = "train_cfg1"
    P, s1, bits, labels, smp, geom = samples_of(name)
    geoms = [geom, wnn.WisardGeometry(geom.s, geom.l, geom.a, 11, geom.p)]
    multi = hewnn.he_train_multi(smp, geoms, P, batch=2)
    for g, m in zip(geoms, multi):
        single = hewnn.he_train(smp, g, P)
        assert torch.equal(m.rams, single.rams) and torch.equal(m.counts_ct, single.counts_ct)


def test_client_helpers():
    name = "train_cfg1"
    P, s1, bits, labels, smp, geom = samples_of(name)
    key = tfhe.SecretKey(P, s1)
    dbits, dlab = hewnn.decrypt_sample(smp[0], key)                          # hw/hewnn.py:122-130
    assert dbits == list(bits[0]) and dlab == int(labels[0])
    model = hewnn.he_train(smp, geom, P)
    nb = tfhe.measure_noise(tfhe.RlweCiphertext(P, tfhe.to_host(model.rams[0, 0])), key)
    assert nb.ok and nb.max_abs == hewnn.model_noise(model, key)[0] or nb.max_abs <= hewnn.model_noise(model, key)[0]
    rows = lut.ivp_batch([[lut.SelectorBit.clear(1)] * 4], tfhe.trivial_rlwe(3, P).data, P)[0]
    polys = lut.EncryptedLut([tfhe.RlweCiphertext(P, r) for r in rows], 4)
    vals = lut.decode_lut(lut.lut_add(polys, polys), key)                     # hw/lut.py:100-110
    expect = np.zeros(16, dtype=np.int64)
    expect[15] = 6
    assert np.array_equal(vals, expect)
