"""Host-side logic of the product (client key generation/encryption, parameter
handling) must be bit-identical to the oracle -- CPU only, no GPU calls."""

import dataclasses

import numpy as np
import pytest

from conftest import assert_u32_equal, golden
from oracle import tfhe32 as o
from paper_2403_20190_b200 import tfhe
from paper_2403_20190_b200.params import GadgetSpec, HeParams, named_params, param_set_names


def test_named_params():
    P = named_params("CFG2")
    assert (P.n, P.lwe_n, P.gadget, P.gadget_ks, P.p) == (1024, 630, GadgetSpec(3, 7), GadgetSpec(8, 2), 8)
    assert P.delta == 1 << 29
    assert P.sigma == 2.0 ** 7 and P.lwe_sigma == 2.0 ** 17
    assert named_params("CFG4").n == 2048 and named_params("CFG4").lwe_n == 750
    assert named_params("CFG1").gadget == GadgetSpec(2, 8)
    assert {"CFG1", "CFG2", "CFG3", "CFG4", "CFG5"} <= set(param_set_names())
    with pytest.raises(KeyError):
        named_params("NOPE")


def test_param_validation():
    # reference hw/params.py:27-31, 60-66
    with pytest.raises(ValueError):
        GadgetSpec(0, 7)
    with pytest.raises(ValueError):
        GadgetSpec(5, 7)          # 35 bits > q
    with pytest.raises(ValueError):
        HeParams("x", 10, 0.0, GadgetSpec(3, 7), GadgetSpec(8, 2), p=6)
    with pytest.raises(ValueError):
        HeParams("x", 1, 0.0, GadgetSpec(3, 7), GadgetSpec(8, 2), p=8)


def test_key_mul_host_matches_oracle():
    rng = np.random.default_rng(1)
    s = rng.integers(0, 2, 2048).astype(np.uint32)
    a = rng.integers(0, 1 << 32, (3, 2, 2048), dtype=np.uint64).astype(np.uint32)
    assert_u32_equal(tfhe._key_mul_host(a, s), o.key_mul(a, s))


@pytest.mark.parametrize("name", ["CFG1", "CFG2"])
def test_pbs_keygen_matches_oracle(name):
    P = named_params(name)
    seed = int(golden(f"pbs_{name.lower()}.npz")["key_seed"])
    K = tfhe.pbs_keygen(P, seed)
    R = o.pbs_keygen(P, seed)
    assert_u32_equal(K.lwe_key.s, R["s0"])
    assert_u32_equal(K.glwe_key.s, R["s1"])
    assert_u32_equal(K.bsk, R["bsk"])
    assert_u32_equal(K.ksk, R["ksk"])


def test_encrypt_and_tv_match_oracle():
    P = named_params("CFG2")
    g = golden("pbs_cfg2.npz")
    K = tfhe.pbs_keygen(dataclasses.replace(P, lwe_n=630), int(g["key_seed"]))
    rng = tfhe.make_rng(int(g["enc_seed"]))
    ms = rng.integers(0, P.p, len(g["ms"]))
    lwe = tfhe.enc_lwe_batch(ms * P.delta, K.lwe_key, rng)
    assert_u32_equal(lwe, g["lwe_in"])
    assert_u32_equal(tfhe.test_polynomial(np.arange(4), P), g["tv"])
    assert np.array_equal(tfhe.dec_lwe_batch(lwe, K.lwe_key), ms)


def test_rgsw_and_rlwe_roundtrip():
    P = named_params("CFG2")
    key = tfhe.SecretKey(P, tfhe.make_rng(1).integers(0, 2, P.n).astype(np.uint32))
    rng = tfhe.make_rng(2)
    m = rng.integers(0, P.p, P.n)
    c = tfhe.enc_rlwe(m, key, rng)
    assert np.array_equal(tfhe.dec_rlwe(c, key), m)
    for bit in (0, 1):
        assert tfhe.dec_rgsw(tfhe.enc_rgsw(bit, key, rng), key) == bit
    with pytest.raises(tfhe.EncodingError):
        tfhe.enc_rgsw(2, key, rng)
    with pytest.raises(tfhe.EncodingError):
        tfhe.enc_rlwe([P.p], key, rng)
    # the same stream as the oracle restatement of hw/tfhe.py:246-263
    r1, r2 = tfhe.make_rng(7), o.make_rng(7)
    a = np.stack([x.data for x in tfhe.enc_rgsw_batch([0, 1, 1], key, r1)])
    b = o.enc_rgsw_batch([0, 1, 1], key.s, P.sigma, 3, 7, r2)
    assert_u32_equal(a, b)


def test_mod_switch_matches_oracle():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 1 << 32, 10000, dtype=np.uint64).astype(np.uint32)
    for N in (1024, 2048):
        assert np.array_equal(tfhe.mod_switch(x, N), o.mod_switch(x, N))


def test_test_polynomial_validation():
    P = named_params("CFG2")
    with pytest.raises(tfhe.TfheError):
        tfhe.test_polynomial(np.arange(8), P)


def test_philox_take_matches_numpy_stream():
    """tfhe.philox_take claims the next words of rng.bytes() (hw/tfhe.py:38-40) without
    drawing them: regenerating them from the returned state (host restatement of the
    GPU kernel) gives rng.bytes's words, and the generator continues identically
    (uint32 buffer, uint64 buffer and counter), also after normals."""
    import numpy as np
    from paper_2403_20190_b200 import tfhe
    for pre in (0, 1, 3, 8, 9, 13):
        for n in (1, 2, 5, 7, 8, 9, 16, 17, 1000, 1001):
            r1, r2 = tfhe.make_rng(5), tfhe.make_rng(5)
            if pre:
                r1.bytes(4 * pre)
                r2.bytes(4 * pre)
            r1.normal(size=3)
            r2.normal(size=3)
            want = np.frombuffer(r1.bytes(4 * n), dtype="<u4")
            st = tfhe.philox_take(r2, n)
            words = list(st.prefix[: st.nprefix])
            g = 0
            while len(words) < n:
                g += 1
                for u in tfhe.philox4x64(tfhe._ctr_add(list(st.ctr), g), list(st.key)):
                    words += [u & 0xFFFFFFFF, u >> 32]
            assert list(want) == words[:n], (pre, n)
            assert np.array_equal(r1.bytes(44), r2.bytes(44))
            assert np.array_equal(r1.normal(size=5), r2.normal(size=5))
            assert np.array_equal(r1.integers(0, 2, 7), r2.integers(0, 2, 7))
