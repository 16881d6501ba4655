"""GPU parity: libhwb200 kernels (through the C ABI) vs the reference-generated
fixtures and the CPU oracle.  Bit-exact everywhere (integer arithmetic mod 2^32)."""

import dataclasses

import numpy as np
import pytest
import torch

from conftest import assert_u32_equal, golden
from oracle import tfhe32 as o
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import HeParams, GadgetSpec, named_params

pytestmark = pytest.mark.gpu


def rand_u32(rng, shape):
    return rng.integers(0, 1 << 32, shape, dtype=np.uint64).astype(np.uint32)


def emb_params(N_log, lv, w, n=0):
    return HeParams("t", N_log, 0.0, GadgetSpec(lv, w), GadgetSpec(8, 2), p=8, lwe_n=n)


@pytest.fixture(params=[0, 1], ids=["regs255", "regs128"])
def variant(request):
    _lib.set_variant(request.param)
    yield request.param
    _lib.set_variant(0)


@pytest.fixture(params=["throughput", "latency"])
def ladder(request):
    """Run the test with the throughput ladder or with every batch on the
    latency-mode ladder (one warp per digit transform)."""
    prev = _lib.set_latency_batch(1 << 40 if request.param == "latency" else 0)
    yield request.param
    _lib.set_latency_batch(prev)


# ---------------------------------------------------------------- external product

@pytest.mark.parametrize("tag,N_log,lv,w", [("cfg2", 10, 3, 7), ("cfg1", 10, 2, 8), ("cfg4", 11, 2, 10)])
def test_ext_product_golden(tag, N_log, lv, w, variant):
    g = golden("ext_product.npz")
    P = emb_params(N_log, lv, w)
    G, cts = g[f"{tag}_G"], g[f"{tag}_cts"]
    assert_u32_equal(tfhe.ext_product_batch(P, G, cts), g[f"{tag}_out"])
    assert_u32_equal(tfhe.ext_product_batch(P, G[:1], cts), g[f"{tag}_out_bcast"])


def test_ext_product_full_precision_gadget_matches_reference():
    """The reference's exact-mode gadget (2 x 16 = 32 bits, hw/params.py:94-101) is
    beyond the two-prime NTT (the C ABI's hwb_ext_product rejects it) and runs on the FP64
    FFT path with 16-bit digits: bit-exact with the reference-generated fixture."""
    g = golden("ext_product.npz")
    P = emb_params(10, 2, 16)
    assert not tfhe.ntt_supported(P)
    assert_u32_equal(tfhe.ext_product_batch(P, g["ins_G"], g["ins_cts"]), g["ins_out"])
    assert_u32_equal(tfhe.ext_product_batch(P, g["ins_G"][:1], g["ins_cts"]), g["ins_out_bcast"])
    with pytest.raises(tfhe.TfheError):
        tfhe.ext_product_batch(P, tfhe.rgsw_to_ntt(emb_params(10, 3, 7), g["cfg2_G"]), g["ins_cts"])


def test_ext_product_random_batch_and_index(coracle):
    rng = np.random.default_rng(11)
    P = emb_params(10, 3, 7)
    G = rand_u32(rng, (7, 6, 2, 1024))
    cts = rand_u32(rng, (64, 2, 1024))
    idx = rng.integers(0, 7, 64)
    ref = coracle.ext_product_batch(G[idx], cts, 3, 7)
    ntt = tfhe.rgsw_to_ntt(P, G)
    assert_u32_equal(tfhe.ext_product_batch(P, ntt, cts, idx=idx), ref)
    # device-resident in, in-place out (aliasing allowed by the ABI)
    d = tfhe.to_device(cts)
    out = tfhe.ext_product_batch(P, ntt, d, idx=idx)
    assert isinstance(out, torch.Tensor)
    assert_u32_equal(tfhe.to_host(out), ref)


def test_ext_product_extreme_inputs(coracle):
    """Maximal-magnitude digits and GGSW words stress the CRT range bound."""
    P = emb_params(10, 3, 7)
    G = np.full((1, 6, 2, 1024), 0x80000000, np.uint32)      # -2^31 everywhere
    cts = np.full((3, 2, 1024), 0, np.uint32)
    cts[0] = 0xFFFFFFFF
    cts[1] = 0x7FFFFFFF
    cts[2, :, ::2] = 0x80000000
    assert_u32_equal(tfhe.ext_product_batch(P, G, cts), coracle.ext_product_batch(G, cts, 3, 7))
    P4 = emb_params(11, 2, 10)
    G4 = np.full((1, 4, 2, 2048), 0x80000000, np.uint32)
    c4 = np.full((2, 2, 2048), 0x7FFFFFFF, np.uint32)
    assert_u32_equal(tfhe.ext_product_batch(P4, G4, c4), coracle.ext_product_batch(G4, c4, 2, 10))


def test_cmux_cdemux(coracle):
    rng = np.random.default_rng(12)
    P = emb_params(10, 3, 7)
    G = rand_u32(rng, (5, 6, 2, 1024))
    c0 = rand_u32(rng, (5, 2, 1024))
    c1 = rand_u32(rng, (5, 2, 1024))
    ext = coracle.ext_product_batch(G, c1 - c0, 3, 7)
    assert_u32_equal(tfhe.cmux_batch(P, G, c1, c0), c0 + ext)
    rot = np.array([0, 1, -7, 2047, 3000])
    c1r = np.stack([o.monomial_mul(c0[i], int(rot[i])) for i in range(5)])
    ext = coracle.ext_product_batch(G, c1r - c0, 3, 7)
    assert_u32_equal(tfhe.cmux_batch(P, G, None, c0, rot=rot), c0 + ext)
    hi = coracle.ext_product_batch(G, c0, 3, 7)
    lo_g, hi_g = tfhe.cdemux_batch(P, G, c0)
    assert_u32_equal(hi_g, hi)
    assert_u32_equal(lo_g, c0 - hi)


# ---------------------------------------------------------------- blind rotation

@pytest.mark.parametrize("tag,N_log,lv,w", [("cfg2", 10, 3, 7), ("cfg4", 11, 2, 10)])
def test_blind_rotate_golden(tag, N_log, lv, w, variant, ladder):
    g = golden("blind_rotate.npz")
    P = emb_params(N_log, lv, w)
    out = tfhe.blind_rotate_batch(P, g[f"{tag}_c"][None], g[f"{tag}_C"], g[f"{tag}_I"][None])[0]
    assert_u32_equal(out, g[f"{tag}_out"])
    ext = tfhe.sample_extract_batch(P, out[None])[0]
    assert_u32_equal(ext[:-1], g[f"{tag}_ext_a"])
    assert int(ext[-1]) == int(g[f"{tag}_ext_b"][0])


def test_blind_rotate_reference_api():
    g = golden("blind_rotate.npz")
    P = emb_params(10, 3, 7)
    c = tfhe.RlweCiphertext(P, g["cfg2_c"])
    C = [tfhe.RgswCiphertext(P, x) for x in g["cfg2_C"]]
    assert_u32_equal(tfhe.blind_rotate(c, C, list(g["cfg2_I"])).data, g["cfg2_out"])
    with pytest.raises(tfhe.TfheError):
        tfhe.blind_rotate(c, C, [1])


def test_blind_rotate_batch_vs_oracle(coracle, ladder):
    rng = np.random.default_rng(13)
    P = emb_params(10, 3, 7)
    L, B = 9, 33
    C = rand_u32(rng, (L, 6, 2, 1024))
    acc = rand_u32(rng, (B, 2, 1024))
    exps = rng.integers(-4096, 4096, (B, L)).astype(np.int32)
    exps[0] = 0                                       # all-skip item
    exps[1, ::2] = 2048                               # exponent == 2N -> skip
    ref = coracle.blind_rotate_batch(acc, C, exps, 3, 7)
    assert_u32_equal(tfhe.blind_rotate_batch(P, acc, C, exps), ref)


@pytest.mark.parametrize("coeff", [0, 1, 17, 1023])
def test_sample_extract_all_positions(coeff):
    rng = np.random.default_rng(14)
    P = emb_params(10, 3, 7)
    c = rand_u32(rng, (2, 1024))
    a, b = o.extract_lwe(c, coeff)
    out = tfhe.extract_lwe(tfhe.RlweCiphertext(P, c), coeff)               # -> LweCiphertext
    assert_u32_equal(out.a, a)
    assert int(out.b) == int(b)
    assert_u32_equal(out.row(), np.concatenate([a, [b]]))


# ---------------------------------------------------------------- key switch and PBS

@pytest.mark.parametrize("lv,w", [(1, 12), (2, 8), (3, 7)])
def test_latency_ladder_gadgets(coracle, lv, w):
    """Latency-mode ladder (4l warps per ciphertext) for every gadget depth."""
    rng = np.random.default_rng(lv)
    P = emb_params(10, lv, w)
    L = 5
    C = rand_u32(rng, (L, 2 * lv, 2, 1024))
    for B in (5, 300):            # 1-CTA/SM build (B <= #SMs) and the 2-CTA/SM build
        acc = rand_u32(rng, (B, 2, 1024))
        exps = rng.integers(-4096, 4096, (B, L)).astype(np.int32)
        exps[0, 1] = 0
        ref = coracle.blind_rotate_batch(acc, C, exps, lv, w)
        prev = _lib.set_latency_batch(1 << 40)
        try:
            out = tfhe.blind_rotate_batch(P, acc, C, exps)
        finally:
            _lib.set_latency_batch(prev)
        assert_u32_equal(out, ref)


def test_keyswitch_vs_oracle(coracle):
    P = dataclasses.replace(named_params("CFG2"), lwe_n=100)
    K = tfhe.pbs_keygen(P, 21)
    _, kd = K.device_keys()
    rng = np.random.default_rng(15)
    for B in (1, 63, 130):
        lwe = rand_u32(rng, (B, P.n + 1))
        gk = P.gadget_ks
        assert_u32_equal(tfhe.lwe_keyswitch(P, lwe, kd), coracle.keyswitch(lwe, K.ksk, gk.levels, gk.base_log))


@pytest.mark.parametrize("N_log,ks,n", [(10, (8, 2), 630), (10, (7, 2), 500), (11, (8, 2), 750),
                                        (10, (4, 8), 70), (10, (3, 7), 64), (10, (1, 1), 1)])
def test_keyswitch_tensor_cores_vs_oracle(coracle, N_log, ks, n):
    """tcgen05 int8 key switch: bit-exact with the C oracle and the integer-pipe
    kernel on ragged batches (partial 128-item and 64-column tiles), the full int8
    digit range (base_log 8) and extreme words."""
    P = HeParams("t", N_log, 0.0, GadgetSpec(2, 8), GadgetSpec(*ks), p=8, lwe_n=n)
    rng = np.random.default_rng(n + N_log)
    ksk = rand_u32(rng, (P.n, ks[0], n + 1))
    kd = tfhe.LweKeySwitchKey(P, tfhe.to_device(ksk))
    assert kd.tensor_core_tiles() is not None
    for B in (1, 127, 129, 300):
        lwe = rand_u32(rng, (B, P.n + 1))
        lwe[0, :] = 0xFFFFFFFF
        if B > 1:
            lwe[1, :] = 0
            lwe[-1, :] = 0x80000000
        want = coracle.keyswitch(lwe, ksk, ks[0], ks[1])
        assert_u32_equal(tfhe.lwe_keyswitch(P, lwe, kd, engine="tc"), want)
        assert_u32_equal(tfhe.lwe_keyswitch(P, lwe, kd, engine="simt"), want)


def test_keyswitch_tensor_cores_full_batch():
    """BASELINE cfg2 size: tensor-core and integer-pipe key switch agree on 4096 items."""
    P = named_params("CFG2")
    rng = np.random.default_rng(77)
    ksk = rand_u32(rng, (P.n, P.gadget_ks.levels, P.lwe_n + 1))
    kd = tfhe.LweKeySwitchKey(P, tfhe.to_device(ksk))
    lwe = tfhe.to_device(rand_u32(rng, (4096, P.n + 1)))
    a = tfhe.lwe_keyswitch(P, lwe, kd, engine="tc")
    b = tfhe.lwe_keyswitch(P, lwe, kd, engine="simt")
    assert torch.equal(a, b)


def test_keyswitch_engine_selection():
    P = HeParams("t", 10, 0.0, GadgetSpec(2, 8), GadgetSpec(2, 10), p=8, lwe_n=16)
    kd = tfhe.LweKeySwitchKey(P, tfhe.to_device(np.zeros((P.n, 2, 17), np.uint32)))
    assert kd.tensor_core_tiles() is None             # base_log 10: digits exceed int8
    lwe = np.ones((3, P.n + 1), np.uint32)
    with pytest.raises(tfhe.TfheError):
        tfhe.lwe_keyswitch(P, lwe, kd, engine="tc")
    with pytest.raises(tfhe.TfheError):
        tfhe.lwe_keyswitch(P, lwe, kd, engine="bogus")
    assert tfhe.lwe_keyswitch(P, lwe, kd).shape == (3, 17)   # auto -> integer pipe


@pytest.mark.parametrize("name", ["CFG1", "CFG2", "CFG4"])
def test_pbs_golden(name, variant, ladder):
    P = named_params(name)
    g = golden(f"pbs_{name.lower()}.npz")
    K = tfhe.pbs_keygen(P, int(g["key_seed"]))
    bsk, ksk = K.device_keys()
    ext = tfhe.pbs_batch(P, g["lwe_in"], g["tv"], bsk, None)
    assert_u32_equal(ext, g["extracted"])
    for engine in ("tc", "simt"):
        out = tfhe.pbs_batch(P, g["lwe_in"], g["tv"], bsk, ksk, engine=engine)
        assert_u32_equal(out, g["lwe_out"])
    if bsk.fft is not None:                       # FP64 FFT ladder (N = 1024, 2048)
        assert_u32_equal(tfhe.pbs_batch(P, g["lwe_in"], g["tv"], bsk, None, ladder="fft"), g["extracted"])
        for engine in ("tc", "simt"):
            out = tfhe.pbs_batch(P, g["lwe_in"], g["tv"], bsk, ksk, engine=engine, ladder="fft")
            assert_u32_equal(out, g["lwe_out"])


def test_pbs_batch_vs_c_oracle_and_decrypt(coracle, ladder):
    P = named_params("CFG2")
    K = tfhe.pbs_keygen(P, 31)
    bsk, ksk = K.device_keys()
    rng = tfhe.make_rng(32)
    B = 48
    ms = rng.integers(0, P.p, B)
    lwe = tfhe.enc_lwe_batch(ms * P.delta, K.lwe_key, rng)
    lwe[0, :-1] = 0                                        # every rotation skipped
    tv = tfhe.test_polynomial(np.arange(4), P)
    out = tfhe.pbs_batch(P, lwe, tv, bsk, ksk)
    assert_u32_equal(out, coracle.pbs(lwe, tv, K.bsk, K.ksk, P))
    # per-item test polynomials (sign LUT for odd items)
    tvs = np.stack([tv if i % 2 == 0 else tfhe.test_polynomial(np.ones(4, int), P) for i in range(B)])
    out2 = tfhe.pbs_batch(P, lwe, tvs, bsk, ksk)
    assert_u32_equal(out2, coracle.pbs(lwe, tvs, K.bsk, K.ksk, P))


@pytest.mark.parametrize("name", ["CFG1", "CFG2", "CFG4", "INSECURE_2048"])
def test_pbs_fft_ladder_vs_c_oracle(coracle, name):
    """FP64 FFT ladder: bit-exact with the C oracle (schoolbook) on random inputs,
    per-item test polynomials, several segment lengths and a ragged batch."""
    P = dataclasses.replace(named_params(name), lwe_n=40)
    K = tfhe.pbs_keygen(P, 61)
    bsk, ksk = K.device_keys()
    assert bsk.fft is not None
    rng = np.random.default_rng(62)
    lwe = rand_u32(rng, (37, P.lwe_n + 1))
    lwe[3, :-1] = 0                                    # every rotation skipped (exact no-op steps)
    lwe[5, ::3] = 0                                    # some rotations skipped
    tvs = rand_u32(rng, (37, 2, P.n))
    want = coracle.pbs(lwe, tvs, K.bsk, K.ksk, P)
    L = _lib.load()
    prev = L.hwb_set_fft_latency_batch(0)               # throughput ladder
    try:
        _lib.check(L.hwb_set_fft_mode(0))               # register accumulators, 1/2/4 items per CTA
        for seg, group in ((1, 1), (7, 2), (64, 4), (64, 1)):
            _lib.check(L.hwb_set_fft_segment(seg))
            _lib.check(L.hwb_set_fft_group(group))     # ragged: 37 items in CTAs of 1, 2 or 4
            assert_u32_equal(tfhe.pbs_batch(P, lwe, tvs, bsk, ksk, ladder="fft"), want)
        sms = torch.cuda.get_device_properties(0).multi_processor_count
        big = 8 * sms + 5                               # the TMEM ladders need >= 8 items per SM; ragged
        rep = np.resize(np.arange(37), big)
        want_big = want[rep]
        for mode in _lib.FFT_MODES[1:]:                  # TMEM accumulators: every CTA shape
            _lib.check(L.hwb_set_fft_mode(mode))
            for seg in (1, 64):
                _lib.check(L.hwb_set_fft_segment(seg))
                assert_u32_equal(tfhe.pbs_batch(P, lwe[rep], tvs[rep], bsk, ksk, ladder="fft"), want_big)
        L.hwb_set_fft_latency_batch(1 << 40)            # latency ladder (N = 1024)
        assert_u32_equal(tfhe.pbs_batch(P, lwe, tvs, bsk, ksk, ladder="fft"), want)
        assert_u32_equal(tfhe.pbs_batch(P, lwe[:1], tvs[:1], bsk, ksk, ladder="fft"), want[:1])
        prev_cl = L.hwb_set_fft_cluster_batch(1 << 40)  # cluster ladder: 2l CTAs per ciphertext
        try:
            for cmode in (0, 1):                        # 2l CTAs per ciphertext / 4 CTAs
                _lib.check(L.hwb_set_fft_cluster_mode(cmode))
                assert_u32_equal(tfhe.pbs_batch(P, lwe, tvs, bsk, ksk, ladder="fft"), want)
                assert_u32_equal(tfhe.pbs_batch(P, lwe[:1], tvs[:1], bsk, ksk, ladder="fft"), want[:1])
        finally:
            L.hwb_set_fft_cluster_batch(prev_cl)
            _lib.check(L.hwb_set_fft_cluster_mode(0))
    finally:
        _lib.check(L.hwb_set_fft_segment(64))
        _lib.check(L.hwb_set_fft_group(1))
        _lib.check(L.hwb_set_fft_mode(_lib.FFT_MODE_DEFAULT))
        L.hwb_set_fft_latency_batch(prev)


@pytest.mark.parametrize("name", ["CFG2", "CFG4"])
def test_pbs_fft_ladder_extreme_key(name):
    """Largest-magnitude key halves (word 0x7FFF8000: lo = -2^15, hi = +2^15) and
    all-ones / alternating inputs: the rounding margin's worst case, checked
    against the NTT ladder (itself pinned to the oracle)."""
    P = dataclasses.replace(named_params(name), lwe_n=24)
    K = tfhe.pbs_keygen(P, 71)
    for word in (0x7FFF8000, 0x80000000, 0x7FFFFFFF):
        K.bsk[:] = word
        bsk, _ = K.device_keys()
        lwe = np.full((8, P.lwe_n + 1), 0xFFFFFFFF, np.uint32)
        lwe[1::2, ::2] = 0x55555555
        lwe[2] = np.arange(P.lwe_n + 1, dtype=np.uint32) * 0x9E3779B9
        tv = np.full((2, P.n), 0x7FFFFFFF, np.uint32)
        a = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="fft")   # 8 items: latency ladder at N = 1024
        b = tfhe.pbs_batch(P, lwe, tv, bsk, None, ladder="ntt")
        assert_u32_equal(a, b)


def test_pbs_full_batch_decrypts():
    """BASELINE cfg2 size (4096): size-independent property -- every output
    decrypts to the negacyclic LUT of its input (identity on [0, 4))."""
    P = named_params("CFG2")
    K = tfhe.pbs_keygen(P, 41)
    bsk, ksk = K.device_keys()
    rng = tfhe.make_rng(42)
    ms = rng.integers(0, P.p, 4096)
    lwe = tfhe.enc_lwe_batch(ms * P.delta, K.lwe_key, rng)
    out = tfhe.pbs_batch(P, tfhe.to_device(lwe), tfhe.test_polynomial(np.arange(4), P), bsk, ksk)
    dec = tfhe.dec_lwe_batch(tfhe.to_host(out), K.lwe_key)
    expect = np.where(ms < 4, ms, (-(ms - 4)) % 8)
    assert np.array_equal(dec, expect)
    # chaining: a second PBS of the outputs is the LUT applied twice
    out2 = tfhe.pbs_batch(P, out, tfhe.test_polynomial(np.arange(4), P), bsk, ksk)
    dec2 = tfhe.dec_lwe_batch(tfhe.to_host(out2), K.lwe_key)
    assert np.array_equal(dec2, np.where(expect < 4, expect, (-(expect - 4)) % 8))


def test_pbs_empty_and_errors():
    P = named_params("CFG2")
    K = tfhe.pbs_keygen(dataclasses.replace(P, lwe_n=4), 1)
    P4 = dataclasses.replace(P, lwe_n=4)
    bsk, ksk = K.device_keys()
    tv = tfhe.test_polynomial(np.arange(4), P4)
    out = tfhe.pbs_batch(P4, np.zeros((0, 5), np.uint32), tv, bsk, ksk)
    assert out.shape == (0, 5)
    with pytest.raises(tfhe.TfheError):
        tfhe.pbs_batch(P4, np.zeros((2, 7), np.uint32), tv, bsk, ksk)
    with pytest.raises(tfhe.TfheError):
        tfhe.pbs_batch(P, np.zeros((2, 631), np.uint32), tfhe.test_polynomial(np.arange(4), P), bsk, ksk)
