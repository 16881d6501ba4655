"""GPU parity at the BASELINE sizes, through the default (`ladder="auto"`) path.

The headline number comes from the TMEM FFT ladder (`blind_rotate_fft_td_kernel`,
FFT mode 5, batches >= 8 ciphertexts per SM) fused with the tcgen05 key switch; cfg4 runs the
N = 2048 FFT ladder.  Each test runs a full-size batch (n = 630 / 500 / 750 steps,
including cfg2's partial last 64-step segment, 630 = 9 x 64 + 54), then

* compares a strided sample of >= 128 outputs bit-for-bit with the C oracle
  (exact schoolbook restatement of hw/tfhe.py:340-361 plus the restated KS), and
* compares the WHOLE batch bit-for-bit with the two-prime NTT ladder (an
  independent exact formulation, itself pinned to the oracle and the reference's
  golden fixtures in test_gpu_parity.py).

Inputs are uniform words (a uniform LWE row is distributed like an encryption)
and per-item uniform test polynomials, the worst case for the digit range.
The FFT rounding margin is measured on the instrumented build
(libhwb200_margin.so): the largest |y - rint(y)| over every rounded FFT output
must stay below 2^-6 (the exactness argument needs < 1/2).
"""

import dataclasses

import numpy as np
import pytest
import torch

from conftest import assert_u32_equal
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import named_params

pytestmark = pytest.mark.gpu


def _rand(rng, shape):
    return rng.integers(0, 1 << 32, shape, dtype=np.uint64).astype(np.uint32)


@pytest.fixture(scope="module")
def keys():
    cache = {}

    def get(name):
        if name not in cache:
            P = named_params(name)
            K = tfhe.pbs_keygen(P, 101)
            cache[name] = (P, K, *K.device_keys())
        return cache[name]
    return get


def _run_and_check(coracle, P, K, bsk, ksk, B, seed, sample):
    rng = np.random.default_rng(seed)
    lwe = _rand(rng, (B, P.lwe_n + 1))
    lwe[7, :-1] = 0                                   # every rotation skipped
    lwe[11, ::5] = 0                                  # some rotations skipped
    tvs = _rand(rng, (B, 2, P.n))
    d_lwe, d_tv = tfhe.to_device(lwe), tfhe.to_device(tvs)
    out = tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk))          # default path
    ntt = tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk, ladder="ntt"))
    assert_u32_equal(out, ntt)
    idx = np.unique(np.concatenate([np.linspace(0, B - 1, sample).astype(int), [7, 11, B - 1]]))
    want = coracle.pbs(lwe[idx], tvs[idx], K.bsk, K.ksk, P)
    assert_u32_equal(out[idx], want)
    return lwe, tvs, out


def test_cfg2_full_batch_tmem_ladder(coracle, keys):
    """cfg2, B = 4096: TMEM FFT ladder + tcgen05 key switch (the bench path)."""
    P, K, bsk, ksk = keys("CFG2")
    _run_and_check(coracle, P, K, bsk, ksk, 4096, 1, 192)


def test_cfg2_ragged_tmem_ladder(coracle, keys):
    """cfg2, B = 8 x #SMs + 5: the smallest TMEM-ladder batch, ragged last CTA."""
    P, K, bsk, ksk = keys("CFG2")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _run_and_check(coracle, P, K, bsk, ksk, 8 * sms + 5, 2, 128)


@pytest.mark.parametrize("name,B", [("CFG2", 8 * 148 + 5), ("CFG4", 4 * 148 + 5)])
def test_single_launch_ladder_matches_per_segment_launches(keys, name, B):
    """FFT mode 5 runs the whole ladder as ONE launch whose CTAs are (segment, group) pairs
    waiting on per-group progress words; mode 8 launches once per segment.  Short segments
    (7 steps: 90 / 108 dependent CTAs per group, thousands of waits) on a ragged batch, against
    the per-segment launches, the NTT ladder and a second run on the recycled workspace (the
    progress words are cleared per call)."""
    P, K, bsk, ksk = keys(name)
    rng = np.random.default_rng(77)
    d_lwe = tfhe.to_device(_rand(rng, (B, P.lwe_n + 1)))
    d_tv = tfhe.to_device(_rand(rng, (B, 2, P.n)))
    L = _lib.load()
    try:
        _lib.check(L.hwb_set_fft_segment(7))
        _lib.check(L.hwb_set_fft_mode(8))
        per_segment = tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk, ladder="fft"))
        _lib.check(L.hwb_set_fft_mode(5))
        single = tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk, ladder="fft"))
        again = tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk, ladder="fft"))
    finally:
        _lib.check(L.hwb_set_fft_segment(64))
        _lib.check(L.hwb_set_fft_mode(_lib.FFT_MODE_DEFAULT))
    assert_u32_equal(single, per_segment)
    assert_u32_equal(again, single)
    assert_u32_equal(single, tfhe.to_host(tfhe.pbs_batch(P, d_lwe, d_tv, bsk, ksk, ladder="ntt")))


def test_cfg2_register_ladder_range(coracle, keys):
    """cfg2 batches between one ciphertext per SM and the TMEM threshold (4 per SM)
    run the register FFT ladder (4 CTAs per SM)."""
    P, K, bsk, ksk = keys("CFG2")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _run_and_check(coracle, P, K, bsk, ksk, 3 * sms + 3, 3, 96)


def test_cfg2_tmem_ladder_one_cta_per_sm(coracle, keys):
    """cfg2, B = 4 x #SMs + 3: the TMEM ladder from its threshold (one CTA per SM)."""
    P, K, bsk, ksk = keys("CFG2")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _run_and_check(coracle, P, K, bsk, ksk, 4 * sms + 3, 7, 96)


def test_cfg1_full_batch(coracle, keys):
    P, K, bsk, ksk = keys("CFG1")
    _run_and_check(coracle, P, K, bsk, ksk, 4096, 4, 192)


def test_cfg4_fft2_ladder(coracle, keys):
    """cfg4 (N = 2048, n = 750): the register N = 2048 FFT ladder at B = 320."""
    P, K, bsk, ksk = keys("CFG4")
    _run_and_check(coracle, P, K, bsk, ksk, 320, 5, 64)


def test_cfg4_fft2_tmem_ladder(coracle, keys):
    """cfg4 (N = 2048, n = 750), B = 4 x #SMs + 3: the N = 2048 TMEM ladder
    (blind_rotate_fft2_td_kernel, >= 4 ciphertexts per SM), ragged last CTA."""
    P, K, bsk, ksk = keys("CFG4")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    _run_and_check(coracle, P, K, bsk, ksk, 4 * sms + 3, 6, 64)


def test_cfg2_encrypted_full_batch_decrypts_and_matches(coracle, keys):
    """Encrypted messages (BASELINE configs[1] workload): every output decrypts to
    the negacyclic LUT and a sample equals the oracle."""
    P, K, bsk, ksk = keys("CFG2")
    rng = tfhe.make_rng(42)
    ms = rng.integers(0, P.p, 4096)
    lwe = tfhe.enc_lwe_batch(ms * P.delta, K.lwe_key, rng)
    tv = tfhe.test_polynomial(np.arange(P.p // 2), P)
    out = tfhe.to_host(tfhe.pbs_batch(P, tfhe.to_device(lwe), tv, bsk, ksk))
    dec = tfhe.dec_lwe_batch(out, K.lwe_key)
    assert np.array_equal(dec, np.where(ms < 4, ms, (-(ms - 4)) % 8))
    idx = np.arange(0, 4096, 32)
    assert_u32_equal(out[idx], coracle.pbs(lwe[idx], tv, K.bsk, K.ksk, P))


@pytest.mark.parametrize("name,B", [("CFG2", 1189), ("CFG2", 600), ("CFG2", 447), ("CFG2", 5), ("CFG1", 1189),
                                    ("CFG4", 300),
                                    ("CFG4", 595),
                                    ("INSECURE_1024", 64), ("INSECURE_2048", 64), ("INSECURE_1024W", 64),
                                    ("INSECURE_2048W", 64)])
def test_fft_rounding_margin(name, B, coracle):
    """Instrumented build: max |y - rint(y)| over every rounded FFT output of a
    full-length ladder (TMEM / register / cluster ladders by batch size) with
    extreme key halves and uniform inputs stays < 2^-6 -- and results are still
    bit-identical to the NTT ladder."""
    P = named_params(name)
    if name.startswith("INSECURE"):
        P = dataclasses.replace(P, lwe_n=64)
    K = tfhe.pbs_keygen(P, 202)
    rng = np.random.default_rng(203)
    lwe = _rand(rng, (B, P.lwe_n + 1))
    tvs = _rand(rng, (B, 2, P.n))
    worst = 0.0
    for word in (None, 0x7FFF8000):                 # the real key; the largest |halves| (-2^15, +2^15)
        if word is not None:
            K.bsk[:] = word
        if tfhe.ntt_supported(P):
            ref_bsk, _ = K.device_keys()
            ntt = tfhe.to_host(tfhe.pbs_batch(P, lwe, tvs, ref_bsk, None, ladder="ntt"))
        else:                                       # 16-bit digits: beyond the NTT, check the oracle
            ntt = coracle.pbs(lwe, tvs, K.bsk, None, P, keyswitch=False)
        with _lib.using_library(_lib.MARGIN_LIB_PATH):
            bsk, _ = K.device_keys()
            _lib.fft_margin(reset=True)
            out = tfhe.to_host(tfhe.pbs_batch(P, lwe, tvs, bsk, None, ladder="fft"))
            torch.cuda.synchronize()
            m = _lib.fft_margin()
        assert_u32_equal(out, ntt)
        assert 0.0 < m < 2.0 ** -6, m
        worst = max(worst, m)
    print(f"{name} B={B}: max FFT rounding residual {worst:.3e} = 2^{np.log2(worst):.2f}")


def test_production_build_has_no_margin_counter():
    with pytest.raises(tfhe.TfheError):
        _lib.fft_margin()
