"""Race stress (compute-sanitizer is closed on this pool, profiles/r02_sanitizer.txt):
the kernels that synchronise through mbarriers, st.async / red.async across cluster
CTAs, TMEM and tcgen05 are re-run many times while another stream keeps the SMs
busy (perturbing the relative timing of CTAs), and every result is compared bit for
bit with an independent formulation (the two-prime NTT ladder / integer-pipe key
switch).  A lost ordering (e.g. the cluster ladder's partial-product buffer reuse,
DESIGN.md §3d) would show up as a mismatch."""

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


def test_cluster_and_tmem_ladders_under_contention():
    P = dataclasses.replace(named_params("CFG2"), lwe_n=64)
    K = tfhe.pbs_keygen(P, 5)
    bsk, ksk = K.device_keys()
    rng = np.random.default_rng(6)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cases = {B: (tfhe.to_device(_rand(rng, (B, P.lwe_n + 1))), tfhe.to_device(_rand(rng, (B, 2, P.n))))
             for B in (1, 3, 22, 8 * sms + 5)}
    want = {B: tfhe.to_host(tfhe.pbs_batch(P, l, t, bsk, ksk, ladder="ntt", engine="simt"))
            for B, (l, t) in cases.items()}
    # background load: a big TMEM-ladder batch on a second stream
    bg = torch.cuda.Stream()
    big_l = tfhe.to_device(_rand(rng, (4 * 8 * sms, P.lwe_n + 1)))
    big_t = tfhe.to_device(_rand(rng, (2, P.n)))
    L = _lib.load()
    prev = L.hwb_set_fft_cluster_batch(-2)
    try:
        for mode in (0, 1):                                  # 2l-CTA and 4-CTA cluster ladders
            _lib.check(L.hwb_set_fft_cluster_mode(mode))
            outs = []
            for it in range(40):
                with torch.cuda.stream(bg):
                    tfhe.pbs_batch(P, big_l, big_t, bsk, None, ladder="fft")
                for B, (l, t) in cases.items():
                    outs.append((B, tfhe.pbs_batch(P, l, t, bsk, ksk, ladder="fft")))
            torch.cuda.synchronize()
            for B, o in outs:
                assert_u32_equal(tfhe.to_host(o), want[B])
    finally:
        _lib.check(L.hwb_set_fft_cluster_mode(0))
        L.hwb_set_fft_cluster_batch(prev)


def test_tensor_core_keyswitch_under_contention():
    P = named_params("CFG2")
    K = tfhe.pbs_keygen(dataclasses.replace(P, lwe_n=630), 7)
    _, ksk = K.device_keys()
    rng = np.random.default_rng(8)
    ext = tfhe.to_device(_rand(rng, (129, P.n + 1)))
    want = tfhe.to_host(tfhe.lwe_keyswitch(P, ext, ksk, engine="simt"))
    bg = torch.cuda.Stream()
    junk = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    outs = []
    for it in range(200):
        with torch.cuda.stream(bg):
            junk.add_(1)
        outs.append(tfhe.lwe_keyswitch(P, ext, ksk, engine="tc"))
    torch.cuda.synchronize()
    for o in outs:
        assert_u32_equal(tfhe.to_host(o), want)


@pytest.mark.parametrize("name,per_sm", [("CFG2", 4), ("CFG4", 4)])
def test_decoupled_tmem_ladders_under_contention(name, per_sm):
    """The decoupled-group TMEM ladders (mode 5 at N = 1024, the N = 2048 TMEM ladder:
    per-group key-slice release counters, mbarrier-tracked TMA slots, shuffle exchanges)
    re-run under a second stream's load, ragged batches from one CTA per SM."""
    P = dataclasses.replace(named_params(name), lwe_n=48)
    K = tfhe.pbs_keygen(P, 7)
    bsk, ksk = K.device_keys()
    rng = np.random.default_rng(8)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    cases = {B: (tfhe.to_device(_rand(rng, (B, P.lwe_n + 1))), tfhe.to_device(_rand(rng, (B, 2, P.n))))
             for B in (per_sm * sms + 3, 2 * per_sm * sms + 1)}
    want = {B: tfhe.to_host(tfhe.pbs_batch(P, l, t, bsk, ksk, ladder="ntt", engine="simt"))
            for B, (l, t) in cases.items()}
    bg = torch.cuda.Stream()
    big_l = tfhe.to_device(_rand(rng, (3 * per_sm * sms, P.lwe_n + 1)))
    big_t = tfhe.to_device(_rand(rng, (2, P.n)))
    outs = []
    for it in range(12):
        with torch.cuda.stream(bg):
            tfhe.pbs_batch(P, big_l, big_t, bsk, None, ladder="fft")
        for B, (l, t) in cases.items():
            outs.append((B, tfhe.pbs_batch(P, l, t, bsk, ksk, ladder="fft")))
    torch.cuda.synchronize()
    for B, o in outs:
        assert_u32_equal(tfhe.to_host(o), want[B])
