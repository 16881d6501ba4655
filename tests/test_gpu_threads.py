"""The C ABI is re-entrant (SURVEY §8(b) threading contract): two host threads,
each on its own CUDA stream with its own THREAD-LOCAL kernel selection, run PBS
batches concurrently and get bit-identical results to a sequential run."""

import threading

import numpy as np
import pytest
import torch

from conftest import assert_u32_equal
from paper_2403_20190_b200 import _lib, tfhe
from paper_2403_20190_b200.params import named_params

pytestmark = pytest.mark.gpu


def test_two_threads_two_streams_bit_exact():
    P = named_params("CFG2")
    K = tfhe.pbs_keygen(P, 301)
    bsk, ksk = K.device_keys()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rng = np.random.default_rng(302)
    batches = [rng.integers(0, 1 << 32, (B, P.lwe_n + 1), dtype=np.uint64).astype(np.uint32)
               for B in (8 * sms + 3, 4 * sms + 1)]
    tv = tfhe.test_polynomial(np.arange(4), P)
    want = [tfhe.to_host(tfhe.pbs_batch(P, b, tv, bsk, ksk)) for b in batches]
    torch.cuda.synchronize()
    results = [[None] * 3 for _ in batches]
    errors = []
    start = threading.Barrier(2)

    def worker(i):
        try:
            torch.cuda.set_device(0)
            L = _lib.load()
            if i == 1:                               # thread-local: must not leak into thread 0
                _lib.check(L.hwb_set_fft_mode(0))
                _lib.check(L.hwb_set_fft_segment(7))
                L.hwb_set_fft_latency_batch(12345)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                lwe = tfhe.to_device(batches[i])
                start.wait()
                for k in range(3):
                    results[i][k] = tfhe.pbs_batch(P, lwe, tv, bsk, ksk)
                s.synchronize()
        except Exception as e:                       # surfaced below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i in range(2):
        for k in range(3):
            assert_u32_equal(tfhe.to_host(results[i][k]), want[i])
    # the main thread's settings were never touched by worker 1
    L = _lib.load()
    before = L.hwb_set_fft_latency_batch(-2)         # < -1 only queries
    assert before != 12345
