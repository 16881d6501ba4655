"""Seeded (compressed) RGSW encryption: the uniform a-halves regenerated on the GPU
from numpy's Philox4x64 stream (hwb_philox_rgsw) are bit-identical to the host
draw (rng.bytes, hw/tfhe.py:38-40, inside enc_rgsw_batch, hw/tfhe.py:246-263), and
training from the wire form (b halves + Philox states, half the PCIe bytes) gives
the same encrypted model."""

import numpy as np
import pytest
import torch

from conftest import assert_u32_equal
from paper_2403_20190_b200 import hewnn, tfhe, wnn
from paper_2403_20190_b200.params import named_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pre", [0, 1, 5, 8])
@pytest.mark.parametrize("rows", [1, 3, 37])
def test_philox_kernel_equals_rng_bytes(pre, rows):
    N = 1024
    r1, r2 = tfhe.make_rng(9), tfhe.make_rng(9)
    for r in (r1, r2):
        r.bytes(4 * pre)
        r.normal(size=2)
    want = np.frombuffer(r1.bytes(4 * rows * N), dtype="<u4").reshape(rows, N)
    st = tfhe.philox_take(r2, rows * N)
    a = tfhe.to_host(tfhe.philox_rgsw(st, rows, N, pair=False))
    assert_u32_equal(a, want)
    b = np.arange(rows * N, dtype=np.uint32).reshape(rows, N)
    full = tfhe.to_host(tfhe.philox_rgsw(st, rows, N, b_rows=tfhe.to_device(b)))
    assert_u32_equal(full[:, 0], want)
    assert_u32_equal(full[:, 1], b)
    assert np.array_equal(r1.normal(size=4), r2.normal(size=4))


def test_seeded_samples_train_identically():
    P = named_params("CFG3", 256)
    geom = wnn.WisardGeometry(40, 3, 8, 7, 256)
    key = tfhe.SecretKey(P, tfhe.make_rng(5).integers(0, 2, P.n).astype(np.uint32))
    rng = np.random.default_rng(6)
    bits, labels = rng.integers(0, 2, (7, 40)), rng.integers(0, 3, 7)
    host = [tfhe.enc_rgsw_batch(bits[0], key, tfhe.make_rng(77))]       # host path for one sample
    r_plain, r_seed = tfhe.make_rng(8), tfhe.make_rng(8)
    plain = [hewnn.encrypt_sample(bits[i], int(labels[i]), key, r_plain, label_bits=geom.label_bits)
             for i in range(7)]
    seeded = [hewnn.encrypt_sample_seeded(bits[i], int(labels[i]), key, r_seed, label_bits=geom.label_bits)
              for i in range(7)]
    for x, y in zip(plain, seeded):
        assert_u32_equal(tfhe.to_host(y.rgsw.expand()), tfhe.to_host(x.rgsw))
        assert y.rgsw.b.is_pinned()
    assert_u32_equal(tfhe.to_host(hewnn.encrypt_sample(bits[0], None, key, tfhe.make_rng(77)).rgsw),
                     np.stack([c.data for c in host[0]]))
    m1 = hewnn.he_train(plain, geom, P, batch=3)
    m2 = hewnn.he_train(seeded, geom, P, batch=3)              # staged: b over PCIe, a regenerated
    assert torch.equal(m1.rams, m2.rams) and torch.equal(m1.counts_ct, m2.counts_ct)
    m3 = hewnn.he_train(seeded, geom, P, batch=1)              # every staging slot reused
    assert torch.equal(m1.rams, m3.rams)
    assert hewnn.decrypt_sample(seeded[2], key) == (list(bits[2]), int(labels[2]))


def test_seeded_full_size_sample_expands_exactly():
    """A BASELINE cfg3-size sample (2352 data bits + 4 label bits, 14,136 rows): the
    gadget-carrying a-words and the regenerated words never race."""
    P = named_params("CFG3", 256)
    key = tfhe.SecretKey(P, tfhe.make_rng(15).integers(0, 2, P.n).astype(np.uint32))
    bits = np.random.default_rng(16).integers(0, 2, 2352)
    plain = hewnn.encrypt_sample(bits, 9, key, tfhe.make_rng(17), label_bits=4)
    seeded = hewnn.encrypt_sample_seeded(bits, 9, key, tfhe.make_rng(17), label_bits=4)
    for _ in range(3):
        assert_u32_equal(tfhe.to_host(seeded.rgsw.expand()), tfhe.to_host(plain.rgsw))
