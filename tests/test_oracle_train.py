"""Pin the training oracle (oracle/wnn32.py) to the reference's he_train run on
embedded q = 2^32 inputs (tests/golden/train_*.npz), and check the product's
host-side selector logic against it.  CPU only."""

import hashlib
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, assert_u32_equal, golden
from oracle import wnn32
from paper_2403_20190_b200 import hewnn, wnn
from paper_2403_20190_b200.params import named_params

sys.path.insert(0, GOLDEN)
from cases import TRAIN_CASES, train_inputs  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module", params=sorted(TRAIN_CASES))
def case(request):
    name = request.param
    return name, train_inputs(name), golden(f"{name}.npz")


def test_inputs_pinned(case):
    name, (P, s1, bits, labels, stacks), g = case
    assert sha(*stacks) == str(g["sha_stacks"])
    assert np.array_equal(bits, g["bits"]) and np.array_equal(labels, g["labels"])


def test_oracle_he_train_matches_reference(case, coracle):
    name, (P, s1, bits, labels, stacks), g = case
    s, l, a, r = TRAIN_CASES[name][2]
    rams, counts = wnn32.he_train(stacks, s, l, a, r, P)
    assert sha(rams) == str(g["sha_rams"])
    assert_u32_equal(rams[:, :2], g["rams_head"])
    assert_u32_equal(counts, g["counts_ct"])
    counters, cc = wnn32.decrypt_model(rams, counts, s1, s, l, a, P.p)
    assert np.array_equal(counters, g["counters"])
    assert np.array_equal(cc, g["class_counts"])


def test_train_integer_matches_reference(case):
    name, (P, s1, bits, labels, stacks), g = case
    s, l, a, r = TRAIN_CASES[name][2]
    counters, counts = wnn32.train_integer(bits, labels, s, l, a, r, P.p)
    assert np.array_equal(counters, g["counters"])
    assert np.array_equal(counts, g["class_counts"])


@pytest.mark.parametrize("geom", [(120, 2, 4, 7, 16), (50, 10, 12, 7, 256), (2352, 10, 12, 7, 256),
                                  (4704, 7, 14, 7, 1024), (2352, 10, 16, 7, 4096)])
def test_selector_template_matches_oracle(geom):
    s, l, a, r, p = geom
    P = named_params("CFG4" if a == 16 else "CFG2", p)
    G = wnn.WisardGeometry(s, l, a, r, p)
    assert np.array_equal(hewnn._selector_template(G, P), wnn32.selector_codes(s, l, a, r, P.degree_log))
    assert np.array_equal(wnn.permutation(r, s), wnn32.permutation(r, s))
    for lab in (0, l - 1):
        assert np.array_equal(hewnn._selector_template(G, P, clear_label=lab),
                              wnn32.selector_codes(s, l, a, r, P.degree_log, clear_label=lab))


def test_host_rgsw_encryption_matches_oracle():
    name = "train_cfg1"
    P, s1, bits, labels, stacks = train_inputs(name)
    from paper_2403_20190_b200 import tfhe
    key = tfhe.SecretKey(P, s1)
    pname, p, (s, l, a, r), count, kseed, eseed, dseed = TRAIN_CASES[name]
    rng = tfhe.make_rng(eseed)
    for i in range(count):
        smp = hewnn.encrypt_sample(bits[i], int(labels[i]), key, rng, label_bits=1, device=False)
        assert_u32_equal(smp.rgsw, stacks[i])


def test_packing_keygen_and_pack_batch_match_reference(coracle):
    from oracle import tfhe32 as o
    from paper_2403_20190_b200 import tfhe
    g = golden("infer_tree.npz")
    P = named_params("CFG2", 256)
    kseed = TRAIN_CASES["train_tree"][4]
    s, ksk = o.keygen_packing(P, kseed)
    assert sha(ksk) == str(g["sha_ksk"])
    key, pk = tfhe.keygen(P, kseed)                    # product restatement of hw/tfhe.py:95-114
    assert_u32_equal(key.s, s)
    assert_u32_equal(pk.data, ksk)
    gp = P.gadget_pks
    assert_u32_equal(coracle.pack_batch(g["pack_a"], g["pack_b"], ksk, gp.levels, gp.base_log), g["pack_out"])
