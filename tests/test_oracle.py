"""Pin the CPU oracle (oracle/tfhe32.py, oracle/c) against fixtures produced by the
REFERENCE on 2^32-embedded operands (tests/golden/make_golden.py), and against
the reference test suite's own known answers restated at q = 2^32."""

import dataclasses
import hashlib

import numpy as np
import pytest

from conftest import assert_u32_equal, golden
from oracle import tfhe32 as o
from paper_2403_20190_b200.params import GadgetSpec, named_params

GADGETS = [(3, 7), (2, 8), (2, 10), (8, 2), (7, 2), (2, 16), (1, 23), (4, 8)]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------- decomposition

@pytest.mark.parametrize("lv,w", GADGETS)
def test_decompose_matches_reference(lv, w):
    g = golden("decompose.npz")
    d = o.gadget_decompose(g[f"x_{lv}_{w}"], lv, w)
    assert np.array_equal(d, g[f"d_{lv}_{w}"])


@pytest.mark.parametrize("lv,w", GADGETS)
def test_decompose_closed_form_used_by_gpu(lv, w):
    """The kernels' closed form ((v >> w(l-1-t)) & mask) - beta/2 equals the
    reference's LSB-first carry loop (hw/ring.py:144-150)."""
    g = golden("decompose.npz")
    x = g[f"x_{lv}_{w}"].astype(np.uint64)
    tot = lv * w
    u = (((x + (1 << (31 - tot))) & 0xFFFFFFFF) >> (32 - tot)) if tot < 32 else x
    half = 1 << (w - 1)
    v = (u + sum(half << (w * k) for k in range(lv))) & 0xFFFFFFFF
    for t in range(lv):
        dt = ((v >> (w * (lv - 1 - t))) & ((1 << w) - 1)).astype(np.int64) - half
        assert np.array_equal(dt, g[f"d_{lv}_{w}"][t])


def test_decompose_zero_and_centred():
    # pkg/tests/test_ring.py:111-130 at q = 2^32
    assert not o.gadget_decompose(np.zeros(8, np.uint32), 2, 8).any()
    rng = np.random.default_rng(6)
    x = rng.integers(0, 1 << 32, 4096, dtype=np.uint64).astype(np.uint32)
    d = o.gadget_decompose(x, 3, 7)
    assert d.min() >= -64 and d.max() < 64


@pytest.mark.parametrize("lv,w", [(3, 7), (2, 8), (2, 16)])
def test_recompose_matches_rounded_input(lv, w):
    # pkg/tests/test_ring.py:145-152 at q = 2^32
    rng = np.random.default_rng(8)
    x = rng.integers(0, 1 << 32, 4096, dtype=np.uint64)
    rec = o.gadget_recompose(o.gadget_decompose(x.astype(np.uint32), lv, w), lv, w)
    step = 1 << (32 - lv * w)
    rounded = (((x + step // 2) // step) * step) & 0xFFFFFFFF
    assert np.array_equal(rec.astype(np.uint64), rounded)


def test_exact_power_recomposes():
    # pkg/tests/test_ring.py:117-122: q/beta recomposes exactly
    g = GadgetSpec(3, 7)
    x = np.full(8, g.power(0), np.uint32)
    assert_u32_equal(o.gadget_recompose(o.gadget_decompose(x, 3, 7), 3, 7), x)


# ---------------------------------------------------------------- ring products

@pytest.mark.parametrize("N", [8, 1024, 2048])
def test_negacyclic_matches_reference(N):
    g = golden("negacyclic.npz")
    for i in range(2):
        assert_u32_equal(o.negacyclic_mul(g[f"a_{N}"][i], g[f"b_{N}"][i]), g[f"c_{N}"][i])


def test_negacyclic_wrap_known_answer():
    # pkg/tests/test_ring.py:52-58: X * X^(N-1) = -1
    n = 8
    x = np.zeros(n, np.uint32); x[1] = 1
    y = np.zeros(n, np.uint32); y[n - 1] = 1
    expect = np.zeros(n, np.uint32); expect[0] = 0xFFFFFFFF
    assert_u32_equal(o.negacyclic_mul(x, y), expect)


def test_monomial_matches_product_and_inverts():
    # pkg/tests/test_ring.py:75-108
    rng = np.random.default_rng(5)
    v = rng.integers(0, 1 << 32, 16, dtype=np.uint64).astype(np.uint32)
    for e in (1, 7, 15, 16, 31, -3):
        mono = np.zeros(16, np.uint32)
        mono[e % 16] = 1 if (e % 32) < 16 else 0xFFFFFFFF
        assert_u32_equal(o.monomial_mul(v, e), o.negacyclic_mul(v, mono))
        assert_u32_equal(o.monomial_mul(o.monomial_mul(v, e), -e), v)


def test_key_mul_matches_schoolbook():
    rng = np.random.default_rng(9)
    s = rng.integers(0, 2, 1024).astype(np.uint32)
    a = rng.integers(0, 1 << 32, (4, 1024), dtype=np.uint64).astype(np.uint32)
    km = o.key_mul(a, s)
    for i in range(4):
        assert_u32_equal(km[i], o.negacyclic_mul(a[i], s))


# ---------------------------------------------------------------- external product

@pytest.mark.parametrize("tag,lv,w", [("cfg2", 3, 7), ("cfg1", 2, 8), ("cfg4", 2, 10), ("ins", 2, 16)])
def test_ext_product_matches_reference(tag, lv, w, coracle):
    g = golden("ext_product.npz")
    G, cts = g[f"{tag}_G"], g[f"{tag}_cts"]
    if tag in ("cfg2", "cfg1"):
        assert_u32_equal(o.ext_product_batch(G, cts, lv, w), g[f"{tag}_out"])
    assert_u32_equal(coracle.ext_product_batch(G, cts, lv, w), g[f"{tag}_out"])
    assert_u32_equal(coracle.ext_product_batch(G[:1], cts, lv, w), g[f"{tag}_out_bcast"])


@pytest.mark.parametrize("tag,lv,w", [("cfg2", 3, 7), ("cfg4", 2, 10)])
def test_blind_rotate_and_extract_match_reference(tag, lv, w, coracle):
    g = golden("blind_rotate.npz")
    c, C, I = g[f"{tag}_c"], g[f"{tag}_C"], g[f"{tag}_I"]
    out = coracle.blind_rotate_batch(c[None], C, I[None].astype(np.int32), lv, w)[0]
    assert_u32_equal(out, g[f"{tag}_out"])
    if tag == "cfg2":
        assert_u32_equal(o.blind_rotate(c, list(C), list(I), lv, w), g[f"{tag}_out"])
    a, b = o.extract_lwe(out, 0)
    assert_u32_equal(a, g[f"{tag}_ext_a"])
    assert b == int(g[f"{tag}_ext_b"][0])
    assert_u32_equal(o.extract_lwe_batch(out[None])[0], np.concatenate([a, [b]]))


# ---------------------------------------------------------------- PBS

@pytest.mark.parametrize("name", ["CFG1", "CFG2", "CFG4"])
def test_keygen_pinned(name):
    P = named_params(name)
    g = golden(f"pbs_{name.lower()}.npz")
    K = o.pbs_keygen(P, int(g["key_seed"]))
    assert sha(K["s0"]) == str(g["sha_s0"])
    assert sha(K["s1"]) == str(g["sha_s1"])
    assert sha(K["bsk"]) == str(g["sha_bsk"])
    assert sha(K["ksk"]) == str(g["sha_ksk"])


@pytest.mark.parametrize("name", ["CFG1", "CFG2", "CFG4"])
def test_pbs_matches_reference_composition(name, coracle):
    P = named_params(name)
    g = golden(f"pbs_{name.lower()}.npz")
    K = o.pbs_keygen(P, int(g["key_seed"]))
    rng = o.make_rng(int(g["enc_seed"]))
    ms = rng.integers(0, P.p, len(g["ms"]))
    lwe = o.enc_lwe_batch(ms * P.delta, K["s0"], P.lwe_sigma, rng)
    assert_u32_equal(lwe, g["lwe_in"])
    tv = o.test_polynomial(np.arange(P.p // 2) % P.p, P.p, P.n)
    assert_u32_equal(tv, g["tv"])
    ext = coracle.pbs(lwe, tv, K["bsk"], None, P, keyswitch=False)
    assert_u32_equal(ext, g["extracted"])
    out = coracle.pbs(lwe, tv, K["bsk"], K["ksk"], P)
    assert_u32_equal(out, g["lwe_out"])
    if name == "CFG1":
        assert_u32_equal(o.pbs(lwe, tv, K["bsk"], K["ksk"], P), g["lwe_out"])
    # decrypt: identity on [0, p/2), negacyclic -f(m - p/2) above.  Only
    # meaningful when a message box (2N/p phase units) exceeds the mod-switch
    # noise; cfg4's p = 4096 (its counter modulus) leaves a box of 1 unit.
    if 2 * P.n // P.p < 64:
        return
    dec = o.dec_lwe(out, K["s0"], P.p)
    half = P.p // 2
    expect = np.where(ms < half, ms, (-(ms - half)) % P.p)
    assert np.array_equal(dec, expect)


def test_keyswitch_c_matches_python(coracle):
    P = dataclasses.replace(named_params("CFG2"), lwe_n=40)
    K = o.pbs_keygen(P, 3)
    rng = np.random.default_rng(4)
    lwe = rng.integers(0, 1 << 32, (5, P.n + 1), dtype=np.uint64).astype(np.uint32)
    gk = P.gadget_ks
    assert_u32_equal(coracle.keyswitch(lwe, K["ksk"], gk.levels, gk.base_log),
                     o.lwe_keyswitch(lwe, K["ksk"], gk.levels, gk.base_log))


def test_keyswitch_preserves_phase():
    P = dataclasses.replace(named_params("CFG2"), lwe_n=64)
    K = o.pbs_keygen(P, 5)
    rng = o.make_rng(6)
    ms = np.arange(8)
    lwe = o.enc_lwe_batch(ms * P.delta, K["s1"], 0.0, rng)      # under s1, dimension N
    gk = P.gadget_ks
    out = o.lwe_keyswitch(lwe, K["ksk"], gk.levels, gk.base_log)
    assert np.array_equal(o.dec_lwe(out, K["s0"], P.p), ms)


def test_mod_switch_rounding():
    N = 1024
    x = np.array([0, (1 << 20) - 1, 1 << 20, 0xFFFFFFFF, 1 << 31], np.uint32)
    assert list(o.mod_switch(x, N)) == [0, 0, 1, 0, 1024]
