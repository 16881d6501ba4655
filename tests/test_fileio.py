"""HWSD files (hw/fileio.py): byte parity with the reference's own writer
(fixtures in tests/golden/hwsd/, made by make_hwsd_golden.py with the reference),
the build's reader on reference-written files, native q = 2^32 round trips and
the reference's error behaviour (bad magic/kind/version, truncation, the
insecure-parameter gate, parameter mismatch)."""

import io
import os
import struct
import sys

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2403_20190_b200 import fileio as F
from paper_2403_20190_b200 import hewnn, tfhe, wnn
from paper_2403_20190_b200.params import GadgetSpec, HeParams, named_params

sys.path.insert(0, GOLDEN)
from make_hwsd_golden import GADGET, GADGET_PKS, GEOM, PARAM_KW, hwsd_objects  # noqa: E402

FIX = os.path.join(GOLDEN, "hwsd")
P = HeParams(gadget=GadgetSpec(*GADGET), gadget_ks=GadgetSpec(8, 2), gadget_pks=GadgetSpec(*GADGET_PKS), **PARAM_KW)
PIN = HeParams(gadget=GadgetSpec(*GADGET), gadget_ks=GadgetSpec(8, 2), gadget_pks=GadgetSpec(*GADGET_PKS),
               insecure=True, **{**PARAM_KW, "name": "HWSD_TOY_INSECURE"})
GEO = wnn.WisardGeometry(**GEOM)
O = hwsd_objects()


def fixture(name):
    with open(os.path.join(FIX, name), "rb") as f:
        return f.read()


def t32(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int32))


def samples():
    out = []
    for d, lab in O["samples"]:
        stack = d if lab is None else np.concatenate([d, lab])
        out.append(hewnn.EncryptedSample.from_stack(P, stack, d.shape[0], 0 if lab is None else lab.shape[0]))
    return out


def model():
    return hewnn.HomWisardModel(GEO, P, t32(O["rams"]), t32(O["counts_ct"]))


def written(fn, *args, **kw):
    path = os.path.join(os.environ.get("PYTEST_TMP", "/tmp"), f"hwsd_{os.getpid()}.bin")
    fn(path, *args, **kw)
    with open(path, "rb") as f:
        data = f.read()
    os.unlink(path)
    return data


# ---------------------------------------------------------------------------
# byte parity with the reference writer (q64 = the reference's layout)

def test_writer_bytes_equal_reference():
    assert written(F.save_secret_key, tfhe.SecretKey(P, O["s1"]), q64=True) == fixture("secret_key.hwsd")
    assert written(F.save_secret_key, tfhe.SecretKey(PIN, O["s1"]), q64=True) == fixture("secret_key_insecure.hwsd")
    assert written(F.save_ksk, tfhe.PackingKeySwitchKey(P, O["pksk"]), q64=True) == fixture("ksk.hwsd")
    assert written(F.write_samples, samples(), P, {"source": "fixture"}, q64=True) == fixture("samples.hwsd")
    assert written(F.save_he_model, model(), {"images": 2}, q64=True) == fixture("he_model.hwsd")
    packs = [hewnn.ScorePack(GEO, P, a, b) for a, b in O["packs"]]
    assert written(F.write_scorepacks, packs, P, GEO, q64=True) == fixture("scorepacks.hwsd")
    assert written(F.save_plain_model, GEO, O["counters"], wnn.ClassCounts(O["class_counts"]),
                   {"note": "fixture"}) == fixture("plain_model.hwsd")
    assert written(F.write_manifest, {"kind": "train", "images": 2, "params": P.name}) == fixture("manifest.txt")


# ---------------------------------------------------------------------------
# the build's reader on reference-written files

def test_reader_loads_reference_files():
    sk = F.load_secret_key(os.path.join(FIX, "secret_key.hwsd"))
    assert np.array_equal(sk.s, O["s1"]) and sk.params.gadget_pks == P.gadget_pks and sk.params.lwe_n == 0
    ksk = F.load_ksk(os.path.join(FIX, "ksk.hwsd"))
    assert ksk.data.dtype == np.uint32 and np.array_equal(ksk.data, O["pksk"])
    got = list(F.read_samples(os.path.join(FIX, "samples.hwsd")))
    assert len(got) == 2
    for g, w in zip(got, samples()):
        assert (g.s, g.n_label_bits) == (w.s, w.n_label_bits) and np.array_equal(g.rgsw, w.rgsw)
    assert F.samples_meta(os.path.join(FIX, "samples.hwsd"))["source"] == "fixture"
    m = F.load_he_model(os.path.join(FIX, "he_model.hwsd"), device=False)
    assert m.geometry == GEO
    assert np.array_equal(m.rams.numpy().view(np.uint32), O["rams"])
    assert np.array_equal(m.counts_ct.numpy().view(np.uint32), O["counts_ct"])
    packs = list(F.read_scorepacks(os.path.join(FIX, "scorepacks.hwsd")))
    assert [(np.array_equal(p.packed, a), np.array_equal(p.counts_ct, b)) for p, (a, b) in zip(packs, O["packs"])] \
        == [(True, True)] * 2
    geo, counters, counts, meta = F.load_plain_model(os.path.join(FIX, "plain_model.hwsd"))
    assert geo == GEO and np.array_equal(counters, O["counters"]) and np.array_equal(counts.counts, O["class_counts"])
    assert meta["note"] == "fixture"
    assert F.read_manifest(os.path.join(FIX, "manifest.txt")) == {"kind": "train", "images": "2", "params": P.name}


def test_q64_words_need_modswitch():
    path = os.path.join(FIX, "he_model_q64.hwsd")
    with pytest.raises(F.FileFormatError, match="modswitch"):
        F.load_he_model(path, device=False)
    m = F.load_he_model(path, device=False, modswitch=True)
    x = O["q64_lowbits"]
    want = (((x >> np.uint64(31)) + np.uint64(1)) >> np.uint64(1)).astype(np.uint32)   # round(x / 2^32) mod 2^32
    assert np.array_equal(m.counts_ct.numpy().view(np.uint32), want)


# ---------------------------------------------------------------------------
# native q = 2^32 files

def test_native_round_trips(tmp_path):
    p = tmp_path / "f.hwsd"
    F.write_samples(p, samples(), P)
    assert all(np.array_equal(a.rgsw, b.rgsw) for a, b in zip(F.read_samples(p, expect_params=P), samples()))
    assert F.read_header(open(p, "rb"), "enc-samples")["params"]["q_bits"] == 32
    F.save_he_model(p, model())
    m = F.load_he_model(p, device=False, expect_params=P)
    assert torch.equal(m.rams, model().rams) and m.params == P
    Pp = named_params("INSECURE_1024")
    keys = tfhe.pbs_keygen(Pp, 3)
    F.save_pbs_keys(p, keys)
    k2 = F.load_pbs_keys(p, allow_insecure=True)
    assert k2.params == Pp
    for a, b in ((k2.lwe_key.s, keys.lwe_key.s), (k2.glwe_key.s, keys.glwe_key.s), (k2.bsk, keys.bsk),
                 (k2.ksk, keys.ksk)):
        assert np.array_equal(a, b)
    sk, pk = tfhe.keygen(P, 5)
    F.save_ksk(p, pk)
    assert np.array_equal(F.load_ksk(p).data, pk.data)
    # native files are smaller than the reference layout (u4 vs u8 words)
    assert len(written(F.save_ksk, pk)) < len(written(F.save_ksk, pk, q64=True))


# ---------------------------------------------------------------------------
# errors (hw/fileio.py:75-91, 109-117, 121-123)

def test_errors(tmp_path):
    good = fixture("he_model.hwsd")
    bad = tmp_path / "bad.hwsd"
    bad.write_bytes(b"XXXX" + good[4:])
    with pytest.raises(F.FileFormatError, match="bad magic"):
        F.load_he_model(bad, device=False)
    bad.write_bytes(good[:4] + struct.pack("<H", 2) + good[6:])
    with pytest.raises(F.FileFormatError, match="version"):
        F.load_he_model(bad, device=False)
    with pytest.raises(F.FileFormatError, match="expected a secret-key file"):
        F.load_secret_key(os.path.join(FIX, "he_model.hwsd"))
    bad.write_bytes(good[:-9])
    with pytest.raises(F.FileFormatError, match="truncated"):
        F.load_he_model(bad, device=False)
    with pytest.raises(F.InsecureParamsError):
        F.load_secret_key(os.path.join(FIX, "secret_key_insecure.hwsd"))
    assert F.load_secret_key(os.path.join(FIX, "secret_key_insecure.hwsd"), allow_insecure=True).params.insecure
    other = HeParams(**{**P.__dict__, "p": 32})
    with pytest.raises(F.FileFormatError, match="does not match"):
        list(F.read_samples(os.path.join(FIX, "samples.hwsd"), expect_params=other))
    with pytest.raises(F.FileFormatError):
        F.read_array(io.BytesIO(b"\x03<u4\x01" + struct.pack("<q", 4) + b"\0" * 8))


@pytest.mark.gpu
def test_pinned_sample_stream(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("pinned host memory needs the CUDA driver")
    p = tmp_path / "s.hwsd"
    F.write_samples(p, samples(), P)
    got = list(F.read_samples(p, pin=True))
    assert all(g.rgsw.is_pinned() for g in got)
    assert all(np.array_equal(g.rgsw.numpy().view(np.uint32), w.rgsw) for g, w in zip(got, samples()))


@pytest.mark.gpu
def test_train_from_hwsd_stream(tmp_path):
    """Storage -> pinned host -> HBM: samples written as an HWSD stream, read back into
    pinned tensors and trained on -- the model equals the reference-pinned fixture."""
    sys.path.insert(0, GOLDEN)
    from cases import TRAIN_CASES, train_inputs
    from conftest import golden
    name = sorted(TRAIN_CASES)[0]
    g = golden(f"{name}.npz")
    P, s1, bits, labels, stacks = train_inputs(name)
    s, l, a, r = TRAIN_CASES[name][2]
    lb = max(1, (l - 1).bit_length())
    smp = [hewnn.EncryptedSample.from_stack(P, st, s, lb) for st in stacks]
    path = tmp_path / "train.hwsd"
    assert F.write_samples(path, smp, P, {"case": name}) == len(smp)
    stream = F.read_samples(path, pin=True, expect_params=P)
    model = hewnn.he_train(stream, wnn.WisardGeometry(s, l, a, r, P.p), P, batch=1)
    import hashlib
    h = hashlib.sha256(np.ascontiguousarray(tfhe.to_host(model.rams)).tobytes()).hexdigest()
    assert h == str(g["sha_rams"])
