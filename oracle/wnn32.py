"""CPU oracle for encrypted WiSARD training at q = 2^32 -- TEST INFRASTRUCTURE.

Restates, with `hw/` cites into /root/reference/pkg/src/hewisard:
* the plaintext integer WiSARD (`hw/wnn.py:189-238`): permutation, addresses,
  train_integer -- the oracle for decrypted counters;
* inverse vertical packing (`hw/lut.py:269-314`) and encrypted training
  (`hw/hewnn.py:134-229`) over exact external products from the C oracle
  (oracle/c), the oracle for ciphertext-level parity.
Pinned against reference-generated fixtures (tests/golden/train_*.npz).
"""

from __future__ import annotations

import numpy as np

from . import coracle
from . import tfhe32 as o

CLEAR0, CLEAR1 = -1, -2


def permutation(r: int, s: int) -> np.ndarray:
    """hw/wnn.py:189-196: Fisher-Yates on the recorded Philox stream."""
    rng = o.make_rng(r)
    perm = np.arange(s)
    for i in range(s - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    return perm


def k0(s, a):
    return -(-s // a)


def label_bits(l):
    return max(1, (l - 1).bit_length())


def addresses(bits: np.ndarray, s: int, a: int, r: int) -> np.ndarray:
    """hw/wnn.py:209-219."""
    bits = np.atleast_2d(bits)
    perm = permutation(r, s)
    px = bits[:, perm]
    pad = k0(s, a) * a - s
    if pad:
        px = np.hstack([px, np.zeros((len(px), pad), dtype=bits.dtype)])
    px = px.reshape(len(px), k0(s, a), a).astype(np.int64)
    return px @ (1 << np.arange(a, dtype=np.int64))


def train_integer(bits: np.ndarray, labels: np.ndarray, s, l, a, r, p):
    """hw/wnn.py:222-238: counters (l, k0, 2^a) mod p and class counts."""
    labels = np.asarray(labels, dtype=np.int64)
    counters = np.zeros((l, k0(s, a), 1 << a), dtype=np.int64)
    counts = np.zeros(l, dtype=np.int64)
    if labels.size == 0:
        return counters, counts
    addr = addresses(bits, s, a, r)
    rams = np.broadcast_to(np.arange(k0(s, a)), addr.shape)
    lab = np.broadcast_to(labels[:, None], addr.shape)
    np.add.at(counters, (lab, rams, addr), 1)
    counters &= p - 1
    counts += np.bincount(labels, minlength=l)
    return counters, counts


def tree_depth(k, degree_log):
    return max(0, k - degree_log)


def selector_codes(s, l, a, r, degree_log, clear_label=None):
    """hw/hewnn.py:134-173: (k0, k) codes (row of the sample's RGSW stack, or clear)."""
    lb = label_bits(l)
    k = lb + a
    z = tree_depth(k, degree_log)
    perm = permutation(r, s)
    weights = [k - 1 - i for i in range(z)] + list(range(min(k, degree_log)))
    out = np.empty((k0(s, a), k), dtype=np.int64)
    for j in range(k0(s, a)):
        for pos, w in enumerate(weights):
            if w < a:
                idx = j * a + w
                out[j, pos] = perm[idx] if idx < s else CLEAR0
            elif clear_label is None:
                out[j, pos] = s + (w - a)
            else:
                out[j, pos] = CLEAR1 if (clear_label >> (w - a)) & 1 else CLEAR0
    return out


def ivp_batch(codes: np.ndarray, table: np.ndarray, payload: np.ndarray, levels: int, base_log: int,
              degree_log: int) -> np.ndarray:
    """hw/lut.py:269-314 on code matrices; table (R, 2l, 2, N) coefficient GGSWs."""
    B, k = codes.shape
    z = tree_depth(k, degree_log)
    n = payload.shape[-1]
    acc = np.broadcast_to(payload, (B, 2, n)).copy()
    clear_e = np.zeros(B, dtype=np.int64)
    for i, w in enumerate(range(min(k, degree_log))):
        col = codes[:, z + i]
        enc = np.nonzero(col >= 0)[0]
        clear_e += (col == CLEAR1).astype(np.int64) << w
        if enc.size:
            rotated = o.monomial_mul(acc, 1 << w)                           # hw/lut.py:289
            diff = (rotated[enc] - acc[enc]).astype(np.uint32)
            acc[enc] = acc[enc] + coracle.ext_product_batch(table[col[enc]], diff, levels, base_log)
    acc = o.monomial_gather(acc, clear_e)                                   # hw/lut.py:292
    cur = acc[:, None]
    for pos in range(z - 1, -1, -1):                                        # hw/lut.py:295-313
        col = codes[:, pos]
        m = cur.shape[1]
        new = np.zeros((B, 2 * m, 2, n), dtype=np.uint32)
        c0 = np.nonzero(col == CLEAR0)[0]
        c1 = np.nonzero(col == CLEAR1)[0]
        enc = np.nonzero(col >= 0)[0]
        new[c0, :m] = cur[c0]
        new[c1, m:] = cur[c1]
        if enc.size:
            sub = cur[enc].reshape(-1, 2, n)
            reps = np.repeat(table[col[enc]], m, axis=0)
            hi = coracle.ext_product_batch(reps, sub, levels, base_log).reshape(len(enc), m, 2, n)
            new[enc, m:] = hi
            new[enc, :m] = cur[enc] - hi
        cur = new
    return cur


def vp_batch(codes: np.ndarray, table: np.ndarray, luts: np.ndarray, levels: int, base_log: int,
             degree_log: int) -> np.ndarray:
    """hw/lut.py:209-266 on code matrices: luts (B, 2^z, 2, N); returns (B, N+1)."""
    B, k = codes.shape
    z = tree_depth(k, degree_log)
    n = luts.shape[-1]
    start = np.zeros(B, dtype=np.int64)
    length = np.full(B, max(1, 1 << z), dtype=np.int64)
    lvl = 0
    while lvl < z and (codes[:, lvl] < 0).all():                            # hw/lut.py:225-230
        length //= 2
        start += np.where(codes[:, lvl] == CLEAR1, length, 0)
        lvl += 1
    cur = np.stack([luts[i][start[i]: start[i] + length[i]] for i in range(B)])
    for pos in range(lvl, z):                                               # hw/lut.py:233-247
        col = codes[:, pos]
        half = cur.shape[1] // 2
        new = np.empty((B, half, 2, n), dtype=np.uint32)
        c0 = np.nonzero(col == CLEAR0)[0]
        c1 = np.nonzero(col == CLEAR1)[0]
        enc = np.nonzero(col >= 0)[0]
        new[c0] = cur[c0][:, :half]
        new[c1] = cur[c1][:, half:]
        if enc.size:
            lo, hi = cur[enc][:, :half], cur[enc][:, half:]
            reps = np.repeat(table[col[enc]], half, axis=0)
            ext = coracle.ext_product_batch(reps, (hi - lo).reshape(-1, 2, n), levels, base_log)
            new[enc] = lo + ext.reshape(len(enc), half, 2, n)
        cur = new
    acc = np.ascontiguousarray(cur[:, 0])
    clear_e = np.zeros(B, dtype=np.int64)
    for i, w in enumerate(range(min(k, degree_log))):                       # hw/lut.py:251-260
        col = codes[:, z + i]
        enc = np.nonzero(col >= 0)[0]
        clear_e += (col == CLEAR1).astype(np.int64) << w
        if enc.size:
            rotated = o.monomial_mul(acc, -(1 << w))
            diff = (rotated[enc] - acc[enc]).astype(np.uint32)
            acc[enc] = acc[enc] + coracle.ext_product_batch(table[col[enc]], diff, levels, base_log)
    acc = o.monomial_gather(acc, -clear_e)
    return o.extract_lwe_batch(acc)                                         # hw/lut.py:263-266


def he_train(stacks: list[np.ndarray], s, l, a, r, params) -> tuple[np.ndarray, np.ndarray]:
    """hw/hewnn.py:189-229: stacks[i] = (s + label_bits, 2l, 2, N) RGSW rows of
    sample i (data bits then label bits LSB-first).  Returns (rams, counts_ct)."""
    g = params.gadget
    n = params.n
    lb = label_bits(l)
    codes = selector_codes(s, l, a, r, params.degree_log)
    k1 = max(1, (1 << (lb + a)) // n)
    rams = np.zeros((k0(s, a), k1, 2, n), dtype=np.uint32)
    counts = np.zeros((2, n), dtype=np.uint32)
    payload = o.trivial_rlwe(1, params.p, n)                                # hw/hewnn.py:203
    for st in stacks:
        rows = ivp_batch(codes, st, payload, g.levels, g.base_log, params.degree_log)
        rams += rows                                                        # hw/hewnn.py:213
        lab = ivp_batch(np.arange(s, s + lb)[None], st, payload, g.levels, g.base_log, params.degree_log)
        counts += lab[0, 0]                                                 # hw/hewnn.py:180-186
    return rams, counts


def decrypt_model(rams: np.ndarray, counts_ct: np.ndarray, s1: np.ndarray, s, l, a, p):
    """hw/hewnn.py:352-365: counters (l, k0, 2^a) and class counts."""
    phase = (rams[:, :, 1] - o.key_mul(rams[:, :, 0], s1)).astype(np.uint32)
    vals = o.decode_phase(phase, p).reshape(rams.shape[0], -1)[:, : 1 << (label_bits(l) + a)]
    counters = np.zeros((l, rams.shape[0], 1 << a), dtype=np.int64)
    for c in range(l):
        counters[c] = vals[:, c << a: (c << a) + (1 << a)]
    counts = o.decode_phase(o.phase_rlwe(counts_ct, s1), p)[:l]
    return counters, counts
