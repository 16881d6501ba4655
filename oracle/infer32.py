"""CPU restatement of the OTF-act inference pipeline -- TEST INFRASTRUCTURE.

Checker for `paper_2403_20190_b200/infer_pbs.py` (bleaching threshold, popcount,
argmax on ciphertexts).  Every bootstrap runs on the exact C oracle
(`coracle.pbs`, the schoolbook restatement of hw/tfhe.py:340-361 with the NEW
mod switch / test polynomial), every affine step in numpy uint32 (exact mod 2^32).
Written without the product's code: the same algorithm, restated from DESIGN.md
§6d, so a bit-for-bit match of the encrypted class indices checks both.

Plaintext semantics it must reproduce (hw/wnn.py:86-109, 296-309): per class c,
score_c = #{j : counter_{c,j} > thr}; prediction = np.argmax(scores).
"""

from __future__ import annotations

import numpy as np

from oracle import coracle, tfhe32 as o

U32 = np.uint32
OUT_LOG = 28
OUT = 1 << OUT_LOG


def _u(x) -> np.ndarray:
    return np.asarray(x, dtype=np.int64).astype(np.int64)


def affine(x, y=None, cx=1, cy=1, cb=0, shift=0) -> np.ndarray:
    """((cx x + cy y) << shift) + cb (body only), mod 2^32, rows (M, W)."""
    x = np.asarray(x, dtype=np.uint64)
    M = x.shape[0]
    cx = np.broadcast_to(_u(cx), (M,)).astype(np.uint64)[:, None] & np.uint64(0xFFFFFFFF)
    v = x * cx
    if y is not None:
        cy = np.broadcast_to(_u(cy), (M,)).astype(np.uint64)[:, None] & np.uint64(0xFFFFFFFF)
        v = v + np.asarray(y, dtype=np.uint64) * cy
    v = (v << np.uint64(shift)) & np.uint64(0xFFFFFFFF)
    v[:, -1] = (v[:, -1] + (np.broadcast_to(_u(cb), (M,)).astype(np.uint64) & np.uint64(0xFFFFFFFF))) \
        & np.uint64(0xFFFFFFFF)
    return v.astype(U32)


def trivial(value, M, N) -> np.ndarray:
    t = np.zeros((M, N + 1), dtype=U32)
    t[:, N] = U32(int(value) & 0xFFFFFFFF)
    return t


def lut_sign(v, N) -> np.ndarray:
    tv = np.zeros((2, N), dtype=U32)
    tv[1] = U32(v & 0xFFFFFFFF)
    return tv


def lut_half(f, p, v, N) -> np.ndarray:
    return o.test_polynomial(np.asarray(f), p, N, delta_out=v)


class Boot:
    """Bootstraps on the C oracle under the self-bootstrapping key (n = N, no KS)."""

    def __init__(self, params, bsk):
        self.P = params
        self.bsk = bsk
        self.count = 0

    def __call__(self, lwe, tvs):
        lwe = np.ascontiguousarray(lwe, dtype=U32)
        tvs = np.ascontiguousarray(np.broadcast_to(tvs, (lwe.shape[0],) + np.shape(tvs)[-2:]), dtype=U32)
        self.count += lwe.shape[0]
        return coracle.pbs(lwe, tvs, self.bsk, None, self.P, keyswitch=False)


def bleach(boot: Boot, lwe, p, thr):
    M, W = lwe.shape
    N = W - 1
    K = p.bit_length() - 1
    t = thr + 1
    if t <= 0:
        return trivial(OUT, M, N)
    if t >= p:
        return trivial(0, M, N)
    c = p - t
    C, carry = lwe, None
    for i in range(K // 2):
        s = 32 - K + 2 * i
        top = i == K // 2 - 1 and K % 2 == 0
        L = affine(C, shift=30 - s, cb=1 << 29)
        b_cmp = boot(L, lut_sign(OUT, N))
        if s < OUT_LOG:
            C1 = affine(C, boot(L, lut_sign(1 << s, N)), cb=-(1 << s))
        else:
            C1 = affine(C, b_cmp, cy=1 << (s - OUT_LOG), cb=-(1 << s))
        Lh = affine(C1, shift=30 - s)
        lo_cmp = boot(Lh, lut_half([0, 1], 4, OUT, N))
        if not top:
            if s < OUT_LOG:
                C = affine(C1, boot(Lh, lut_half([0, 1], 4, 1 << s, N)), cy=-1)
            else:
                C = affine(C1, lo_cmp, cy=-(1 << (s - OUT_LOG)))
        y = affine(lo_cmp, b_cmp, cy=-1, cb=OUT + ((c >> (2 * i)) & 3) * OUT)
        if carry is not None:
            y = affine(y, carry)
        carry = boot(y, lut_half([int(v >= 4) for v in range(8)], 16, OUT, N))
    if K % 2:                                   # odd K: a single top bit at 2^31
        sg = boot(affine(C, cb=1 << 30), lut_sign(OUT >> 1, N))
        y = affine(sg, cx=-1, cb=(OUT >> 1) + ((c >> (K - 1)) & 1) * OUT)
        if carry is not None:
            y = affine(y, carry)
        carry = boot(y, lut_half([int(v >= 2) for v in range(8)], 16, OUT, N))
    return carry


def _add(boot, A, B, max_digits):
    D = max(len(A), len(B))
    M, W = (A or B)[0].shape
    zero = np.zeros((M, W), dtype=U32)
    out, carry = [], None
    for i in range(D):
        s = affine(A[i] if i < len(A) else zero, B[i] if i < len(B) else zero)
        if carry is not None:
            s = affine(s, carry)
        out.append(boot(s, lut_half([v % 4 for v in range(8)], 16, OUT, W - 1)))
        carry = None if (i == D - 1 and D >= max_digits) else boot(s, lut_half([v // 4 for v in range(8)], 16, OUT,
                                                                                W - 1))
    if carry is not None:
        out.append(carry)
    return out


def popcount(boot, bits, max_value):
    """bits (M, k, W) -> radix-4 digits (M, W) each."""
    M, k, W = bits.shape
    max_digits = max(1, int(np.ceil(np.log(max_value + 1) / np.log(4))))
    G = -(-k // 7)
    padded = np.zeros((M, G * 7, W), dtype=U32)
    padded[:, :k] = bits
    g = padded.reshape(M * G, 7, W)
    v = g[:, 0]
    for j in range(1, 7):
        v = affine(v, g[:, j])
    nums = [boot(v, lut_half([x % 4 for x in range(8)], 16, OUT, W - 1)).reshape(M, G, W)]
    if max_digits >= 2:
        nums.append(boot(v, lut_half([x // 4 for x in range(8)], 16, OUT, W - 1)).reshape(M, G, W))
    count = G
    while count > 1:
        half = count // 2
        S = _add(boot, [d[:, 0:2 * half:2].reshape(M * half, W) for d in nums],
                 [d[:, 1:2 * half:2].reshape(M * half, W) for d in nums], max_digits)
        S = [d.reshape(M, half, W) for d in S]
        if count % 2:
            tail = [d[:, count - 1:count] for d in nums]
            tail += [np.zeros((M, 1, W), dtype=U32)] * (len(S) - len(tail))
            S = [np.concatenate([a, b], axis=1) for a, b in zip(S, tail)]
        nums, count = S, half + count % 2
    return [d[:, 0] for d in nums]


def argmax(boot, scores, l):
    SL, W = scores[0].shape
    S = SL // l
    N = W - 1
    nd = max(1, int(np.ceil(np.log(l) / np.log(4))))
    cand = [d.reshape(S, l, W) for d in scores]
    idx = [np.stack([trivial(((c >> (2 * k)) & 3) * OUT, S, N) for c in range(l)], axis=1) for k in range(nd)]
    count = l
    while count > 1:
        half = count // 2

        def pairs(ds, off):
            return [d[:, off:2 * half:2].reshape(S * half, W) for d in ds]
        A, B, IA, IB = pairs(cand, 0), pairs(cand, 1), pairs(idx, 0), pairs(idx, 1)
        r = None
        for i in range(len(A)):
            c2 = boot(affine(B[i], A[i], cy=-1, cb=3 * OUT), lut_half([0, 0, 0, 2, 4, 4, 4, 0], 16, OUT, N))
            r = boot(c2 if r is None else affine(c2, r), lut_half([int(y >= 3) for y in range(8)], 16, OUT, N))
        sel_a = lut_half([x if x < 4 else 0 for x in range(8)], 16, OUT, N)
        sel_b = lut_half([x - 4 if x >= 4 else 0 for x in range(8)], 16, OUT, N)
        pick = [affine(boot(affine(a, r, cy=4), sel_a), boot(affine(b, r, cy=4), sel_b))
                for a, b in zip(A + IA, B + IB)]
        win = [d.reshape(S, half, W) for d in pick[:len(A)]]
        wix = [d.reshape(S, half, W) for d in pick[len(A):]]
        if count % 2:
            win = [np.concatenate([w, d[:, count - 1:count]], axis=1) for w, d in zip(win, cand)]
            wix = [np.concatenate([w, d[:, count - 1:count]], axis=1) for w, d in zip(wix, idx)]
        cand, idx, count = win, wix, half + count % 2
    return [d[:, 0] for d in idx]


def infer(boot: Boot, lookups: np.ndarray, S: int, l: int, k0: int, p: int, thr: int):
    """lookups (S*l*k0, N+1) VP outputs -> index digits (S, D, N+1) and score digits."""
    W = lookups.shape[1]
    bits = bleach(boot, lookups, p, thr)
    scores = popcount(boot, bits.reshape(S * l, k0, W), k0)
    idx = argmax(boot, scores, l)
    return np.stack(idx, axis=1), np.stack([d.reshape(S, l, W) for d in scores], axis=1)


def plain_predict(counters_lookup: np.ndarray, thr: int) -> np.ndarray:
    """(S, l, k0) decrypted lookups -> np.argmax of the bin-activated scores (hw/wnn.py:275-287)."""
    return np.argmax((counters_lookup > thr).sum(axis=2), axis=1)
