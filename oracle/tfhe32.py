"""CPU oracle for batched TFHE bootstrapping at q = 2^32 -- TEST INFRASTRUCTURE.

This module is the parity checker, not the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may import it.
The product (`paper_2403_20190_b200`) never routes through it.

It restates the reference (`/root/reference/pkg/src/hewisard`, cited as
`hw/<file>:<line>`) with q lowered from 2^64 to 2^32.  Everything is exact
integer arithmetic mod 2^32:

* functions that exist in the reference follow its algorithm line by line
  (schoolbook negacyclic products via `np.convolve`, the LSB-first signed
  digit loop, the CMUX algebra, the extraction sign pattern);
* functions the reference lacks (mod switch, test polynomial, LWE key
  switch, PBS composition, the q=2^32 key/LWE generation) are NEW and say so.

Pinning: `tests/golden/make_golden.py` runs the real reference on operands
embedded as x << 32 (exact_mul parameter sets; SURVEY.md §0 finding 4) and
commits the results under `tests/golden/`; `tests/test_oracle.py` checks this
module (and the C oracle in `oracle/c/`) against those fixtures.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

U32 = np.uint32
U64 = np.uint64
Q_BITS = 32
MASK32 = (1 << 32) - 1


# ---------------------------------------------------------------------------
# RNG idioms (hw/tfhe.py:33-47) at 4-byte words


def make_rng(seed) -> np.random.Generator:
    """hw/tfhe.py:33-35."""
    return np.random.Generator(np.random.Philox(seed))


def uniform_u32(rng: np.random.Generator, shape) -> np.ndarray:
    """hw/tfhe.py:38-40 with 4-byte little-endian words."""
    n = int(np.prod(shape)) if shape else 1
    return np.frombuffer(rng.bytes(4 * n), dtype="<u4").reshape(shape).astype(U32)


def gaussian_u32(rng: np.random.Generator, sigma: float, shape) -> np.ndarray:
    """hw/tfhe.py:43-47: rint(normal) wrapped into Z_q; sigma == 0 draws nothing."""
    if sigma == 0.0:
        return np.zeros(shape, dtype=U32)
    e = np.rint(rng.normal(0.0, sigma, shape))
    return (e.astype(np.int64) & MASK32).astype(U32)


# ---------------------------------------------------------------------------
# ring arithmetic (hw/ring.py)


def negacyclic_mul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """hw/ring.py:92-98: uint64 schoolbook convolution folded by X^N = -1.

    The uint64 wrap is mod 2^64, a multiple of 2^32, so reducing the result
    mod 2^32 afterwards is exact.
    """
    a = np.asarray(a).astype(np.int64).astype(U64)
    b = np.asarray(b).astype(np.int64).astype(U64)
    n = a.shape[-1]
    conv = np.convolve(a, b)
    out = conv[:n].copy()
    out[: n - 1] -= conv[n:]
    return (out & U64(MASK32)).astype(U32)


def monomial_mul(x: np.ndarray, e: int) -> np.ndarray:
    """hw/ring.py:106-113: x * X^e, e taken mod 2N."""
    n = x.shape[-1]
    e = int(e) % (2 * n)
    if e == 0:
        return x.copy()
    ext = np.concatenate([x, (np.zeros_like(x) - x)], axis=-1)
    idx = (np.arange(n) - e) % (2 * n)
    return ext[..., idx]


def monomial_gather(x: np.ndarray, es) -> np.ndarray:
    """hw/lut.py:317-325: per-item x_i * X^(es_i)."""
    n = x.shape[-1]
    es = np.asarray(es, dtype=np.int64) % (2 * n)
    if not es.any():
        return x
    ext = np.concatenate([x, np.zeros_like(x) - x], axis=-1)
    idx = (np.arange(n) - es.reshape(es.shape + (1,) * (x.ndim - 1))) % (2 * n)
    return np.take_along_axis(ext, idx, axis=-1)


def gadget_decompose(x: np.ndarray, levels: int, base_log: int) -> np.ndarray:
    """hw/ring.py:126-151 at Q = 32: u32 (..., N) -> int64 (..., levels, N).

    Round to a multiple of 2^(32 - levels*w), then peel signed digits in
    [-beta/2, beta/2) LSB-first with carry; digit t carries q / beta^(t+1).
    """
    w = base_log
    total = levels * w
    x = np.asarray(x, dtype=U32).astype(U64)
    beta = U64(1 << w)
    half = U64(1 << (w - 1))
    mask = beta - U64(1)
    if total < Q_BITS:
        u = (x + U64(1 << (Q_BITS - total - 1))) & U64(MASK32)
        u >>= U64(Q_BITS - total)
    else:
        u = x.copy()
    out = np.empty(x.shape[:-1] + (levels, x.shape[-1]), dtype=U64)
    for t in range(levels - 1, -1, -1):
        d = u & mask
        d -= (d >= half) * beta            # two's-complement wrap (mod 2^64)
        u -= d
        u >>= U64(w)
        out[..., t, :] = d
    return out.view(np.int64)


def gadget_recompose(digits: np.ndarray, levels: int, base_log: int) -> np.ndarray:
    """hw/ring.py:154-160 on a (..., levels, N) digit array."""
    acc = np.zeros(digits.shape[:-2] + digits.shape[-1:], dtype=np.int64)
    for t in range(levels):
        acc += digits[..., t, :] * (1 << (Q_BITS - (t + 1) * base_log))
    return (acc & MASK32).astype(U32)


def digits_of(cts: np.ndarray, levels: int, base_log: int) -> np.ndarray:
    """hw/tfhe.py:290-298: (..., 2, N) -> (..., 2*levels, N), b digits first."""
    d = gadget_decompose(cts, levels, base_log)        # (..., 2, levels, N)
    return np.concatenate([d[..., 1, :, :], d[..., 0, :, :]], axis=-2)


# ---------------------------------------------------------------------------
# homomorphic operations (hw/tfhe.py)


def ext_product_batch(rgsw: np.ndarray, cts: np.ndarray, levels: int,
                      base_log: int) -> np.ndarray:
    """hw/tfhe.py:301-315 (exact branch): rgsw (B|1, 2l, 2, N), cts (B, 2, N)."""
    cts = np.asarray(cts, dtype=U32)
    digits = digits_of(cts, levels, base_log)
    rows = np.broadcast_to(rgsw, digits.shape[:-2] + rgsw.shape[-3:])
    out = np.zeros(cts.shape, dtype=U32)
    flat_d = digits.reshape(-1, digits.shape[-2], digits.shape[-1])
    flat_r = rows.reshape(-1, rows.shape[-3], 2, rows.shape[-1])
    flat_o = out.reshape(-1, 2, out.shape[-1])
    for i in range(flat_d.shape[0]):
        for r in range(flat_d.shape[1]):
            for c in range(2):
                flat_o[i, c] += negacyclic_mul(flat_d[i, r], flat_r[i, r, c])
    return out


def cmux(rgsw: np.ndarray, c1: np.ndarray, c2: np.ndarray, levels: int,
         base_log: int) -> np.ndarray:
    """hw/tfhe.py:334-337: c2 + C (*) (c1 - c2)."""
    diff = (c1 - c2).astype(U32)
    return (c2 + ext_product_batch(rgsw[np.newaxis], diff[np.newaxis], levels,
                                   base_log)[0]).astype(U32)


def blind_rotate(c: np.ndarray, C: Sequence[np.ndarray], I: Sequence[int],
                 levels: int, base_log: int) -> np.ndarray:
    """hw/tfhe.py:340-349: acc <- cmux(C_i, acc * X^(-I_i), acc)."""
    if len(C) != len(I):
        raise ValueError("selector/exponent length mismatch")
    acc = np.array(c, dtype=U32)
    for Ci, Ii in zip(C, I):
        rotated = monomial_mul(acc, -int(Ii))
        acc = cmux(Ci, rotated, acc, levels, base_log)
    return acc


def extract_lwe(c: np.ndarray, i: int = 0) -> tuple[np.ndarray, int]:
    """hw/tfhe.py:352-361: LWE of coefficient i under the coefficients of S1."""
    n = c.shape[-1]
    if not 0 <= i < n:
        raise ValueError(f"coefficient index {i} out of range [0, {n})")
    a = c[0]
    out = np.empty(n, dtype=U32)
    out[: i + 1] = a[: i + 1][::-1]
    out[i + 1:] = np.zeros(n - i - 1, dtype=U32) - a[i + 1:][::-1]
    return out, int(c[1][i])


def extract_lwe_batch(cts: np.ndarray) -> np.ndarray:
    """Batched coefficient-0 extraction (hw/lut.py:263-266) -> (B, N+1), b last."""
    B, _, n = cts.shape
    out = np.empty((B, n + 1), dtype=U32)
    out[:, 0] = cts[:, 0, 0]
    out[:, 1:n] = np.zeros((B, n - 1), dtype=U32) - cts[:, 0, :0:-1]
    out[:, n] = cts[:, 1, 0]
    return out


# ---------------------------------------------------------------------------
# keys, encryption, decryption


def key_mul(x: np.ndarray, s: np.ndarray) -> np.ndarray:
    """x * s mod 2^32 for a binary key s; batched over leading axes.

    Restates the limb-exact FFT product of hw/fft.py:88-119 with 16-bit limbs:
    every limb convolution is < N * 2^16 < 2^53, so rounding recovers exact
    integers.  Cross-checked against `negacyclic_mul` in tests/test_oracle.py.
    """
    x = np.asarray(x, dtype=U32)
    n = x.shape[-1]
    fs = np.fft.rfft(np.asarray(s, dtype=np.float64), 2 * n)
    out = np.zeros(x.shape, dtype=U64)
    for shift in (0, 16):
        limb = ((x >> U32(shift)) & U32(0xFFFF)).astype(np.float64)
        conv = np.fft.irfft(np.fft.rfft(limb, 2 * n, axis=-1) * fs, 2 * n, axis=-1)
        conv = np.rint(conv).astype(np.int64)
        fold = conv[..., :n] - np.concatenate(
            [conv[..., n:2 * n - 1], np.zeros(x.shape[:-1] + (1,), dtype=np.int64)], axis=-1)
        out += (fold.astype(U64) << U64(shift))
    return (out & U64(MASK32)).astype(U32)


def decode_phase(phase: np.ndarray, p: int) -> np.ndarray:
    """hw/tfhe.py:223-225 at Q = 32."""
    half = U64((1 << Q_BITS) // p // 2)
    ph = np.asarray(phase).astype(U64)
    return (((ph + half) & U64(MASK32)) >> U64(Q_BITS - p.bit_length() + 1)).astype(np.int64)


def phase_rlwe(ct: np.ndarray, s: np.ndarray) -> np.ndarray:
    """hw/tfhe.py:214-215."""
    return (ct[..., 1, :] - key_mul(ct[..., 0, :], s)).astype(U32)


def dec_rlwe(ct: np.ndarray, s: np.ndarray, p: int) -> np.ndarray:
    """hw/tfhe.py:218-220."""
    return decode_phase(phase_rlwe(ct, s), p)


def phase_lwe(lwe: np.ndarray, s: np.ndarray) -> np.ndarray:
    """hw/tfhe.py:364-366 on (..., n+1) rows with b last."""
    lwe = np.asarray(lwe, dtype=U32)
    dot = (lwe[..., :-1].astype(U64) * np.asarray(s, dtype=U64)).sum(axis=-1, dtype=U64)
    return ((lwe[..., -1].astype(U64) - dot) & U64(MASK32)).astype(U32)


def dec_lwe(lwe: np.ndarray, s: np.ndarray, p: int) -> np.ndarray:
    """hw/tfhe.py:369-370."""
    return decode_phase(phase_lwe(lwe, s), p)


def enc_rlwe_raw(mu: np.ndarray, s: np.ndarray, sigma: float,
                 rng: np.random.Generator) -> np.ndarray:
    """hw/tfhe.py:200-206."""
    n = len(s)
    a = uniform_u32(rng, (n,))
    e = gaussian_u32(rng, sigma, (n,))
    b = key_mul(a, s) + np.asarray(mu, dtype=U32) + e
    return np.stack([a, b.astype(U32)])


def encode(m, p: int, n: int) -> np.ndarray:
    """hw/tfhe.py:181-190."""
    m = np.atleast_1d(np.asarray(m, dtype=np.int64))
    mu = np.zeros(n, dtype=U32)
    mu[: m.size] = (m.astype(np.int64) * ((1 << Q_BITS) // p)) & MASK32
    return mu


def trivial_rlwe(m, p: int, n: int) -> np.ndarray:
    """hw/tfhe.py:193-197."""
    data = np.zeros((2, n), dtype=U32)
    data[1] = encode(m, p, n)
    return data


def enc_rgsw_batch(ms, s: np.ndarray, sigma: float, levels: int, base_log: int,
                   rng: np.random.Generator) -> np.ndarray:
    """hw/tfhe.py:246-263 at Q = 32 -> (B, 2l, 2, N).

    Stream order: all a (B, 2l, N) via rng.bytes, then all e (B, 2l, N).
    Gadget on the b component of rows t, on the a component of rows l+t.
    """
    ms = np.asarray(ms, dtype=np.int64)
    n = len(s)
    rows = 2 * levels
    a = uniform_u32(rng, (len(ms), rows, n))
    e = gaussian_u32(rng, sigma, (len(ms), rows, n))
    b = (key_mul(a, s) + e).astype(U32)
    data = np.stack([a, b], axis=2)
    for t in range(levels):
        g = U32(1 << (Q_BITS - (t + 1) * base_log))
        data[:, t, 1, 0] += ms.astype(U32) * g
        data[:, levels + t, 0, 0] += ms.astype(U32) * g
    return data


def dec_rgsw(ct: np.ndarray, s: np.ndarray, base_log: int) -> int:
    """hw/tfhe.py:278-283."""
    phase = phase_rlwe(ct[0], s)
    g0 = 1 << (Q_BITS - base_log)
    val = ((int(phase[0]) + g0 // 2) & MASK32) >> (Q_BITS - base_log)
    return val % (1 << base_log)


# ---------------------------------------------------------------------------
# NEW (absent from the reference): LWE side of programmable bootstrapping


def enc_lwe_batch(mu: np.ndarray, s0: np.ndarray, sigma: float,
                  rng: np.random.Generator) -> np.ndarray:
    """NEW: LWE_{s0}(mu) rows (B, n+1), b last.  Stream: a (B, n) then e (B,)."""
    mu = np.asarray(mu, dtype=np.int64)
    B, n = len(mu), len(s0)
    a = uniform_u32(rng, (B, n))
    e = gaussian_u32(rng, sigma, (B,))
    dot = (a.astype(U64) * np.asarray(s0, dtype=U64)).sum(axis=-1, dtype=U64)
    b = (dot + e.astype(U64) + (mu & MASK32).astype(U64)) & U64(MASK32)
    return np.concatenate([a, b.astype(U32)[:, None]], axis=1)


def pbs_keygen(params, rng_seed) -> dict:
    """NEW: keys for PBS at q = 2^32 from one Philox stream.

    Order: s1 = integers(0,2,N) (as hw/tfhe.py:99), s0 = integers(0,2,n),
    BSK = enc_rgsw_batch(s0 under s1) (hw/tfhe.py:246-263), then the LWE
    key-switch key KSK[j, t] = LWE_{s0}(s1_j * q / beta_ks^(t+1)) with
    a (N, l_ks, n) drawn first and e (N, l_ks) after.
    """
    rng = make_rng(rng_seed)
    N, n = params.n, params.lwe_n
    s1 = rng.integers(0, 2, N).astype(U32)
    s0 = rng.integers(0, 2, n).astype(U32)
    g = params.gadget
    bsk = enc_rgsw_batch(s0, s1, params.sigma, g.levels, g.base_log, rng)
    gk = params.gadget_ks
    a = uniform_u32(rng, (N, gk.levels, n))
    e = gaussian_u32(rng, params.lwe_sigma, (N, gk.levels))
    dot = (a.astype(U64) * s0.astype(U64)).sum(axis=-1, dtype=U64)
    msg = np.zeros((N, gk.levels), dtype=U64)
    for t in range(gk.levels):
        msg[:, t] = s1.astype(U64) * U64(1 << (Q_BITS - (t + 1) * gk.base_log))
    b = (dot + e.astype(U64) + msg) & U64(MASK32)
    ksk = np.concatenate([a, b.astype(U32)[..., None]], axis=-1)   # (N, l_ks, n+1)
    return dict(s0=s0, s1=s1, bsk=bsk, ksk=ksk)


def keygen_packing(params, rng_seed) -> tuple[np.ndarray, np.ndarray]:
    """hw/tfhe.py:95-114 at q = 2^32: S1 and the packing key-switch key
    (N, l, 2, N), in the reference's chunked RNG order."""
    rng = make_rng(rng_seed)
    n = params.n
    s = rng.integers(0, 2, n).astype(U32)
    g = params.gadget_pks
    ksk = np.empty((n, g.levels, 2, n), dtype=U32)
    step = max(1, 2 ** 20 // (g.levels * n))
    for j0 in range(0, n, step):
        j1 = min(n, j0 + step)
        a = uniform_u32(rng, (j1 - j0, g.levels, n))
        e = gaussian_u32(rng, params.sigma, (j1 - j0, g.levels, n))
        b = (key_mul(a, s) + e).astype(U32)
        for t in range(g.levels):
            b[:, t, 0] += s[j0:j1] * U32(1 << (Q_BITS - (t + 1) * g.base_log))
        ksk[j0:j1, :, 0, :] = a
        ksk[j0:j1, :, 1, :] = b
    return s, ksk


def mod_switch(x, n_ring: int) -> np.ndarray:
    """NEW: round(x * 2N / q) mod 2N with the rounding idiom of hw/ring.py:139-140."""
    logm = (2 * n_ring).bit_length() - 1
    x = np.asarray(x, dtype=U64)
    return (((x + U64(1 << (Q_BITS - logm - 1))) & U64(MASK32)) >> U64(Q_BITS - logm)).astype(np.int64)


def test_polynomial(f, p: int, n_ring: int, delta_out: int | None = None) -> np.ndarray:
    """NEW: trivial GLWE (0, TV) for the LUT m -> f(m), m in [0, p/2).

    Box of 2N/p phase units per message, centred (half-box offset); the
    negacyclic wrap makes m in [p/2, p) evaluate to -f(m - p/2).
    """
    if delta_out is None:
        delta_out = (1 << Q_BITS) // p
    box = 2 * n_ring // p
    f = np.asarray(f, dtype=np.int64)
    j = np.arange(n_ring)
    m = (j + box // 2) // box
    val = np.where(m < p // 2, f[np.minimum(m, p // 2 - 1)] * delta_out,
                   -f[np.clip(m - p // 2, 0, p // 2 - 1)] * delta_out)
    tv = np.zeros((2, n_ring), dtype=U32)
    tv[1] = (val & MASK32).astype(U32)
    return tv


def lwe_keyswitch(lwe: np.ndarray, ksk: np.ndarray, levels: int,
                  base_log: int) -> np.ndarray:
    """NEW: LWE (B, N+1) under s1 -> (B, n+1) under s0.

    Algebra of the packing key switch hw/tfhe.py:397-420: signed digits of
    each a'_j (hw/ring.py:126-151), out = (0, b') - sum_{j,t} d_{j,t} KSK[j,t].
    """
    lwe = np.asarray(lwe, dtype=U32)
    B = lwe.shape[0]
    N = lwe.shape[1] - 1
    d = gadget_decompose(lwe[:, :N], levels, base_log)        # (B, levels, N)
    d = np.swapaxes(d, 1, 2).reshape(B, N * levels)          # index j*levels + t
    K = ksk.reshape(N * levels, -1).astype(np.int64)          # (N*l, n+1)
    acc = np.zeros((B, K.shape[1]), dtype=np.int64)
    for c0 in range(0, N * levels, 512):                      # bounded int64 sums
        acc = (acc + (d[:, c0:c0 + 512] @ K[c0:c0 + 512])) & MASK32
    out = (np.zeros((B, K.shape[1]), dtype=np.int64) - acc) & MASK32
    out[:, -1] = (lwe[:, N].astype(np.int64) - acc[:, -1]) & MASK32
    return out.astype(U32)


def pbs(lwe: np.ndarray, tv: np.ndarray, bsk: np.ndarray, ksk: np.ndarray,
        params, *, keyswitch: bool = True) -> np.ndarray:
    """NEW composition, one ciphertext at a time:

    mod switch -> acc0 = TV * X^(-b~) (hw/ring.py:106) -> blind_rotate with
    I_i = -a~_i (hw/tfhe.py:340-349) -> extract coefficient 0
    (hw/tfhe.py:352-361) -> LWE key switch.
    """
    lwe = np.asarray(lwe, dtype=U32)
    N = params.n
    g = params.gadget
    tv = np.asarray(tv, dtype=U32)
    out = []
    for i, row in enumerate(lwe):
        ms = mod_switch(row, N)
        t = tv if tv.ndim == 2 else tv[i]
        acc = monomial_mul(t, -int(ms[-1]))
        acc = blind_rotate(acc, list(bsk), [-int(x) for x in ms[:-1]], g.levels, g.base_log)
        a, b = extract_lwe(acc, 0)
        out.append(np.concatenate([a, [U32(b)]]).astype(U32))
    out = np.stack(out)
    if keyswitch:
        gk = params.gadget_ks
        out = lwe_keyswitch(out, ksk, gk.levels, gk.base_log)
    return out
