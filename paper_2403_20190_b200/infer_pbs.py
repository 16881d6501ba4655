"""Encrypted WiSARD inference with a bleaching threshold, popcount and argmax on the
batched PBS engine (second half; BASELINE configs[3]).

The reference stops at PD-act (`hw/hewnn.py:278-345`): the server packs the raw
counter lookups and the CLIENT activates, sums and takes the argmax in the clear
(`hw/wnn.py:275-309`).  Here the server does all of it on ciphertexts and returns
only an encrypted class index -- the OTF-act path the reference lists as a
non-goal (`SPEC.md:8`).  Plaintext semantics matched exactly:
`wnn.evaluate_dataset(model, bits, ActivationSpec("bin", thr))` -- per class c,
score_c = #{RAM j : counter_{c,j}(addr_j) > thr}, prediction = the first class
with the largest score (np.argmax ties).

Precision design.  A PBS at q = 2^32 resolves only a few bits: the
mod switch to 2N = 2048 phase units adds rounding noise sigma ~ 6.5 units, so one
bootstrap can tell apart at most 16 slots of 128 units.  The counters carry K =
log2 p bits (8 at cfg3) -- too many for one PBS.  So:

* every bootstrap is a SELF-bootstrap under the training key S1 (BSK = RGSW_S1(S1_j),
  j < N; no key switch, so no key-switch noise), fed straight back as input;
* counters are decomposed into radix-4 digits from the bottom by exact modulus
  reduction (the LWE shifted left, `C << (30 - s)`, is an exact LWE of the phase mod
  2^(s+2)) and two bootstraps per digit -- the sign (top bit) of the 4-slot torus,
  then the identity on the half torus for the low bit -- whose outputs are
  subtracted, clearing the digit (Liu-Micciancio-Wang's homomorphic floor);
* [m > thr] is the carry out of m + (p - thr - 1), a ripple-carry chain over the
  digits (one bootstrap per digit on values in [0, 8) with a padding bit);
* popcount: groups of 7 activated bits are added (value <= 7 fits one padded
  digit), split into radix-4 digits, and summed by a tree of ripple-carry adders;
* argmax: a tournament of strict comparisons (the higher class wins only if
  strictly larger: first-max ties) with bootstrapped digit selection.

All digits and bits live at scale 2^28 (16 slots, values 0..7 on the padded half
torus).  Every affine step is `hwb_lwe_lincomb`, every bootstrap
`tfhe.pbs_batch` (the FP64 FFT ladders, per-item test polynomials gathered by
`hwb_gather_rows`); each round batches all items of all images.  The C oracle
restates the pipeline in `oracle/infer32.py`.
"""

from __future__ import annotations

import ctypes
import dataclasses
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, tfhe
from ._lib import TfheError
from .params import HeParams

OUT_LOG = 28                    # scale of every digit / bit: q / 16
OUT = 1 << OUT_LOG
U32 = np.uint32


# ---------------------------------------------------------------------------
# keys


@dataclass
class SelfBootstrapKey:
    """RGSW_{S1}(S1_j) for j < N (NEW): bootstraps LWEs under the extracted key
    S1 back to S1 without a key switch.  `bsk` is the client's coefficient copy
    (the oracle's input), `device` the FFT/NTT-domain key on the GPU."""

    params: HeParams            # lwe_n = N
    bsk: np.ndarray             # (N, 2l, 2, N) uint32
    device: tfhe.BootstrapKey = field(repr=False)


def self_bootstrap_keygen(key: tfhe.SecretKey, rng_seed) -> SelfBootstrapKey:
    """BSK = enc_rgsw_batch(S1 bits under S1) (hw/tfhe.py:246-263, RNG idioms of
    hw/tfhe.py:33-47) for a client's existing RLWE key."""
    P = dataclasses.replace(key.params, lwe_n=key.params.n)
    rng = tfhe.make_rng(rng_seed)
    bsk = np.stack([c.data for c in tfhe.enc_rgsw_batch(key.s.astype(np.int64), key, rng)])
    return SelfBootstrapKey(P, bsk, tfhe.BootstrapKey.from_coefficients(P, bsk))


# ---------------------------------------------------------------------------
# device primitives


def _i32(a, dev) -> torch.Tensor | None:
    if a is None:
        return None
    w = (np.asarray(a, dtype=np.int64) & 0xFFFFFFFF).astype(np.uint32)
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32)).to(dev)


def lincomb(x: torch.Tensor, y: torch.Tensor | None = None, cx=None, cy=None, cb=None, shift: int = 0) -> torch.Tensor:
    """((cx x + cy y) << shift) + cb on the LWE bodies, mod 2^32, per row (hwb_lwe_lincomb).
    cx, cy, cb: None, a scalar or one value per row."""
    x = x.contiguous()                                  # the kernel reads dense (B, W) rows
    y = None if y is None else y.contiguous()
    B, W = x.shape
    dev = x.device

    def vec(v):
        if v is None:
            return None
        return _i32(np.broadcast_to(np.asarray(v, dtype=np.int64), (B,)), dev)
    out = torch.empty_like(x)
    vcx, vcy, vcb = vec(cx), vec(cy), vec(cb)
    if y is not None and cy is None:
        vcy = _i32(np.ones(B, dtype=np.int64), dev)
    _lib.check(_lib.load().hwb_lwe_lincomb(tfhe._ptr(x), tfhe._ptr(y), tfhe._ptr(out), tfhe._ptr(vcx),
                                           tfhe._ptr(vcy), tfhe._ptr(vcb), B, W, int(shift), tfhe._stream()))
    return out


def trivial(value: int, B: int, N: int, dev) -> torch.Tensor:
    """B trivial LWEs (0, value) under any key."""
    t = torch.zeros((B, N + 1), dtype=torch.int32, device=dev)
    v = int(value) & 0xFFFFFFFF
    t[:, N] = v - (1 << 32) if v >= 1 << 31 else v
    return t


class Luts:
    """The pipeline's test polynomials (one table on the device, rows addressed by name)."""

    def __init__(self, params: HeParams):
        self.P = params
        self.names: dict = {}
        self.rows: list[np.ndarray] = []
        self._dev = None

    def id(self, name, make) -> int:
        if name not in self.names:
            self.names[name] = len(self.rows)
            self.rows.append(np.asarray(make(), dtype=U32))
            self._dev = None
        return self.names[name]

    def table(self) -> torch.Tensor:
        if self._dev is None:
            self._dev = tfhe.to_device(np.stack(self.rows))
        return self._dev

    # --- the LUTs (test_polynomial: centred boxes of 2N/p units, negacyclic upper half)
    def sign(self, v: int) -> int:
        """+v for phase in [0, q/2), -v above: the sign / top bit of the 4-slot torus."""
        def mk():
            tv = np.zeros((2, self.P.n), dtype=U32)
            tv[1, :] = U32(v & 0xFFFFFFFF)
            return tv
        return self.id(("sign", v), mk)

    def half(self, f, p: int, v: int) -> int:
        """m -> f(m) * v for m in [0, p/2) (messages at q/p on the padded half torus)."""
        f = tuple(int(x) for x in f)
        return self.id(("half", f, p, v),
                       lambda: tfhe.test_polynomial(np.array(f), dataclasses.replace(self.P, p=p), delta_out=v))


def pbs(sbk: SelfBootstrapKey, luts: Luts, lwe: torch.Tensor, lut_ids, stats: dict | None = None) -> torch.Tensor:
    """One bootstrap round: item b evaluates LUT lut_ids[b] on lwe[b] (under S1)."""
    B = lwe.shape[0]
    if B == 0:
        return lwe.clone()
    P = sbk.params
    table = luts.table()
    idx = _i32(np.broadcast_to(np.asarray(lut_ids, dtype=np.int64), (B,)), lwe.device)
    tvs = torch.empty((B, 2, P.n), dtype=torch.int32, device=lwe.device)
    _lib.check(_lib.load().hwb_gather_rows(tfhe._ptr(table), tfhe._ptr(idx), tfhe._ptr(tvs), B, 2 * P.n,
                                           tfhe._stream()))
    out = tfhe.pbs_batch(P, lwe.contiguous(), tvs, sbk.device, None)
    if stats is not None:
        stats["pbs"] = stats.get("pbs", 0) + B
        stats["rounds"] = stats.get("rounds", 0) + 1
    return out


# ---------------------------------------------------------------------------
# bleaching: [m > thr] for m in Z_p at q/p


def bleach(sbk: SelfBootstrapKey, luts: Luts, lwe: torch.Tensor, p: int, thr: int, stats=None) -> torch.Tensor:
    """LWEs of m in Z_p at q/p -> LWEs of [m > thr] at 2^28 (wnn ActivationSpec("bin", thr),
    hw/wnn.py:86-109).  Radix-4 homomorphic floor + ripple carry of m + (p - thr - 1)."""
    B, W = lwe.shape
    N = W - 1
    K = p.bit_length() - 1
    if p != 1 << K or K < 1:
        raise TfheError("bleach needs a power-of-two counter modulus p >= 2")
    t = thr + 1
    if t <= 0:
        return trivial(OUT, B, N, lwe.device)
    if t >= p:
        return trivial(0, B, N, lwe.device)
    c = p - t                                               # [m >= t] = carry out of m + c
    D = K // 2
    C = lwe
    carry = None
    for i in range(D):                                      # radix-4 digits (odd K: plus a top bit)
        s = 32 - K + 2 * i                                  # C = (m >> 2i) 2^s + e
        top = i == D - 1 and K % 2 == 0                     # s = 30: nothing left to clear after it
        fine = s < OUT_LOG                                  # floor outputs need their own scale 2^s
        L = lincomb(C, shift=30 - s, cb=1 << 29)            # digit at 2^30, + half a slot
        ids = [luts.sign(OUT)] + ([luts.sign(1 << s)] if fine else [])
        sg = pbs(sbk, luts, L.repeat(len(ids), 1), np.repeat(ids, B), stats)
        b_cmp = sg[:B]                                      # (1 - 2b) 2^28, b = top bit of the digit
        b_flr, mb = (sg[B:], 1) if fine else (b_cmp, 1 << (s - OUT_LOG))
        C1 = lincomb(C, b_flr, cy=mb, cb=-(1 << s))         # C - b 2^(s+1): top bit cleared
        Lh = lincomb(C1, shift=30 - s)                      # low bit at 2^30 (half torus)
        ids = [luts.half((0, 1), 4, OUT)] + ([luts.half((0, 1), 4, 1 << s)] if fine and not top else [])
        lo = pbs(sbk, luts, Lh.repeat(len(ids), 1), np.repeat(ids, B), stats)
        lo_cmp = lo[:B]                                     # lo 2^28
        if not top:
            lo_flr, ml = (lo[B:], 1) if fine else (lo_cmp, 1 << (s - OUT_LOG))
            C = lincomb(C1, lo_flr, cy=-ml)                 # digit cleared: (m >> 2i+2) 2^(s+2) + e'
        # digit (2b + lo) + c_i + carry_in at 2^28, in [0, 7]
        ci = (c >> (2 * i)) & 3
        y = lincomb(lo_cmp, b_cmp, cy=-1, cb=OUT + ci * OUT)
        if carry is not None:
            y = lincomb(y, carry)
        carry = pbs(sbk, luts, y, luts.half([int(v >= 4) for v in range(8)], 16, OUT), stats)
    if K % 2:
        # the last, single-bit digit sits at 2^31: its sign bootstrap (offset by half a
        # slot) is the bit; carry out of bit + c_top + carry_in (base 2)
        L = lincomb(C, cb=1 << 30)
        sg = pbs(sbk, luts, L, luts.sign(OUT >> 1), stats)            # (1 - 2b) 2^27
        ct = (c >> (K - 1)) & 1
        y = lincomb(sg, cx=-1, cb=(OUT >> 1) + ct * OUT)                 # b 2^28 + c_top 2^28
        if carry is not None:
            y = lincomb(y, carry)
        carry = pbs(sbk, luts, y, luts.half([int(v >= 2) for v in range(8)], 16, OUT), stats)
    return carry


# ---------------------------------------------------------------------------
# radix-4 integers (digits at 2^28, values in [0, 4))


def _add_numbers(sbk, luts, A: list, Bn: list, max_digits: int, stats=None) -> list:
    """Ripple-carry sum of batches of radix-4 numbers (lists of (M, W) digit tensors)."""
    D = max(len(A), len(Bn))
    M, W = (A or Bn)[0].shape
    dev = (A or Bn)[0].device
    zero = trivial(0, M, W - 1, dev)
    out, carry = [], None
    mod4 = luts.half([v % 4 for v in range(8)], 16, OUT)
    div4 = luts.half([v // 4 for v in range(8)], 16, OUT)
    for i in range(D):
        a = A[i] if i < len(A) else zero
        b = Bn[i] if i < len(Bn) else zero
        s = lincomb(a, b)
        if carry is not None:
            s = lincomb(s, carry)
        last = i == D - 1 and D >= max_digits
        r = pbs(sbk, luts, s.repeat(1 if last else 2, 1), np.repeat([mod4] if last else [mod4, div4], M), stats)
        out.append(r[:M])
        carry = None if last else r[M:]
    if carry is not None:
        out.append(carry)
    return out


def popcount(sbk, luts, bits: torch.Tensor, max_value: int, stats=None) -> list:
    """bits (M, k, W) at 2^28 -> radix-4 digits of the M sums (list of (M, W))."""
    M, k, W = bits.shape
    dev = bits.device
    max_digits = max(1, int(np.ceil(np.log(max_value + 1) / np.log(4))))
    G = -(-k // 7)
    pad = G * 7 - k
    if pad:
        bits = torch.cat([bits, torch.zeros((M, pad, W), dtype=torch.int32, device=dev)], dim=1)
    g = bits.reshape(M * G, 7, W)
    v = g[:, 0].contiguous()
    for j in range(1, 7):
        v = lincomb(v, g[:, j].contiguous())              # group value in [0, 7]
    r = pbs(sbk, luts, v.repeat(2, 1), np.repeat([luts.half([x % 4 for x in range(8)], 16, OUT),
                                                  luts.half([x // 4 for x in range(8)], 16, OUT)], M * G), stats)
    nums = [r[: M * G].reshape(M, G, W), r[M * G:].reshape(M, G, W)]       # digits of each group value
    if max_digits < 2:
        nums = nums[:1]
    count = G
    while count > 1:
        half = count // 2
        A = [d[:, 0: 2 * half: 2].reshape(M * half, W) for d in nums]
        Bn = [d[:, 1: 2 * half: 2].reshape(M * half, W) for d in nums]
        S = _add_numbers(sbk, luts, A, Bn, max_digits, stats)
        S = [d.reshape(M, half, W) for d in S]
        if count % 2:                                       # the odd one rides along
            tail = [d[:, count - 1: count] for d in nums]
            tail += [torch.zeros((M, 1, W), dtype=torch.int32, device=dev)] * (len(S) - len(tail))
            S = [torch.cat([s_, t_], dim=1) for s_, t_ in zip(S, tail)]
            count = half + 1
        else:
            count = half
        nums = S
    return [d[:, 0].contiguous() for d in nums]


def _greater(sbk, luts, A: list, Bn: list, stats=None) -> torch.Tensor:
    """[B > A] for batches of radix-4 numbers (LSB-first ripple of 3-way digit compares)."""
    M, W = A[0].shape
    cmp2 = luts.half([0, 0, 0, 2, 4, 4, 4, 0], 16, OUT)     # b - a + 3 -> 2 sign3(b - a) + 2
    gt = luts.half([int(y >= 3) for y in range(8)], 16, OUT)
    r = None
    for i in range(len(A)):
        x = lincomb(Bn[i], A[i], cy=-1, cb=3 * OUT)        # b - a + 3 in [0, 6]
        c2 = pbs(sbk, luts, x, cmp2, stats)                # 0 / 2 / 4: b < a / = / > at this digit
        y = c2 if r is None else lincomb(c2, r)
        r = pbs(sbk, luts, y, gt, stats)
    return r


def _select(sbk, luts, gt: torch.Tensor, A: list, Bn: list, stats=None) -> list:
    """Digit-wise gt ? B : A."""
    M, W = gt.shape
    n = len(A)
    sel_a = luts.half([x if x < 4 else 0 for x in range(8)], 16, OUT)
    sel_b = luts.half([x - 4 if x >= 4 else 0 for x in range(8)], 16, OUT)
    xs = torch.cat([lincomb(d, gt, cy=4) for d in A] + [lincomb(d, gt, cy=4) for d in Bn])
    r = pbs(sbk, luts, xs, np.repeat([sel_a] * n + [sel_b] * n, M), stats)
    return [lincomb(r[i * M:(i + 1) * M], r[(n + i) * M:(n + i + 1) * M]) for i in range(n)]


def argmax(sbk, luts, scores: list, l: int, stats=None) -> list:
    """scores: digits (list of (S*l, W), class-major within a sample) -> radix-4 digits of
    the first maximal class per sample (np.argmax ties): a tournament where the
    higher-numbered candidate wins only when strictly greater."""
    SL, W = scores[0].shape
    S = SL // l
    dev = scores[0].device
    nd = max(1, int(np.ceil(np.log(l) / np.log(4))))
    cand = [d.reshape(S, l, W) for d in scores]
    idx = [torch.stack([trivial(((c >> (2 * k)) & 3) * OUT, S, W - 1, dev) for c in range(l)], dim=1)
           for k in range(nd)]                              # public class numbers, trivially encrypted
    count = l
    while count > 1:
        half = count // 2

        def pairs(ds, o):
            return [d[:, o: 2 * half: 2].reshape(S * half, W).contiguous() for d in ds]
        A, Bn, IA, IB = pairs(cand, 0), pairs(cand, 1), pairs(idx, 0), pairs(idx, 1)
        g = _greater(sbk, luts, A, Bn, stats)               # [B > A]: ties keep the lower class
        sel = _select(sbk, luts, g, A + IA, Bn + IB, stats)
        win = [d.reshape(S, half, W) for d in sel[: len(A)]]
        wix = [d.reshape(S, half, W) for d in sel[len(A):]]
        if count % 2:                                       # the odd one rides along
            win = [torch.cat([w, d[:, count - 1: count]], dim=1) for w, d in zip(win, cand)]
            wix = [torch.cat([w, d[:, count - 1: count]], dim=1) for w, d in zip(wix, idx)]
        cand, idx, count = win, wix, half + count % 2
    return [d[:, 0].contiguous() for d in idx]


# ---------------------------------------------------------------------------
# the inference entry point


@dataclass
class EncryptedPrediction:
    """Server output: radix-4 digits (LSB first) of the predicted class, LWEs under S1
    at 2^28; optionally the per-class scores (digits) for inspection."""

    params: HeParams
    index_digits: np.ndarray            # (D, N+1) uint32
    score_digits: np.ndarray | None = None   # (D', l, N+1)


def he_infer_bin_batch(model, samples, sbk: SelfBootstrapKey, thr: int, ladder: str = "auto",
                       keep_scores: bool = False, stats: dict | None = None) -> list[EncryptedPrediction]:
    """OTF-act inference: VP lookups (as he_infer_pd, hw/hewnn.py:278-320), then the
    bleaching threshold, per-class popcount and argmax on ciphertexts."""
    from . import hewnn
    geometry, params = model.geometry, model.params
    if sbk.params.n != params.n or sbk.params.gadget != params.gadget:
        raise TfheError("self-bootstrapping key does not match the model's ring")
    l, k0 = geometry.l, geometry.k0
    S = len(samples)
    lwe = hewnn.vp_lookups(model, samples, ladder=ladder)                 # (S*l*k0, N+1) under S1
    luts = Luts(params)
    bits = bleach(sbk, luts, lwe, params.p, thr, stats)                    # (S*l*k0, N+1) at 2^28
    scores = popcount(sbk, luts, bits.reshape(S * l, k0, -1), k0, stats)    # digits of (S*l) scores
    idx = argmax(sbk, luts, scores, l, stats)
    out_idx = np.stack([tfhe.to_host(d) for d in idx], axis=1)              # (S, D, N+1)
    sc = np.stack([tfhe.to_host(d).reshape(S, l, -1) for d in scores], axis=1) if keep_scores else None
    return [EncryptedPrediction(params, out_idx[i], None if sc is None else sc[i]) for i in range(S)]


def decrypt_prediction(pred: EncryptedPrediction, key: tfhe.SecretKey) -> int:
    """Client: decrypt the radix-4 index digits (values at 2^28, p = 16)."""
    P16 = dataclasses.replace(pred.params, p=16)
    digits = tfhe.dec_lwe_batch(pred.index_digits, key, P16)
    return int(sum(int(d) << (2 * k) for k, d in enumerate(digits)))


def decrypt_scores(pred: EncryptedPrediction, key: tfhe.SecretKey) -> np.ndarray:
    P16 = dataclasses.replace(pred.params, p=16)
    D, l, W = pred.score_digits.shape
    d = tfhe.dec_lwe_batch(pred.score_digits.reshape(D * l, W), key, P16).reshape(D, l)
    return (d * (4 ** np.arange(D))[:, None]).sum(axis=0)
