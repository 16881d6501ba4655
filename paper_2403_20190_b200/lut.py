"""Encrypted lookup tables on B200: vertical packing and its inverse.

Mirror of the reference's `hewisard.lut` (`pkg/src/hewisard/lut.py`).  The
selector order is the reference's: a k-bit selector feeds the CMUX/CDEMUX tree
with the most-significant index bits first (positions 0..z-1, z = max(0, k -
log2 N)) and the blind rotation with the least-significant bits (position z+i
carries weight 2^i); table entry m lives at polynomial m // N, coefficient
m % N (`lut.py:1-11`).

Every homomorphic step runs in libhwb200: the rotation CMUXes (`hwb_cmux` with a
per-item rotation and GGSW), the tree levels (`hwb_ivp_level` / `hwb_vp_level`),
clear rotations (`hwb_monomial_gather`) and extraction.  Encrypted selector bits
are addressed as rows of one device GGSW table (`tfhe.GgswNtt`); the batched
entry points take an int32 code matrix: code >= 0 is a table row, -1 a clear 0,
-2 a clear 1.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, tfhe
from ._lib import TfheError
from .params import HeParams, named_params
from .tfhe import GgswFft, GgswNtt, RgswCiphertext, RlweCiphertext

CLEAR0, CLEAR1 = -1, -2
# ring geometry only (the gather needs N): parameter sets of each supported degree
_ANY_1024 = named_params("CFG2")
_ANY_2048 = named_params("CFG4")


@dataclass
class SelectorBit:
    """Either a public bit or an RGSW encryption of one (hw/lut.py:25-44)."""

    ct: RgswCiphertext | None = None
    bit: int | None = None

    @classmethod
    def clear(cls, bit: int) -> "SelectorBit":
        if bit not in (0, 1):
            raise ValueError("selector bits are binary")
        return cls(bit=bit)

    @classmethod
    def enc(cls, ct: RgswCiphertext) -> "SelectorBit":
        return cls(ct=ct)

    @property
    def is_clear(self) -> bool:
        return self.ct is None


@dataclass
class EncryptedLut:
    """2^k-entry table packed into max(1, 2^k / N) RLWE ciphertexts (hw/lut.py:47-63)."""

    polys: list[RlweCiphertext]
    k: int

    def __post_init__(self):
        n = self.polys[0].params.n
        want = max(1, (1 << self.k) // n)
        if len(self.polys) != want:
            raise TfheError(f"a LUT with k = {self.k} holds {want} polynomials, not {len(self.polys)}")

    @property
    def params(self) -> HeParams:
        return self.polys[0].params


def tree_depth(k: int, params: HeParams) -> int:
    """hw/lut.py:66-67."""
    return max(0, k - params.degree_log)


def rotate_weights(k: int, params: HeParams) -> list[int]:
    """Index weights of the rotation positions, LSB-first (hw/lut.py:70-72)."""
    return list(range(min(k, params.degree_log)))


def selector_index(bits: list[int], k: int, params: HeParams) -> int:
    """Table index encoded by a full selector vector (hw/lut.py:75-83)."""
    z = tree_depth(k, params)
    m = 0
    for i in range(z):
        m += bits[i] << (k - 1 - i)
    for i, w in enumerate(rotate_weights(k, params)):
        m += bits[z + i] << w
    return m


# ---------------------------------------------------------------------------
# device primitives


def _cp(params):
    return ctypes.byref(_lib.c_params(params))


def _i32(x, device) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.int64))
    return t.to(device=device, dtype=torch.int32).contiguous()


def monomial_gather(*args):
    """Per-item x_i * X^(es_i) (hw/lut.py:317-325) on the GPU.  Reference form
    `monomial_gather(x, es)` (ring degree from x), or `monomial_gather(params, x, es)`."""
    if len(args) == 3:
        params, x, es = args
    elif len(args) == 2:
        x, es = args
        n = int(np.shape(x)[-1]) if not isinstance(x, torch.Tensor) else int(x.shape[-1])
        params = {1024: _ANY_1024, 2048: _ANY_2048}.get(n)
        if params is None:
            raise TfheError(f"ring degree {n} is not supported (1024 or 2048)")
    else:
        raise TypeError("monomial_gather(x, es) or monomial_gather(params, x, es)")
    t = tfhe.to_device(x)
    shape = t.shape
    t = t.reshape(-1, 2, params.n) if t.dim() != 3 else t
    B = t.shape[0]
    e = _i32(np.asarray(es, dtype=np.int64) % (2 * params.n) if not isinstance(es, torch.Tensor) else es, t.device)
    if e.numel() != B:
        raise TfheError("one exponent per ciphertext")
    out = torch.empty_like(t)
    _lib.check(_lib.load().hwb_monomial_gather(_cp(params), tfhe._ptr(t), tfhe._ptr(out), tfhe._ptr(e), B,
                                               tfhe._stream()))
    return tfhe._wrap(x, out.reshape(shape))


def accumulate_(dst: torch.Tensor, src: torch.Tensor, negate: bool = False) -> torch.Tensor:
    """dst += src (mod 2^32, in place); src may be a shorter block repeated over dst."""
    if dst.numel() % max(1, src.numel()):
        raise TfheError("accumulate: shapes do not tile")
    _lib.check(_lib.load().hwb_accumulate(tfhe._ptr(dst), tfhe._ptr(src), dst.numel(), src.numel(),
                                          1 if negate else 0, tfhe._stream()))
    return dst


def accumulate_rows_(dst: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    """dst += sum_i rows[i] (mod 2^32, in place, one pass over rows)."""
    words = dst.numel()
    if rows.numel() % words:
        raise TfheError("accumulate_rows: rows do not tile dst")
    _lib.check(_lib.load().hwb_accumulate_rows(tfhe._ptr(dst), tfhe._ptr(rows), words, rows.numel() // words,
                                               tfhe._stream()))
    return dst


def _upload_i32(arrays, device) -> list[torch.Tensor]:
    """Several small host index arrays -> device int32 views through ONE pinned,
    non-blocking copy.  A pageable copy would block the host until the stream
    drains and queue behind in-flight bulk transfers (he_train stages the next
    chunk's RGSW stacks on a copy stream)."""
    flat = [np.ascontiguousarray(np.asarray(a, dtype=np.int64).astype(np.int32)).ravel() for a in arrays]
    host = torch.from_numpy(np.concatenate(flat) if flat else np.zeros(0, np.int32)).pin_memory()
    dev = host.to(device, non_blocking=True)
    out, off = [], 0
    for a, f in zip(arrays, flat):
        out.append(dev[off: off + f.size].view(np.shape(a)))
        off += f.size
    return out


def _rotation_ladder(params, table: GgswNtt | GgswFft, acc: torch.Tensor, cols: np.ndarray, sign: int,
                     dev_args: tuple | None = None) -> torch.Tensor:
    """All encrypted rotation positions of a selector batch in ONE launch
    (hwb_blind_rotate with per-item GGSW rows): for position i (weight 2^i),
    acc <- cmux(C, acc * X^(sign 2^i), acc) where the bit is encrypted; clear
    positions (code < 0) are skipped here and applied by the caller's gather,
    exactly the reference's order (hw/lut.py:249-261, 280-292)."""
    B, L = cols.shape
    if L == 0 or not (cols >= 0).any():
        return acc
    dev = acc.device
    if dev_args is not None:
        idx, exps = dev_args
    else:
        idx = _i32(np.where(cols >= 0, cols, -1), dev)
        exps = _i32(_rotation_exps(params, B, L, sign), dev)
    out = acc.contiguous().clone()
    fn = _lib.load().hwb_blind_rotate_fft if isinstance(table, GgswFft) else _lib.load().hwb_blind_rotate
    _lib.check(fn(_cp(params), tfhe._ptr(table.data), tfhe._ptr(idx), tfhe._ptr(exps), tfhe._ptr(out), L, B,
                  tfhe._stream()))
    return out


def _rotation_exps(params, B: int, L: int, sign: int) -> np.ndarray:
    return np.broadcast_to(-sign * (1 << np.arange(L, dtype=np.int64)), (B, L)) % (2 * params.n)


def _level(params, table: GgswNtt | GgswFft, cur: torch.Tensor, idx: torch.Tensor, inverse: bool) -> torch.Tensor:
    B, mm = cur.shape[0], cur.shape[1]
    fft = isinstance(table, GgswFft)
    if inverse:
        nxt = torch.empty((B, 2 * mm) + tuple(cur.shape[2:]), dtype=torch.int32, device=cur.device)
        fn, m = (_lib.load().hwb_ivp_level_fft if fft else _lib.load().hwb_ivp_level), mm
    else:
        nxt = torch.empty((B, mm // 2) + tuple(cur.shape[2:]), dtype=torch.int32, device=cur.device)
        fn, m = (_lib.load().hwb_vp_level_fft if fft else _lib.load().hwb_vp_level), mm // 2
    _lib.check(fn(_cp(params), tfhe._ptr(table.data), tfhe._ptr(idx), tfhe._ptr(cur), tfhe._ptr(nxt), m, B,
                  tfhe._stream()))
    return nxt


# ---------------------------------------------------------------------------
# batched engines over code matrices


def ivp_codes(params: HeParams, codes, table: GgswNtt | None, payload,
              dev_codes: torch.Tensor | None = None) -> torch.Tensor:
    """Inverse vertical packing (hw/lut.py:269-314) for B items sharing one payload.

    codes: (B, k) int (row of `table`, CLEAR0 or CLEAR1).  Returns the device
    tensor (B, max(1, 2^z), 2, N) of single-valued LUT rows.  dev_codes: the
    same codes already on the device (int32), so the pass issues no host->device
    copy at all (he_train uploads one chunk's codes once and reuses them)."""
    codes = np.asarray(codes, dtype=np.int64)
    B, k = codes.shape
    z = tree_depth(k, params)
    n = params.n
    pay = tfhe.to_device(payload)
    dev = pay.device
    acc = pay.reshape(1, 2, n).expand(B, 2, n).contiguous()
    nrot = len(rotate_weights(k, params))
    rcols = codes[:, z: z + nrot]
    clear_e = ((rcols == CLEAR1).astype(np.int64) << np.arange(nrot, dtype=np.int64)).sum(axis=1)
    # every index array of the pass in one pinned upload: rotation GGSW rows and
    # exponents, then the tree levels' columns
    if dev_codes is not None:
        d_idx = dev_codes[:, z: z + nrot].contiguous()                       # CLEAR codes are < 0: skipped
        d_exps = torch.remainder(-(2 ** torch.arange(nrot, device=dev, dtype=torch.int64)), 2 * n)
        d_exps = d_exps.to(torch.int32).expand(B, nrot).contiguous()
        d_cols = [dev_codes[:, pos].contiguous() for pos in range(z)]
    else:
        d_idx, d_exps, d_cols = _upload_i32([np.where(rcols >= 0, rcols, -1), _rotation_exps(params, B, nrot, +1),
                                             codes[:, :z].T], dev)
    acc = _rotation_ladder(params, table, acc, rcols, +1, (d_idx, d_exps))    # X^{+2^w} (hw/lut.py:289)
    if clear_e.any():
        acc = monomial_gather(params, acc, clear_e)
    cur = acc.unsqueeze(1)
    for pos in range(z - 1, -1, -1):
        col = codes[:, pos]
        enc = col >= 0
        if enc.all():
            cur = _level(params, table, cur.contiguous(), d_cols[pos], inverse=True)
            continue
        mm = cur.shape[1]
        new = torch.zeros((B, 2 * mm, 2, n), dtype=torch.int32, device=dev)
        c0 = torch.as_tensor(np.nonzero(col == CLEAR0)[0], device=dev)
        c1 = torch.as_tensor(np.nonzero(col == CLEAR1)[0], device=dev)
        if c0.numel():
            new[c0, :mm] = cur[c0]
        if c1.numel():
            new[c1, mm:] = cur[c1]
        if enc.any():
            sel = torch.as_tensor(np.nonzero(enc)[0], device=dev)
            new[sel] = _level(params, table, cur[sel].contiguous(), _i32(col[enc], dev), inverse=True)
        cur = new
    return cur


def vp_codes(params: HeParams, codes, table: GgswNtt | None, lut_table: torch.Tensor, lut_idx):
    """Vertical packing (hw/lut.py:209-266) for B items.

    lut_table: device (T, 2^z, 2, N) tables; lut_idx: (B,) which table each item
    reads.  Returns the extracted LWE pieces as a device tensor (B, N+1) (b last)."""
    codes = np.asarray(codes, dtype=np.int64)
    lut_idx = np.asarray(lut_idx, dtype=np.int64)
    B, k = codes.shape
    z = tree_depth(k, params)
    n = params.n
    dev = lut_table.device
    # clear-prefix tree levels are pure index arithmetic (hw/lut.py:221-231)
    start = np.zeros(B, dtype=np.int64)
    length = np.full(B, max(1, 1 << z), dtype=np.int64)
    lvl = 0
    while lvl < z and (codes[:, lvl] < 0).all():
        length //= 2
        start += np.where(codes[:, lvl] == CLEAR1, length, 0)
        lvl += 1
    L = int(length[0]) if B else 1
    rows = (lut_idx[:, None] * lut_table.shape[1] + start[:, None] + np.arange(L)[None, :]).reshape(-1)
    cur = lut_table.reshape(-1, 2, n)[torch.as_tensor(rows, device=dev)].reshape(B, L, 2, n)
    for pos in range(lvl, z):
        col = codes[:, pos]
        enc = col >= 0
        half = cur.shape[1] // 2
        if enc.all():
            cur = _level(params, table, cur.contiguous(), _i32(col, dev), inverse=False)
            continue
        new = torch.empty((B, half, 2, n), dtype=torch.int32, device=dev)
        c0 = torch.as_tensor(np.nonzero(col == CLEAR0)[0], device=dev)
        c1 = torch.as_tensor(np.nonzero(col == CLEAR1)[0], device=dev)
        if c0.numel():
            new[c0] = cur[c0, :half]
        if c1.numel():
            new[c1] = cur[c1, half:]
        if enc.any():
            sel = torch.as_tensor(np.nonzero(enc)[0], device=dev)
            new[sel] = _level(params, table, cur[sel].contiguous(), _i32(col[enc], dev), inverse=False)
        cur = new
    acc = cur[:, 0].contiguous()
    nrot = len(rotate_weights(k, params))
    rcols = codes[:, z: z + nrot]
    clear_e = ((rcols == CLEAR1).astype(np.int64) << np.arange(nrot, dtype=np.int64)).sum(axis=1)
    acc = _rotation_ladder(params, table, acc, rcols, -1)                  # X^{-2^w} (hw/lut.py:258)
    if clear_e.any():
        acc = monomial_gather(params, acc, -clear_e)
    return tfhe.sample_extract_batch(params, acc)


# ---------------------------------------------------------------------------
# reference-shaped API over SelectorBit lists


def _codes_of(selectors: list[list[SelectorBit]], params: HeParams):
    """Code matrix + one device GGSW table for the distinct encrypted bits."""
    rows: dict[int, int] = {}
    cts: list[RgswCiphertext] = []
    codes = np.empty((len(selectors), len(selectors[0]) if selectors else 0), dtype=np.int64)
    for i, sel in enumerate(selectors):
        if len(sel) != codes.shape[1]:
            raise TfheError("selector vectors must share one arity")
        for j, s in enumerate(sel):
            if s.is_clear:
                codes[i, j] = CLEAR1 if s.bit else CLEAR0
            else:
                key = id(s.ct)
                if key not in rows:
                    rows[key] = len(cts)
                    cts.append(s.ct)
                codes[i, j] = rows[key]
    table = None
    if cts:
        stack = np.stack([np.asarray(c.data) for c in cts])
        # the FP64 FFT ladders wherever they apply (as he_train's "auto"), else the NTT;
        # full-precision gadgets have only the former (bit-identical where both exist)
        table = (tfhe.rgsw_to_fft(params, stack) if tfhe.ggsw_fft_bytes(params) > 0
                 else tfhe.rgsw_to_ntt(params, stack))
    return codes, table


def ivp_batch(selectors: list[list[SelectorBit]], payload, params: HeParams):
    """hw/lut.py:269-314: returns (B, max(1, 2^z), 2, N) uint32 rows (numpy)."""
    codes, table = _codes_of(selectors, params)
    return tfhe.to_host(ivp_codes(params, codes, table, np.asarray(payload)))


def vp_batch(selectors: list[list[SelectorBit]], luts: list, params: HeParams):
    """hw/lut.py:209-266: returns (lwe_a (B, N), lwe_b (B,)) uint32 (numpy)."""
    codes, table = _codes_of(selectors, params)
    lut_table = tfhe.to_device(np.stack([np.asarray(x) for x in luts]))
    out = tfhe.to_host(vp_codes(params, codes, table, lut_table, np.arange(len(luts))))
    return out[:, :-1], out[:, -1].copy()


def encode_lut(values, params: HeParams) -> EncryptedLut:
    """Pack 2^k public values mod p into trivial (noiseless) ciphertexts (hw/lut.py:86-97)."""
    values = np.asarray(values, dtype=np.int64)
    size = len(values)
    if size < 1 or size & (size - 1):
        raise TfheError("LUT size must be a power of two")
    n = params.n
    chunks = [values[i: i + n] for i in range(0, size, n)] if size >= n else [values]
    return EncryptedLut([tfhe.trivial_rlwe(c, params) for c in chunks], size.bit_length() - 1)


def decode_lut(lut: EncryptedLut, key: tfhe.SecretKey) -> np.ndarray:
    """Decrypt every entry (hw/lut.py:100-103, test helper)."""
    vals = np.concatenate([tfhe.dec_rlwe(c, key) for c in lut.polys])
    return vals[: 1 << lut.k]


def lut_add(a: EncryptedLut, b: EncryptedLut) -> EncryptedLut:
    """Entry-wise sum of equally shaped LUTs (hw/lut.py:106-110)."""
    if a.k != b.k or len(a.polys) != len(b.polys):
        raise TfheError("LUT geometries differ")
    return EncryptedLut([x + y for x, y in zip(a.polys, b.polys)], a.k)


def vertical_packing(bits: list[SelectorBit], lut: EncryptedLut) -> tfhe.LweCiphertext:
    """hw/lut.py:122-149: LWE of lut[m], m the index the selector bits encode (one
    item of vp_codes: CMUX tree, rotation ladder, extraction on the GPU)."""
    params = lut.params
    if len(bits) != lut.k:
        raise TfheError(f"selector arity {len(bits)} != LUT k {lut.k}")
    a, b = vp_batch([bits], [np.stack([np.asarray(c.data) for c in lut.polys])], params)
    return tfhe.LweCiphertext(params, a[0].astype(np.uint32), np.uint32(b[0]))


def inverse_vertical_packing(bits: list[SelectorBit], payload: RlweCiphertext) -> EncryptedLut:
    """hw/lut.py:152-189: deposit the payload's constant term at the selected entry
    (rotation ladder + CDEMUX tree on the GPU); every other entry encrypts zero."""
    rows = ivp_batch([bits], payload.data, payload.params)[0]
    return EncryptedLut([RlweCiphertext(payload.params, r) for r in rows], len(bits))


def cdemux(C: RgswCiphertext, d: RlweCiphertext) -> tuple[RlweCiphertext, RlweCiphertext]:
    """hw/lut.py:113-119."""
    lo, hi = tfhe.cdemux_batch(d.params, C.spectra(), np.asarray(d.data)[None])
    return RlweCiphertext(d.params, lo[0]), RlweCiphertext(d.params, hi[0])
