"""WiSARD training and inference over TFHE-encrypted data, on B200.

Mirror of the reference's `hewisard.hewnn` (`pkg/src/hewisard/hewnn.py`):
training deposits, per sample and RAM, an encrypted +1 at the (label,
address) entry of the RAM's row by inverse vertical packing of the payload
(0, q/p) (`hewnn.py:189-229`); a small IVP over the label bits accumulates
encrypted class counts (`hewnn.py:180-186`).  Rows are added by exact ring
addition, so sample order and batching cannot change the ciphertexts.

Differences in mechanics (not results): samples are processed in batches of
`batch` images whose RGSW bits share one device GGSW table, so every kernel
launch covers batch*k0 items; the model lives in device memory.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np
import torch

from . import lut, tfhe
from ._lib import TfheError
from .params import HeParams
from .tfhe import RgswCiphertext, RlweCiphertext
from .wnn import ClassCounts, IntegerWisardModel, WisardGeometry, permutation


class EncryptedSample:
    """One preprocessed sample encrypted bit by bit as RGSW (hw/hewnn.py:33-43).

    Reference constructor: `EncryptedSample(params, data_bits, label_bits=None)`
    with lists of RgswCiphertext (label bits LSB-first).  The batched GPU path
    keeps all s data bits then the label bits as ONE stacked (s + nl, 2l, 2, N)
    uint32 array -- numpy, a pinned host tensor or a device tensor -- built by
    `from_stack` (or lazily from the lists); the list views are materialised on
    demand from the stack."""

    def __init__(self, params: HeParams, data_bits: Sequence[RgswCiphertext],
                 label_bits: Sequence[RgswCiphertext] | None = None):
        self.params = params
        self._data = list(data_bits)
        self._labels = None if label_bits is None else list(label_bits)
        self._stack = None
        self._s = len(self._data)
        self._nl = 0 if self._labels is None else len(self._labels)

    @classmethod
    def from_stack(cls, params: HeParams, stack, s: int, n_label_bits: int = 0) -> "EncryptedSample":
        obj = cls.__new__(cls)
        obj.params, obj._stack, obj._s, obj._nl = params, stack, int(s), int(n_label_bits)
        obj._data = obj._labels = None
        return obj

    @property
    def s(self) -> int:
        return self._s

    @property
    def n_label_bits(self) -> int:
        return self._nl

    @property
    def rgsw(self):
        """(s + nl, 2l, 2, N) stacked words (the batched path's input)."""
        if self._stack is None:
            g = self.params.gadget
            rows = [np.asarray(c.data, dtype=np.uint32) for c in self._data + (self._labels or [])]
            self._stack = (np.stack(rows) if rows else
                           np.zeros((0, 2 * g.levels, 2, self.params.n), dtype=np.uint32))
        return self._stack

    def _host_rows(self, lo: int, hi: int) -> list[RgswCiphertext]:
        st = self._stack
        if isinstance(st, SeededRgsw):
            st = st.expand()
        host = st[lo:hi] if isinstance(st, np.ndarray) else tfhe.to_host(st[lo:hi])
        return [RgswCiphertext(self.params, np.asarray(host[i], dtype=np.uint32)) for i in range(hi - lo)]

    @property
    def data_bits(self) -> list[RgswCiphertext]:
        if self._data is None:
            self._data = self._host_rows(0, self._s)
        return self._data

    @property
    def label_bits(self) -> list[RgswCiphertext] | None:
        """The label's RGSW bits (LSB-first), None for an unlabelled sample."""
        if self._labels is None and self._stack is not None and self._nl:
            self._labels = self._host_rows(self._s, self._s + self._nl)
        return self._labels

    labels = label_bits       # round-1 name

    def __repr__(self) -> str:
        return f"EncryptedSample(s={self._s}, label_bits={self._nl}, params={self.params.name})"


@dataclass
class HomWisardModel:
    """Encrypted integer WiSARD: k0 x k1 RLWE rows plus encrypted class counts
    (hw/hewnn.py:46-64), resident on the device."""

    geometry: WisardGeometry
    params: HeParams
    rams: torch.Tensor            # int32 (k0, k1, 2, N)
    counts_ct: torch.Tensor       # int32 (2, N)

    @classmethod
    def zeros(cls, geometry: WisardGeometry, params: HeParams) -> "HomWisardModel":
        k1 = model_row_polys(geometry, params)
        dev = tfhe._device()
        return cls(geometry, params,
                   torch.zeros((geometry.k0, k1, 2, params.n), dtype=torch.int32, device=dev),
                   torch.zeros((2, params.n), dtype=torch.int32, device=dev))

    def copy(self) -> "HomWisardModel":
        return HomWisardModel(self.geometry, self.params, self.rams.clone(), self.counts_ct.clone())


def model_row_polys(geometry: WisardGeometry, params: HeParams) -> int:
    """RLWE ciphertexts per RAM row: max(1, 2^(label_bits + a) / N) (hw/hewnn.py:95-97)."""
    return max(1, (1 << geometry.selector_bits) // params.n)


def _check_geometry(geometry: WisardGeometry, params: HeParams):
    if geometry.p != params.p:
        raise TfheError(f"geometry counter modulus {geometry.p} != params p {params.p}")


# ---------------------------------------------------------------------------
# encryption (client side)


class DeviceKey:
    """A secret key's NTT image on the device, for GPU-side key products.

    Remembers what it was built from (parameters, device, a digest of the key
    coefficients) so a cached image is never used for a different key."""

    def __init__(self, key: tfhe.SecretKey):
        params = key.params
        self.params = params
        self.device = torch.cuda.current_device()
        self.digest = _key_digest(key)
        s = tfhe.to_device(key.s)
        cp = _lib_params(params)
        self.ntt = torch.empty((2, params.n), dtype=torch.int32, device=s.device)
        tfhe._lib.check(tfhe._lib.load().hwb_poly_to_ntt(cp, tfhe._ptr(s), tfhe._ptr(self.ntt), 1,
                                                         tfhe._stream()))

    def matches(self, key: tfhe.SecretKey) -> bool:
        return (self.params == key.params and self.device == torch.cuda.current_device()
                and self.digest == _key_digest(key))


def _key_digest(key: tfhe.SecretKey) -> bytes:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(key.s, dtype=np.uint32).tobytes()).digest()


def _lib_params(params):
    import ctypes
    return ctypes.byref(tfhe._lib.c_params(params))


def _device_key(key: tfhe.SecretKey) -> DeviceKey:
    """The key's device image, cached on the key object itself (not by id(), which
    CPython reuses) and rebuilt when the key, its parameters or the device change."""
    dk = getattr(key, "_device_key", None)
    if dk is None or not dk.matches(key):
        dk = DeviceKey(key)
        object.__setattr__(key, "_device_key", dk)
    return dk


def enc_rgsw_batch_device(ms, key: tfhe.SecretKey, rng, seeded: bool = False, device_noise: bool = False):
    """enc_rgsw_batch (hw/tfhe.py:246-263) with the uniform half AND the key product on
    the GPU: the host claims the a-words of rng's Philox stream without generating
    them (tfhe.philox_take), draws only the normals e, and the GPU regenerates a
    (hwb_philox_rgsw) and forms b = a s + e + m g.  Same stream as the host version;
    returns the device tensor (B, 2l, 2, N), bit-identical to tfhe.enc_rgsw_batch.
    seeded=True returns (b rows on the device (B 2l, N), hwb_philox) instead: the
    compressed wire form the server expands with hwb_philox_rgsw."""
    ms = np.asarray(ms, dtype=np.int64)
    params = key.params
    g = params.gadget
    rows = 2 * g.levels
    B = len(ms)
    N = params.n
    if np.any((ms != 0) & (ms != 1)):
        raise tfhe.EncodingError("RGSW messages are bits")
    st = tfhe.philox_take(rng, B * rows * N)                   # a: claimed, not drawn
    dev = tfhe._device()
    if device_noise:
        # large-scale runs: the normals drawn on the GPU from a generator seeded by the
        # host stream -- a valid encryption, but NOT the reference's rint(rng.normal)
        # stream
        gen = torch.Generator(device=dev)
        gen.manual_seed(int(rng.integers(0, 1 << 62)))
        e = torch.round(torch.randn((B, rows, N), generator=gen, device=dev, dtype=torch.float64) * params.sigma)
        e = e.to(torch.int64).bitwise_and(0xFFFFFFFF)
        e = torch.where(e >= 1 << 31, e - (1 << 32), e).to(torch.int32)
    else:
        e = tfhe.gaussian_u32(rng, params.sigma, (B, rows, N))
    out = torch.empty((B, rows, 2, N), dtype=torch.int32, device=dev)
    if B == 0:
        return (out.view(0, N), st, out[:, :0, 0, 0]) if seeded else out
    a_d = tfhe.philox_rgsw(st, B * rows, N, pair=False)        # (B rows, N) on the GPU
    e_d = tfhe.to_device(e)
    b_d = torch.empty_like(a_d)
    dk = _device_key(key)
    cp = _lib_params(params)
    L = tfhe._lib.load()
    tfhe._lib.check(L.hwb_key_mul(cp, tfhe._ptr(dk.ntt), tfhe._ptr(a_d), tfhe._ptr(e_d), tfhe._ptr(b_d),
                                  B * rows, tfhe._stream()))
    out[:, :, 0] = a_d.view(B, rows, N)
    out[:, :, 1] = b_d.view(B, rows, N)
    bits = torch.as_tensor(ms, dtype=torch.int32).to(dev)
    tfhe._lib.check(L.hwb_rgsw_add_gadget(cp, tfhe._ptr(out), tfhe._ptr(bits), B, tfhe._stream()))
    if seeded:
        # wire form: the b rows, the Philox state of the a draw, and the l words per
        # RGSW whose a[0] carries the gadget term (they cannot be regenerated)
        return out[:, :, 1].reshape(B * rows, N).contiguous(), st, out[:, g.levels:, 0, 0].contiguous()
    return out


class SeededRgsw:
    """A sample's RGSW stack in compressed (seeded) form: only the b halves
    (R = n_rgsw 2l rows of N words, pinned host or device) plus, per encryption
    call, the Philox state its a-words were drawn from.  expand() rebuilds the
    full (n_rgsw, 2l, 2, N) stack on the device, bit-identical (hwb_philox_rgsw):
    half the bytes of a plain stack cross PCIe."""

    def __init__(self, params: HeParams, b_rows: torch.Tensor, a0: torch.Tensor, segments: list):
        self.params = params
        self.b = b_rows                                  # (R, N) int32
        self.a0 = a0                                     # (R / 2l, l): gadget-carrying a[l+t][0] words
        self.segments = segments                         # [(hwb_philox, row0, rows)]
        g = params.gadget
        self.shape = (b_rows.shape[0] // (2 * g.levels), 2 * g.levels, 2, params.n)
        self.is_cuda = False

    def numel(self) -> int:
        return int(np.prod(self.shape))

    def expand(self, out: torch.Tensor | None = None, b_dev: torch.Tensor | None = None,
               a0_dev: torch.Tensor | None = None) -> torch.Tensor:
        """Full stack on the device; b_dev / a0_dev: the wire words already on the device."""
        N = self.params.n
        lv = self.params.gadget.levels
        if out is None:
            out = torch.empty(self.shape, dtype=torch.int32, device=tfhe._device())
        bd = b_dev if b_dev is not None else tfhe.to_device(self.b)
        ad = a0_dev if a0_dev is not None else tfhe.to_device(self.a0)
        flat = out.view(-1, 2, N)
        for st, r0, rows in self.segments:
            g0 = r0 // (2 * lv)
            tfhe.philox_rgsw(st, rows, N, b_rows=bd[r0: r0 + rows], out=flat[r0: r0 + rows],
                             a0fix=ad[g0: g0 + rows // (2 * lv)], levels=lv)
        return out


def encrypt_sample_seeded(bits: Sequence[int], label: int | None, key: tfhe.SecretKey, rng, *,
                          label_bits: int = 0, pin: bool = True) -> "EncryptedSample":
    """encrypt_sample (hw/hewnn.py:109-119) in the compressed wire form: same RNG stream
    (the data batch, then the label batch), but the sample carries only b halves and
    Philox states (host pinned), expanded on the server's GPU."""
    P = key.params
    segs, parts, row = [], [], 0
    rows_per = 2 * P.gadget.levels
    batches = [np.asarray(bits, dtype=np.int64)]
    if label is not None:
        if label >= (1 << label_bits):
            raise TfheError(f"label {label} does not fit in {label_bits} bits")
        batches.append(np.array([(label >> i) & 1 for i in range(label_bits)], dtype=np.int64))
    a0s = []
    for ms in batches:
        b_d, st, a0 = enc_rgsw_batch_device(ms, key, rng, seeded=True)
        segs.append((st, row, len(ms) * rows_per))
        parts.append(b_d)
        a0s.append(a0)
        row += len(ms) * rows_per
    b, a0 = torch.cat(parts).cpu(), torch.cat(a0s).cpu()
    if pin:
        b, a0 = b.pin_memory(), a0.pin_memory()
    lb = label_bits if label is not None else 0
    return EncryptedSample.from_stack(P, SeededRgsw(P, b, a0, segs), len(bits), lb)


def encrypt_sample(bits: Sequence[int], label: int | None, key: tfhe.SecretKey, rng, *,
                   label_bits: int = 0, device: bool = True, device_noise: bool = False) -> EncryptedSample:
    """Encrypt preprocessed input bits and the label (hw/hewnn.py:109-119).

    RNG stream as the reference: the data batch, then the label batch.
    device_noise=True draws the normals on the GPU (a valid encryption at GPU speed for
    large synthetic workloads, not the reference's RNG stream)."""
    if device_noise:
        def enc(ms, key, rng):
            return enc_rgsw_batch_device(ms, key, rng, device_noise=True)
    else:
        enc = enc_rgsw_batch_device if device else _enc_rgsw_host
    data = enc(np.asarray(bits, dtype=np.int64), key, rng)
    lb = 0
    if label is not None:
        if label >= (1 << label_bits):
            raise TfheError(f"label {label} does not fit in {label_bits} bits")
        lab = enc(np.array([(label >> i) & 1 for i in range(label_bits)], dtype=np.int64), key, rng)
        data = torch.cat([data, lab]) if device else np.concatenate([data, lab])
        lb = label_bits
    return EncryptedSample.from_stack(key.params, data, len(bits), lb)


def _enc_rgsw_host(ms, key, rng) -> np.ndarray:
    if len(ms) == 0:
        g = key.params.gadget
        return np.zeros((0, 2 * g.levels, 2, key.params.n), dtype=np.uint32)
    return np.stack([c.data for c in tfhe.enc_rgsw_batch(ms, key, rng)])


# ---------------------------------------------------------------------------
# selector construction (hw/hewnn.py:134-173)


def _selector_template(geometry: WisardGeometry, params: HeParams, *, clear_label: int | None = None):
    """(k0, k) codes relative to a sample's first RGSW row.

    Positions follow the canonical tree-MSB / rotate-LSB order
    (hw/hewnn.py:134-150); address bit w of RAM j is permuted input bit
    perm[j*a + w] (hw/wnn.py:189-196), zero padding past s is a clear 0
    (hw/hewnn.py:164-166); label bit i is row s + i, or the clear bits of
    `clear_label` (inference, hw/hewnn.py:303-304)."""
    k = geometry.selector_bits
    z = lut.tree_depth(k, params)
    a, s = geometry.a, geometry.s
    perm = permutation(geometry.r, geometry.s)
    weights = np.array([k - 1 - i for i in range(z)] + lut.rotate_weights(k, params), dtype=np.int64)
    j = np.arange(geometry.k0, dtype=np.int64)[:, None]
    idx = j * a + weights[None, :]                                  # address-bit input index
    addr = np.where(idx < s, perm[np.minimum(idx, s - 1)], lut.CLEAR0)
    lw = weights - a                                                # label-bit number (w >= a)
    if clear_label is None:
        lab = np.broadcast_to(s + lw, addr.shape)
    else:
        bit = (clear_label >> np.maximum(lw, 0)) & 1
        lab = np.broadcast_to(np.where(bit == 1, lut.CLEAR1, lut.CLEAR0), addr.shape)
    return np.where(weights[None, :] < a, addr, lab).astype(np.int64)


def _shift(codes: np.ndarray, base: int) -> np.ndarray:
    return np.where(codes >= 0, codes + base, codes)


_PAYLOADS: dict = {}


def _payload(params: HeParams) -> torch.Tensor:
    """Trivial RLWE (0, q/p) payload of the IVP, cached on the device."""
    key = (params, torch.cuda.current_device())
    if key not in _PAYLOADS:
        _PAYLOADS[key] = tfhe.to_device(tfhe.trivial_rlwe(1, params).data)
    return _PAYLOADS[key]


# ---------------------------------------------------------------------------
# training


_TRACE = None          # list of (label, cuda.Event) when tracing the pipeline (tools/)


def _ev(stream=None):
    e = torch.cuda.Event(enable_timing=True)
    e.record(stream)
    return e


class _StageRing:
    """Two device staging slots for the RGSW stacks of consecutive chunks, allocated
    once per training call (two large blocks instead of one allocation per sample):
    chunk k's host->device copy lands in slot k % 2 on the copy stream, and waits
    for the GPU to have consumed chunk k-2 from that slot (its table conversion)."""

    def __init__(self, words: int, bwords: int = 0):
        dev = tfhe._device()
        self.slots = [torch.empty(words, dtype=torch.int32, device=dev) for _ in range(2)]
        # seeded samples (SeededRgsw): their b halves land here, then expand into the slot
        self.bslots = [torch.empty(bwords, dtype=torch.int32, device=dev) for _ in range(2)] if bwords else None
        self.free = [None, None]        # main-stream event: the slot's last reader is done
        self.k = 0

    def take(self) -> int:
        slot = self.k % 2
        self.k += 1
        return slot


def _stack_to_device(stack) -> torch.Tensor:
    return stack.expand() if isinstance(stack, SeededRgsw) else tfhe.to_device(stack)


class _Staged:
    """A chunk's host RGSW stacks copied to the device on a side stream, so the
    H2D of chunk k+1 overlaps the ladders of chunk k (pinned host tensors)."""

    _copy_stream = None

    def __init__(self, samples: list[EncryptedSample], ring: _StageRing | None = None):
        self.samples = samples
        self.dev: list | None = None
        self.event = None
        self.ring, self.slot = ring, None
        self.pending: list = []          # seeded samples: expanded on the main stream in tensors()
        if not any(isinstance(s.rgsw, (np.ndarray, SeededRgsw)) or
                   (isinstance(s.rgsw, torch.Tensor) and not s.rgsw.is_cuda) for s in samples):
            return                                          # already device-resident
        if _Staged._copy_stream is None:
            _Staged._copy_stream = torch.cuda.Stream(device=tfhe._device())
        cs = _Staged._copy_stream
        need = sum(int(np.prod(s.rgsw.shape)) for s in samples)
        bneed = sum(int(s.rgsw.b.numel() + s.rgsw.a0.numel()) for s in samples if isinstance(s.rgsw, SeededRgsw))
        if ring is not None and need <= ring.slots[0].numel() and (
                bneed == 0 or (ring.bslots is not None and bneed <= ring.bslots[0].numel())):
            self.slot = ring.take()
            if ring.free[self.slot] is not None:
                cs.wait_event(ring.free[self.slot])         # chunk k-2 has left the slot
        else:
            self.ring = None
            cs.wait_stream(torch.cuda.current_stream())     # buffers freed on the main stream
        with torch.cuda.stream(cs):
            if _TRACE is not None:
                _TRACE.append(("copy_start", _ev(cs)))
            if self.ring is None:
                self.dev = [_stack_to_device(s.rgsw) for s in samples]
            else:
                buf, off, self.dev = ring.slots[self.slot], 0, []
                boff = 0
                for smp in samples:
                    src = smp.rgsw
                    if isinstance(src, SeededRgsw):
                        # half the bytes over PCIe: b rows, then the GPU regenerates a
                        nb, na = src.b.numel(), src.a0.numel()
                        bd = ring.bslots[self.slot][boff: boff + nb].view(src.b.shape)
                        bd.copy_(src.b, non_blocking=True)
                        ad = ring.bslots[self.slot][boff + nb: boff + nb + na].view(src.a0.shape)
                        ad.copy_(src.a0, non_blocking=True)
                        boff += nb + na
                        n = src.numel()
                        dst = buf[off: off + n].view(src.shape)
                        # the a-regeneration runs on the MAIN stream (tensors()), so the copy
                        # stream only moves bytes and the next chunk's H2D is not delayed
                        self.pending.append((src, dst, bd, ad))
                        self.dev.append(dst)
                        off += n
                        continue
                    if isinstance(src, np.ndarray):
                        src = torch.from_numpy(np.ascontiguousarray(src, dtype=np.uint32).view(np.int32))
                    src = src.view(torch.int32) if src.dtype == torch.uint32 else src
                    n = src.numel()
                    dst = buf[off: off + n].view(src.shape)
                    dst.copy_(src, non_blocking=True)
                    self.dev.append(dst)
                    off += n
            self.event = torch.cuda.Event(enable_timing=_TRACE is not None)
            self.event.record(cs)
            if _TRACE is not None:
                _TRACE.append(("copy_end", self.event))

    def tensors(self) -> list:
        if self.dev is None:
            return [_stack_to_device(s.rgsw) for s in self.samples]
        main = torch.cuda.current_stream()
        main.wait_event(self.event)
        for src, dst, bd, ad in self.pending:
            src.expand(dst, bd, ad)
        self.pending = []
        if self.ring is None:
            for t in self.dev:
                t.record_stream(main)                       # allocator: used on the main stream
        return self.dev

    def release(self):
        """The main stream has enqueued the last reader of this chunk's slot."""
        if self.ring is not None:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream())
            self.ring.free[self.slot] = ev


def _use_fft(params: HeParams, ladder: str) -> bool:
    """Vertical-packing ladders on the FP64 FFT path ("auto": wherever it applies,
    N = 1024 and 2048) or the two-prime NTT path; both are bit-identical."""
    if ladder not in ("auto", "fft", "ntt"):
        raise TfheError(f"unknown ladder {ladder!r}")
    ok = tfhe.ggsw_fft_bytes(params) > 0
    if ladder == "fft" and not ok:
        raise TfheError("the FFT ladder does not apply to these parameters (N = 1024 or 2048, narrow gadgets)")
    return ok and ladder != "ntt"


def _table_bytes(params: HeParams, rows: int, ladder: str = "auto") -> int:
    """Device bytes of a GGSW table of `rows` RGSW ciphertexts (FFT or NTT domain)."""
    cp = _lib_params(params)
    L = tfhe._lib.load()
    per = L.hwb_ggsw_fft_bytes(cp) if _use_fft(params, ladder) else L.hwb_ggsw_ntt_words(cp) * 4
    return rows * int(per)


def _stack_table(params: HeParams, samples: list[EncryptedSample], staged: _Staged | None = None,
                 ladder: str = "auto", arena: torch.Tensor | None = None):
    """One device GGSW table (NTT or FFT domain) holding every sample's RGSW rows,
    each sample transformed straight into its slice (no stacking copy).  `arena`
    (uint8, reused across a training call's chunks) holds the table when given."""
    import ctypes
    cp = _lib_params(params)
    L = tfhe._lib.load()
    rows = [int(s.rgsw.shape[0]) for s in samples]
    fft = _use_fft(params, ladder)
    nbytes = L.hwb_ggsw_fft_bytes(cp) if fft else L.hwb_ggsw_ntt_words(cp) * 4
    total = sum(rows) * nbytes
    if arena is not None and arena.numel() >= total:
        raw = arena[:total]
    else:
        raw = torch.empty(total, dtype=torch.uint8, device=tfhe._device())
    if fft:
        table = raw
        conv = L.hwb_ggsw_to_fft
    else:
        table = raw.view(torch.int32).view(sum(rows), nbytes // 4)
        conv = L.hwb_ggsw_to_ntt
    st = staged or _Staged(samples)
    srcs = st.tensors()
    off = 0
    for src, r in zip(srcs, rows):
        dst = ctypes.c_void_p(table.data_ptr() + off * nbytes)
        tfhe._lib.check(conv(cp, tfhe._ptr(src), dst, r, tfhe._stream()))
        off += r
    st.release()
    return tfhe.GgswFft(params, table, sum(rows)) if fft else tfhe.GgswNtt(params, table)


def he_count_labels(label_bits: Sequence[RgswCiphertext], counts_ct, params: HeParams):
    """hw/hewnn.py:180-186: add one to the encrypted per-class counter selected by
    the label bits (an IVP of the payload (0, q/p) over the label bits alone).
    Returns a new (2, N) ciphertext (numpy in -> numpy out, device -> device)."""
    sel = [[lut.SelectorBit.enc(c) for c in label_bits]]
    codes, table = lut._codes_of(sel, params)
    row = lut.ivp_codes(params, codes, table, _payload(params))[0, 0]          # (2, N) on the device
    if isinstance(counts_ct, torch.Tensor):
        return lut.accumulate_(counts_ct.to(row.device).clone().contiguous(), row)
    return (np.asarray(counts_ct, dtype=np.uint32) + tfhe.to_host(row)).astype(np.uint32)


def he_count_labels_batch(params: HeParams, counts_ct: torch.Tensor, table, label_rows: np.ndarray,
                          dev_rows: torch.Tensor | None = None):
    """hw/hewnn.py:180-186 for several samples: counts += IVP(label bits, (0, q/p))."""
    rows = lut.ivp_codes(params, label_rows, table, _payload(params), dev_rows)     # (I, 1, 2, N)
    lut.accumulate_rows_(counts_ct, rows)
    return counts_ct


def he_train(samples: Iterable[EncryptedSample], geometry: WisardGeometry, params: HeParams,
             model: HomWisardModel | None = None, threads: int = 1, batch: int = 16,
             ladder: str = "auto") -> HomWisardModel:
    """Homomorphic integer WiSARD training (hw/hewnn.py:189-229); pass an
    existing model to continue training.  `threads` is accepted for API
    compatibility (the GPU batches `batch` samples per launch instead)."""
    _check_geometry(geometry, params)
    if model is None:
        model = HomWisardModel.zeros(geometry, params)
    if model.geometry != geometry or model.params != params:
        raise TfheError("model geometry/params mismatch")
    tmpl = _selector_template(geometry, params)
    # a chunk's selector codes and label rows depend only on the sample's slot in
    # the chunk: build them once for a full chunk and upload them now, before
    # the staged RGSW transfers start (no host->device copy inside the pipeline)
    stride = geometry.s + geometry.label_bits
    k0 = geometry.k0
    all_codes = np.concatenate([_shift(tmpl, i * stride) for i in range(batch)])
    all_labels = np.array([[i * stride + geometry.s + b for b in range(geometry.label_bits)]
                           for i in range(batch)], dtype=np.int64).reshape(batch, geometry.label_bits)
    d_codes, d_labels = lut._upload_i32([all_codes, all_labels], tfhe._device())
    _payload(params)
    # one table buffer for every chunk (the ladders of chunk k precede chunk k+1's
    # conversion on the same stream) and, for host samples, two staging slots
    # (sized by the first chunk, the largest)
    arena = ring = None

    def run(chunk: list[EncryptedSample], staged: _Staged):
        nonlocal arena
        if arena is None:
            nbytes = _table_bytes(params, sum(int(x.rgsw.shape[0]) for x in chunk), ladder)
            arena = torch.empty(nbytes, dtype=torch.uint8, device=tfhe._device())
        table = _stack_table(params, chunk, staged, ladder, arena)
        I = len(chunk)
        rows = lut.ivp_codes(params, all_codes[: I * k0], table, _payload(params),
                             d_codes[: I * k0])                              # (I*k0, k1, 2, N)
        lut.accumulate_rows_(model.rams, rows)                             # hw/hewnn.py:213
        he_count_labels_batch(params, model.counts_ct, table, all_labels[:I], d_labels[:I])

    def check(sample):
        if sample.s != geometry.s:
            raise TfheError(f"sample has {sample.s} bits, geometry wants {geometry.s}")
        if sample.n_label_bits != geometry.label_bits:
            raise TfheError("training samples need encrypted label bits"
                            if not sample.n_label_bits else
                            f"sample has {sample.n_label_bits} label bits, geometry wants {geometry.label_bits}")

    # one chunk in flight: chunk k+1's H2D is enqueued on the copy stream before
    # chunk k's ladders, so host->device traffic overlaps the GPU work
    def stage(chunk):
        nonlocal ring
        if ring is None and any(not (isinstance(x.rgsw, torch.Tensor) and x.rgsw.is_cuda) for x in chunk):
            ring = _StageRing(sum(int(np.prod(x.rgsw.shape)) for x in chunk),
                              sum(int(x.rgsw.b.numel() + x.rgsw.a0.numel()) for x in chunk
                                  if isinstance(x.rgsw, SeededRgsw)))
        return _Staged(chunk, ring)

    for chunk, staged in _chunks_staged(samples, batch, check, stage):
        if _TRACE is not None:
            _TRACE.append(("run_start", _ev()))
        run(chunk, staged)
        if _TRACE is not None:
            _TRACE.append(("run_end", _ev()))
    return model


def _chunks_staged(samples: Iterable[EncryptedSample], batch: int, check=None, stage=None):
    """Yield (chunk, staged) with the next chunk's H2D already enqueued."""
    stage = stage or _Staged
    pending = None
    chunk: list[EncryptedSample] = []
    for sample in samples:
        if check:
            check(sample)
        chunk.append(sample)
        if len(chunk) == batch:
            nxt = (chunk, stage(chunk))
            chunk = []
            if pending is not None:
                yield pending
            pending = nxt
    if chunk:
        nxt = (chunk, stage(chunk))
        if pending is not None:
            yield pending
        pending = nxt
    if pending is not None:
        yield pending


def he_train_multi(samples: Iterable[EncryptedSample], geometries: Sequence[WisardGeometry], params: HeParams,
                   batch: int = 16) -> list[HomWisardModel]:
    """One model per permutation seed in a single streaming pass (hw/hewnn.py:232-261):
    every sample's IVP items for all geometries run in the same launches; the
    models are bit-identical to separate he_train runs."""
    base = geometries[0]
    for g in geometries:
        if (g.s, g.l, g.a, g.p) != (base.s, base.l, base.a, base.p):
            raise TfheError("multi-seed training requires geometries differing only in r")
        _check_geometry(g, params)
    models = [HomWisardModel.zeros(g, params) for g in geometries]
    tmpls = [_selector_template(g, params) for g in geometries]
    k0 = base.k0
    stride = base.s + base.label_bits
    chunk: list[EncryptedSample] = []

    def flush():
        if not chunk:
            return
        table = _stack_table(params, chunk)
        codes = np.concatenate([_shift(t, i * stride) for i in range(len(chunk)) for t in tmpls])
        rows = lut.ivp_codes(params, codes, table, _payload(params))       # (I*G*k0, k1, 2, N)
        rows = rows.reshape(len(chunk), len(geometries), k0, *rows.shape[1:])
        for gi, m in enumerate(models):
            lut.accumulate_rows_(m.rams, rows[:, gi].contiguous())
        label_rows = np.array([[i * stride + base.s + b for b in range(base.label_bits)]
                               for i in range(len(chunk))], dtype=np.int64)
        cnt = torch.zeros_like(models[0].counts_ct)
        he_count_labels_batch(params, cnt, table, label_rows)
        for m in models:
            lut.accumulate_(m.counts_ct, cnt)
        chunk.clear()

    for sample in samples:
        if sample.n_label_bits != base.label_bits:
            raise TfheError("training samples need encrypted label bits")
        chunk.append(sample)
        if len(chunk) == batch:
            flush()
    flush()
    return models


def decrypt_sample(sample: EncryptedSample, key: tfhe.SecretKey) -> tuple[list[int], int | None]:
    """hw/hewnn.py:122-130 (client side)."""
    bits = [tfhe.dec_rgsw(c, key) for c in sample.data_bits]
    labs = sample.label_bits
    if labs is None:
        return bits, None
    return bits, sum(tfhe.dec_rgsw(c, key) << i for i, c in enumerate(labs))


def he_train_sharded(samples: Sequence[EncryptedSample], geometry: WisardGeometry, params: HeParams,
                     rank: int, world: int, group=None, batch: int = 16) -> HomWisardModel:
    """Multi-GPU training: rank trains the stripe samples[rank::world] (the
    reference's thread stripes, hw/hewnn.py:216-229) and the partial models are
    summed mod 2^32 across ranks -- bit-identical to he_train on all samples."""
    from . import distributed
    model = he_train(distributed.stripe(list(samples), rank, world), geometry, params, batch=batch)
    if world > 1:
        distributed.merge_models_(model.rams, model.counts_ct, group)
    return model


def he_merge(m1: HomWisardModel, m2: HomWisardModel) -> HomWisardModel:
    """Federated merge: entry-wise RLWE addition (hw/hewnn.py:264-271)."""
    if m1.geometry != m2.geometry:
        raise TfheError("cannot merge models with different geometry or seed")
    if m1.params != m2.params:
        raise TfheError("cannot merge models with different parameters")
    out = m1.copy()
    lut.accumulate_(out.rams, m2.rams)
    lut.accumulate_(out.counts_ct, m2.counts_ct)
    return out


# ---------------------------------------------------------------------------
# homomorphic inference (PD-act, hw/hewnn.py:278-320)


@dataclass
class ScorePack:
    """PD-act output: packed raw scores plus encrypted class counts (hw/hewnn.py:67-78).
    Coefficient i*k0 + j (chunked over RLWEs of N coefficients) holds the
    class-i, RAM-j counter lookup."""

    geometry: WisardGeometry
    params: HeParams
    packed: np.ndarray            # (ceil(l*k0/N), 2, N)
    counts_ct: np.ndarray         # (2, N)


@dataclass
class FinalizeResult:
    prediction: int
    scores: np.ndarray
    raw: np.ndarray
    counts: ClassCounts
    noise_max: int
    noise_margin: int

    @property
    def noise_ok(self) -> bool:
        return self.noise_max < self.noise_margin


def vp_lookups(model: HomWisardModel, samples: Sequence[EncryptedSample], ladder: str = "auto") -> torch.Tensor:
    """Every (sample, class, RAM) counter lookup of PD-act inference (hw/hewnn.py:278-311):
    vertical packing with clear label bits and the sample's encrypted address bits.
    Returns the extracted LWEs under S1, (S * l * k0, N+1) on the device, ordered
    (sample, class, RAM)."""
    geometry, params = model.geometry, model.params
    for smp in samples:
        if smp.s != geometry.s:
            raise TfheError(f"sample has {smp.s} bits, geometry wants {geometry.s}")
        if smp.params != params:
            raise TfheError("sample parameter set differs from the model's")
    l, k0 = geometry.l, geometry.k0
    tmpl = np.concatenate([_selector_template(geometry, params, clear_label=i) for i in range(l)])
    strides = np.cumsum([0] + [int(np.asarray(smp.rgsw.shape[0])) for smp in samples])
    codes = np.concatenate([_shift(tmpl, int(strides[i])) for i in range(len(samples))])
    lut_idx = np.tile(np.tile(np.arange(k0), l), len(samples))
    table = _stack_table(params, list(samples), ladder=ladder)
    return lut.vp_codes(params, codes, table, model.rams, lut_idx)


def he_infer_pd_batch(model: HomWisardModel, samples: Sequence[EncryptedSample],
                      ksk: tfhe.PackingKeySwitchKey, ladder: str = "auto") -> list[ScorePack]:
    """he_infer_pd (hw/hewnn.py:278-320) for several samples in one pass: every
    (sample, class, RAM) triple is one vertical-packing item (clear label bits,
    encrypted address bits), then each sample's l*k0 extracted LWEs are packed."""
    geometry, params = model.geometry, model.params
    n = params.n
    l, k0 = geometry.l, geometry.k0
    total = l * k0
    lwe = vp_lookups(model, samples, ladder)                               # (S*l*k0, N+1)
    n_ct = -(-total // n)
    S = len(samples)
    a_st = torch.zeros((S * n_ct, n, n), dtype=torch.int32, device=lwe.device)
    b_p = torch.zeros((S * n_ct, n), dtype=torch.int32, device=lwe.device)
    for si in range(S):
        for t in range(n_ct):
            lo, hi = si * total + t * n, si * total + min(total, (t + 1) * n)
            a_st[si * n_ct + t, : hi - lo] = lwe[lo:hi, :n]
            b_p[si * n_ct + t, : hi - lo] = lwe[lo:hi, n]
    packed = tfhe.to_host(tfhe.pack_batch(a_st, b_p, ksk)).reshape(S, n_ct, 2, n)
    cc = tfhe.to_host(model.counts_ct)
    return [ScorePack(geometry, params, packed[si], cc.copy()) for si in range(S)]


def he_infer_pd(model: HomWisardModel, sample: EncryptedSample, ksk: tfhe.PackingKeySwitchKey) -> ScorePack:
    """Score every (class, RAM) pair and pack the results (hw/hewnn.py:278-320)."""
    return he_infer_pd_batch(model, [sample], ksk)[0]


def client_finalize(pack: ScorePack, key: tfhe.SecretKey, activation, *, balance: bool = False) -> FinalizeResult:
    """Decrypt, rescale, activate and argmax (hw/hewnn.py:329-345), on the client."""
    from . import wnn
    geometry, params = pack.geometry, pack.params
    raw_flat, noise_max = [], 0
    delta = params.delta
    for t in range(pack.packed.shape[0]):
        ct = RlweCiphertext(params, pack.packed[t])
        phase = tfhe.phase_rlwe(ct, key).astype(np.int64)
        raw_flat.append(tfhe.decode_phase(phase, params))
        err = (phase + delta // 2) % delta - delta // 2
        noise_max = max(noise_max, int(np.abs(err).max()))
    raw = np.concatenate(raw_flat)[: geometry.l * geometry.k0].reshape(geometry.l, geometry.k0)
    counts = decrypt_counts(pack.counts_ct, params, geometry.l, key)
    pred = wnn.predict_from_lookups(raw, activation, counts if balance else None)
    scores = wnn.scores_from_lookups(raw, activation, counts if balance else None)
    return FinalizeResult(pred, scores, raw, counts, noise_max, delta // 2)


# ---------------------------------------------------------------------------
# client side: decryption of a trained model (oracle bridge, hw/hewnn.py:352-365)


def decrypt_counts(counts_ct, params: HeParams, l: int, key: tfhe.SecretKey) -> ClassCounts:
    data = counts_ct if isinstance(counts_ct, np.ndarray) else tfhe.to_host(counts_ct)
    vals = tfhe.dec_rlwe(RlweCiphertext(params, data), key)
    return ClassCounts(vals[:l].astype(np.int64))


def model_noise(model: HomWisardModel, key: tfhe.SecretKey) -> tuple[int, int]:
    """Max |phase - nearest codeword| over every model coefficient and the
    decryption margin q/(2p) (hw/tfhe.py:446-473 measure_noise)."""
    params = model.params
    rams = tfhe.to_host(model.rams)
    phase = (rams[:, :, 1] - tfhe._key_mul_host(rams[:, :, 0], key.s)).astype(np.int64)
    delta = params.delta
    err = (phase + delta // 2) % delta - delta // 2
    return int(np.abs(err).max()), delta // 2


def decrypt_model(model: HomWisardModel, key: tfhe.SecretKey):
    """Decrypt the RLWE matrix back into a plaintext integer model (hw/hewnn.py:352-365):
    (IntegerWisardModel with counters (l, k0, 2^a), ClassCounts)."""
    g, params = model.geometry, model.params
    rams = tfhe.to_host(model.rams)                               # (k0, k1, 2, N)
    phase = (rams[:, :, 1] - tfhe._key_mul_host(rams[:, :, 0], key.s)).astype(np.uint32)
    vals = tfhe.decode_phase(phase, params).reshape(g.k0, -1)[:, : 1 << g.selector_bits]
    plain = IntegerWisardModel.zeros(g)
    for c in range(g.l):
        plain.counters[c] = vals[:, c << g.a: (c << g.a) + (1 << g.a)]
    return plain, decrypt_counts(model.counts_ct, params, g.l, key)
