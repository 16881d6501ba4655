"""TFHE at q = 2^32 on B200: the drop-in mirror of the reference's `hewisard.tfhe`.

Client-side operations (key generation, encryption, decryption) run on the host
with numpy, exactly as in the reference (`pkg/src/hewisard/tfhe.py:33-283`),
with the reference's RNG idioms at 4-byte words.  Every homomorphic operation
on the hot path -- external product, CMUX, CDEMUX, blind rotation, sample
extraction, LWE key switch and programmable bootstrapping -- runs in
libhwb200.so (hand-written sm_100a kernels, C ABI in include/hwb.h).  There is
no CPU fallback: without the library or a GPU those calls raise.

Array conventions: ciphertext words are uint32 (stored as torch.int32 on the
device).  Each batched function accepts numpy arrays (host; the result comes
back as numpy) or CUDA tensors (device-resident; the result stays on device).
"""

from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np
import torch

from . import _lib
from ._lib import EncodingError, TfheError
from .params import HeParams, Q_BITS

U32 = np.uint32
U64 = np.uint64
MASK32 = (1 << 32) - 1
PRNG_ID = "numpy-philox4x64"

__all__ = [
    "TfheError", "EncodingError", "make_rng", "uniform_u32", "gaussian_u32",
    "SecretKey", "LweSecretKey", "RlweCiphertext", "RgswCiphertext", "GgswNtt",
    "BootstrapKey", "LweKeySwitchKey", "PbsKeys", "pbs_keygen", "trivial_rlwe",
    "enc_rlwe", "enc_rlwe_raw", "dec_rlwe", "phase_rlwe", "decode_phase", "enc_rgsw",
    "enc_rgsw_batch", "trivial_rgsw", "dec_rgsw", "enc_lwe_batch", "dec_lwe_batch",
    "phase_lwe_batch", "rgsw_rep", "rgsw_to_ntt", "ext_product_batch", "external_product",
    "cmux", "cmux_batch", "cdemux_batch", "blind_rotate", "blind_rotate_batch", "extract_lwe",
    "sample_extract_batch", "mod_switch", "LweCiphertext", "phase_lwe", "dec_lwe", "packing_key_switch",
    "keygen", "pack_batch", "PackingKeySwitchKey", "measure_noise", "NoiseBudget", "test_polynomial", "lwe_keyswitch", "pbs_batch",
    "GgswFft", "rgsw_to_fft", "ggsw_fft_bytes",
]


# ---------------------------------------------------------------------------
# device plumbing (torch for memory and streams only)


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("libhwb200 needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x) -> torch.Tensor:
    """uint32 words -> contiguous torch.int32 CUDA tensor (bit-identical view)."""
    if isinstance(x, torch.Tensor):
        if x.dtype not in (torch.int32, torch.uint32):
            raise TfheError(f"ciphertext tensors must be 32-bit, got {x.dtype}")
        x = x.view(torch.int32) if x.dtype == torch.uint32 else x
        return x.to(_device(), non_blocking=True).contiguous()
    a = np.ascontiguousarray(np.asarray(x), dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).to(_device(), non_blocking=False)


def to_host(t) -> np.ndarray:
    """uint32 words on the host (a torch tensor is copied; numpy passes through)."""
    if isinstance(t, np.ndarray):
        return np.ascontiguousarray(t, dtype=np.uint32) if t.dtype != np.int32 else t.view(np.uint32)
    return t.detach().cpu().numpy().view(np.uint32)


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _wrap(like, t: torch.Tensor):
    return t if isinstance(like, torch.Tensor) else to_host(t)


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
    """hw/tfhe.py:43-47; sigma == 0 draws nothing."""
    if sigma == 0.0:
        return np.zeros(shape, dtype=U32)
    e = np.rint(rng.normal(0.0, sigma, shape))
    return (e.astype(np.int64) & MASK32).astype(U32)


# numpy Philox4x64-10 (Random123 constants; numpy/random/src/philox/philox.h): the
# host side of seeded uniform draws whose words the GPU regenerates (hwb_philox_rgsw)
_PH_M0, _PH_M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_PH_W0, _PH_W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_M64 = (1 << 64) - 1


def philox4x64(ctr, key) -> list[int]:
    """One Philox4x64-10 block (4 uint64) for a 256-bit counter and 128-bit key."""
    c, k0, k1 = [int(x) for x in ctr], int(key[0]), int(key[1])
    for r in range(10):
        if r:
            k0, k1 = (k0 + _PH_W0) & _M64, (k1 + _PH_W1) & _M64
        p0, p1 = _PH_M0 * c[0], _PH_M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & _M64, (p0 >> 64) ^ c[3] ^ k1, p0 & _M64]
    return c


def _ctr_add(ctr, n: int) -> list[int]:
    v = sum(int(x) << (64 * i) for i, x in enumerate(ctr)) + n
    v &= (1 << 256) - 1
    return [(v >> (64 * i)) & _M64 for i in range(4)]


def philox_take(rng: np.random.Generator, nwords: int):
    """Claim the next `nwords` uint32 of rng's stream -- exactly what rng.bytes(4 nwords)
    (hw/tfhe.py:38-40) would return -- WITHOUT generating them on the host: returns the
    hwb_philox block the GPU regenerates them from and leaves rng in the state
    rng.bytes would have left (bit-identical continuation)."""
    bg = rng.bit_generator
    st = bg.state
    if st.get("bit_generator") != "Philox":
        raise TfheError("seeded draws need a numpy Philox generator (make_rng)")
    inner = st["state"]
    ctr = [int(x) for x in inner["counter"]]
    key = [int(x) for x in inner["key"]]
    buf = [int(x) for x in st["buffer"]]
    pos, has32, uint = int(st["buffer_pos"]), int(st["has_uint32"]), int(st["uinteger"])
    prefix = [uint] if has32 else []
    for u in buf[pos:]:
        prefix += [u & 0xFFFFFFFF, u >> 32]
    out = _lib.HwbPhilox()
    out.key[:] = key
    out.ctr[:] = ctr
    if nwords <= len(prefix):
        # served from the host buffer alone
        take = prefix[:nwords]
        out.prefix[: len(take)] = take
        out.nprefix = len(take)
        used = nwords - (1 if has32 else 0)              # words taken from buffer uint64s
        if has32 and nwords >= 1:
            has32 = 0
        if used > 0:
            pos += (used + 1) // 2
            if used % 2:
                has32, uint = 1, buf[pos - 1] >> 32
        new = dict(st, buffer_pos=pos, has_uint32=has32, uinteger=uint)
        bg.state = new
        return out
    out.prefix[: len(prefix)] = prefix
    out.nprefix = len(prefix)
    m = nwords - len(prefix)                             # words from fresh blocks ctr+1, ctr+2, ...
    n64 = (m + 1) // 2
    nblk = (n64 + 3) // 4
    last_ctr = _ctr_add(ctr, nblk)
    last = philox4x64(last_ctr, key)
    new_pos = n64 - 4 * (nblk - 1)
    if m % 2:
        has32, uint = 1, last[new_pos - 1] >> 32
    else:
        has32, uint = 0, last[new_pos - 1] >> 32
    bg.state = {"bit_generator": "Philox",
                "state": {"counter": np.array(last_ctr, dtype=np.uint64), "key": np.array(key, dtype=np.uint64)},
                "buffer": np.array(last, dtype=np.uint64), "buffer_pos": new_pos, "has_uint32": has32,
                "uinteger": uint}
    return out


def philox_rgsw(st, rows: int, N: int, b_rows: torch.Tensor | None = None, out: torch.Tensor | None = None,
                pair: bool = True, a0fix: torch.Tensor | None = None, levels: int = 0) -> torch.Tensor:
    """GPU regeneration of a seeded draw (hwb_philox_rgsw): (rows, 2, N) RGSW rows with
    a from the stream (gadget-carrying words from a0fix) and b from b_rows, or (rows, N)
    a words (pair=False)."""
    dev = _device()
    if out is None:
        out = torch.empty((rows, 2, N) if pair else (rows, N), dtype=torch.int32, device=dev)
    _lib.check(_lib.load().hwb_philox_rgsw(ctypes.byref(st), _ptr(b_rows), _ptr(a0fix), int(levels), _ptr(out),
                                           rows, N, int(pair), _stream()))
    return out


def _key_mul_host(x: np.ndarray, s: np.ndarray) -> np.ndarray:
    """x * s mod 2^32 for binary s, exactly: 16-bit limbs through a float64 FFT
    (the limb-exact product of hw/fft.py:88-119; limb sums < N 2^16 < 2^53)."""
    x = np.asarray(x, dtype=U32)
    n = x.shape[-1]
    fs = np.fft.rfft(np.asarray(s, dtype=np.float64), 2 * n)
    out = np.zeros(x.shape, dtype=U64)
    for shift in (0, 16):
        limb = ((x >> U32(shift)) & U32(0xFFFF)).astype(np.float64)
        conv = np.rint(np.fft.irfft(np.fft.rfft(limb, 2 * n, axis=-1) * fs, 2 * n, axis=-1)).astype(np.int64)
        hi = np.zeros(x.shape, dtype=np.int64)
        hi[..., : n - 1] = conv[..., n: 2 * n - 1]
        out += ((conv[..., :n] - hi).astype(U64) << U64(shift))
    return (out & U64(MASK32)).astype(U32)


# ---------------------------------------------------------------------------
# keys and ciphertext types (hw/tfhe.py:54-173)


@dataclass
class SecretKey:
    """Binary RLWE key S1 (hw/tfhe.py:54-78); extracted LWEs use its coefficients."""

    params: HeParams
    s: np.ndarray

    @property
    def extracted(self) -> np.ndarray:
        return self.s

    def _key_mul(self, x: np.ndarray) -> np.ndarray:
        return _key_mul_host(x, self.s)


@dataclass
class LweSecretKey:
    """Binary LWE key s0 of dimension n (NEW: the PBS input/output key)."""

    params: HeParams
    s: np.ndarray


@dataclass
class RlweCiphertext:
    params: HeParams
    data: np.ndarray            # (2, N): [a, b]

    def __add__(self, other):
        _check_params(self.params, other.params)
        return RlweCiphertext(self.params, self.data + other.data)

    def __sub__(self, other):
        _check_params(self.params, other.params)
        return RlweCiphertext(self.params, self.data - other.data)

    def copy(self):
        return RlweCiphertext(self.params, self.data.copy())


@dataclass
class LweCiphertext:
    """LWE ciphertext (a, b) (hw/tfhe.py:169-173): a uint32 (n,), b uint32.  The
    batched entry points use packed (B, n+1) rows instead (b last); `row()` and
    `from_row()` convert."""

    params: HeParams
    a: np.ndarray
    b: np.uint32

    def row(self) -> np.ndarray:
        return np.concatenate([np.asarray(self.a, dtype=U32), np.asarray([self.b], dtype=U32)])

    @classmethod
    def from_row(cls, params: HeParams, row) -> "LweCiphertext":
        r = np.asarray(row if isinstance(row, np.ndarray) else to_host(row), dtype=U32)
        return cls(params, r[:-1].copy(), U32(r[-1]))


@dataclass
class GgswNtt:
    """Device-resident NTT-domain GGSWs: (count, hwb_ggsw_ntt_words) int32.

    The B200 counterpart of the reference's cached RGSW spectra
    (RgswCiphertext.spectra, hw/tfhe.py:158-162)."""

    params: HeParams
    data: torch.Tensor

    @property
    def count(self) -> int:
        return int(self.data.shape[0])


@dataclass
class GgswFft:
    """Device-resident FFT-domain GGSWs (hwb_ggsw_to_fft): `count` GGSWs of
    hwb_ggsw_fft_bytes each -- the spectra of the signed 16-bit halves of every key
    polynomial, consumed by the FP64 FFT ladders (N = 1024 and 2048)."""

    params: HeParams
    data: torch.Tensor       # uint8, count * ggsw_bytes
    count: int


def ggsw_fft_bytes(params: HeParams) -> int:
    """Bytes of one FFT-domain GGSW, 0 where the FFT ladders do not apply."""
    cp = _lib.c_params(params)
    return int(_lib.load().hwb_ggsw_fft_bytes(ctypes.byref(cp)))


def rgsw_to_fft(params: HeParams, ggsw) -> GgswFft:
    """Transform (count, 2l, 2, N) GGSWs into the FFT domain on the GPU."""
    t = to_device(ggsw if not (isinstance(ggsw, np.ndarray) and ggsw.ndim == 3) else ggsw[np.newaxis])
    if t.dim() != 4 or t.shape[1:] != (2 * params.gadget.levels, 2, params.n):
        raise TfheError(f"GGSW batch must be (count, {2 * params.gadget.levels}, 2, {params.n})")
    nb = ggsw_fft_bytes(params)
    if nb == 0:
        raise TfheError("no FFT-domain GGSWs for these parameters (N = 1024 or 2048, narrow gadgets)")
    out = torch.empty(t.shape[0] * nb, dtype=torch.uint8, device=t.device)
    cp = _lib.c_params(params)
    _lib.check(_lib.load().hwb_ggsw_to_fft(ctypes.byref(cp), _ptr(t), _ptr(out), t.shape[0], _stream()))
    return GgswFft(params, out, int(t.shape[0]))


@dataclass
class RgswCiphertext:
    """2*ell RLWE rows C + m*G; rows 0..l-1 gadget on b, l..2l-1 on a (hw/tfhe.py:146-166)."""

    params: HeParams
    data: np.ndarray            # (2l, 2, N)
    _ntt: GgswNtt | None = field(default=None, repr=False)

    def spectra(self) -> GgswNtt:
        if self._ntt is None:
            self._ntt = rgsw_to_ntt(self.params, self.data[np.newaxis])
        return self._ntt


@dataclass
class BootstrapKey:
    """RGSW_{S1}(s0_i) for i < n, resident on the device in the NTT domain and,
    where the FP64 FFT ladder applies (N = 1024 and 2048), as the FFT spectra of its signed
    16-bit key halves (hwb_bsk_to_fft)."""

    params: HeParams
    ntt: GgswNtt | None
    fft: torch.Tensor | None = field(default=None, repr=False)
    count: int = 0

    @staticmethod
    def from_coefficients(params: HeParams, bsk) -> "BootstrapKey":
        """NTT image where the exact two-prime range allows it, FFT image where the FP64
        ladders apply (full-precision 2 x 16 gadgets have only the latter)."""
        coeff = to_device(bsk)
        key = BootstrapKey(params, rgsw_to_ntt(params, coeff) if ntt_supported(params) else None,
                           count=int(coeff.shape[0]))
        cp = _lib.c_params(params)
        L = _lib.load()
        nbytes = L.hwb_bsk_fft_bytes(ctypes.byref(cp))
        if nbytes:
            key.fft = torch.empty(nbytes, dtype=torch.uint8, device=coeff.device)
            _lib.check(L.hwb_bsk_to_fft(ctypes.byref(cp), _ptr(coeff), _ptr(key.fft), _stream()))
        if key.ntt is None and key.fft is None:
            raise TfheError("neither exact ladder supports these parameters")
        return key


@dataclass
class LweKeySwitchKey:
    """KSK[j, t] = LWE_{s0}(s1_j q / beta_ks^(t+1)), (N, ks_l, n+1) on the device."""

    params: HeParams
    data: torch.Tensor
    _tiles: torch.Tensor | None = field(default=None, repr=False)

    def tensor_core_tiles(self) -> torch.Tensor | None:
        """The key split into byte limbs and tiled for the tcgen05 key switch
        (built once on the device); None when ks_base_log > 8."""
        if self._tiles is None:
            cp = _lib.c_params(self.params)
            L = _lib.load()
            nbytes = L.hwb_ksk_tc_bytes(ctypes.byref(cp))
            if nbytes == 0:
                return None
            tiles = torch.empty(nbytes, dtype=torch.uint8, device=self.data.device)
            _lib.check(L.hwb_ksk_to_tc(ctypes.byref(cp), _ptr(self.data), _ptr(tiles), _stream()))
            self._tiles = tiles
        return self._tiles


def _ks_engine(params: HeParams, ksk, engine: str) -> bool:
    """True -> tensor-core key switch.  engine: "auto" (tensor cores when the
    gadget allows it), "tc" (required), "simt" (integer-pipe kernel)."""
    if engine not in ("auto", "tc", "simt"):
        raise TfheError(f"unknown key-switch engine {engine!r}")
    if ksk is None or engine == "simt":
        return False
    if ksk.tensor_core_tiles() is not None:
        return True
    if engine == "tc":
        raise TfheError("tensor-core key switch needs ks_base_log <= 8")
    return False


@dataclass
class PbsKeys:
    params: HeParams
    lwe_key: LweSecretKey          # s0
    glwe_key: SecretKey            # s1
    bsk: np.ndarray                # (n, 2l, 2, N) coefficient domain (client copy)
    ksk: np.ndarray                # (N, ks_l, n+1)

    def device_keys(self) -> tuple[BootstrapKey, LweKeySwitchKey]:
        """Upload once: the BSK is transformed to the NTT (and FFT) domain on the GPU."""
        return (BootstrapKey.from_coefficients(self.params, self.bsk),
                LweKeySwitchKey(self.params, to_device(self.ksk)))


def _check_params(p1: HeParams, p2: HeParams):
    if p1 is not p2 and p1 != p2:
        raise TfheError("ciphertext parameter sets differ")


# ---------------------------------------------------------------------------
# client side: key generation, encryption, decryption (host)


def pbs_keygen(params: HeParams, rng_seed) -> PbsKeys:
    """NEW: PBS keys from one Philox stream (same stream as oracle/tfhe32.py).

    s1 = integers(0,2,N) (hw/tfhe.py:99), s0 = integers(0,2,n), BSK =
    enc_rgsw_batch(s0 under s1) (hw/tfhe.py:246-263), then the LWE key-switch
    key with a (N, ks_l, n) drawn before e (N, ks_l)."""
    if params.lwe_n < 1:
        raise TfheError("parameter set has no LWE dimension (lwe_n)")
    rng = make_rng(rng_seed)
    N, n = params.n, params.lwe_n
    s1 = rng.integers(0, 2, N).astype(U32)
    s0 = rng.integers(0, 2, n).astype(U32)
    key1 = SecretKey(params, s1)
    bsk = np.stack([c.data for c in enc_rgsw_batch(s0, key1, rng)])
    gk = params.gadget_ks
    a = uniform_u32(rng, (N, gk.levels, n))
    e = gaussian_u32(rng, params.lwe_sigma, (N, gk.levels))
    dot = (a.astype(U64) * s0.astype(U64)).sum(axis=-1, dtype=U64)
    msg = np.zeros((N, gk.levels), dtype=U64)
    for t in range(gk.levels):
        msg[:, t] = s1.astype(U64) * U64(gk.power(t))
    b = (dot + e.astype(U64) + msg) & U64(MASK32)
    ksk = np.concatenate([a, b.astype(U32)[..., None]], axis=-1)
    return PbsKeys(params, LweSecretKey(params, s0), key1, bsk, ksk)


@dataclass
class PackingKeySwitchKey:
    """RLWE encryptions of s_j * q/beta^(t+1) for every key coefficient j
    (hw/tfhe.py:81-92), (N, l_pks, 2, N); spectra() uploads the NTT image."""

    params: HeParams
    data: np.ndarray
    _ntt: torch.Tensor | None = field(default=None, repr=False)

    def spectra(self) -> torch.Tensor:
        if self._ntt is None:
            t = to_device(self.data)
            npolys = t.numel() // self.params.n
            out = torch.empty((npolys, 2, self.params.n), dtype=torch.int32, device=t.device)
            cp = _lib.c_params(self.params)
            _lib.check(_lib.load().hwb_poly_to_ntt(ctypes.byref(cp), _ptr(t), _ptr(out), npolys, _stream()))
            self._ntt = out
        return self._ntt


def keygen(params: HeParams, rng_seed) -> tuple[SecretKey, PackingKeySwitchKey]:
    """hw/tfhe.py:95-114 at q = 2^32: binary RLWE key S1 and the packing
    key-switch key, drawn in the reference's chunked order (step = 2^20 //
    (l N) key rows per chunk: a, then e, per chunk)."""
    rng = make_rng(rng_seed)
    n = params.n
    s = rng.integers(0, 2, n).astype(U32)
    key = SecretKey(params, s)
    g = params.gadget_pks
    ksk = np.empty((n, g.levels, 2, n), dtype=U32)
    step = max(1, 2 ** 20 // (g.levels * n))
    for j0 in range(0, n, step):
        j1 = min(n, j0 + step)
        a = uniform_u32(rng, (j1 - j0, g.levels, n))
        e = gaussian_u32(rng, params.sigma, (j1 - j0, g.levels, n))
        b = (key._key_mul(a) + e).astype(U32)
        for t in range(g.levels):
            b[:, t, 0] += s[j0:j1] * U32(g.power(t))
        ksk[j0:j1, :, 0, :] = a
        ksk[j0:j1, :, 1, :] = b
    return key, PackingKeySwitchKey(params, ksk)


def pack_batch(a_stacks, b_polys, ksk: PackingKeySwitchKey):
    """Batched packing key switch (hw/tfhe.py:390-439): a_stacks (B, k, N) LWE
    a-vectors (k <= N, row i = input i), b_polys (B, N) with coefficient i = b
    of input i -> (B, 2, N) RLWEs whose coefficient i decrypts to input i."""
    params = ksk.params
    n = params.n
    a = to_device(a_stacks)
    bp = to_device(b_polys)
    if a.dim() != 3 or a.shape[2] != n or a.shape[1] > n:
        raise TfheError(f"cannot pack {a.shape[1] if a.dim() == 3 else '?'} > N = {n} ciphertexts")
    B, k = a.shape[0], a.shape[1]
    apolys = torch.zeros((B, n, n), dtype=torch.int32, device=a.device)   # apolys[b][j][i] = a^(i)_j
    apolys[:, :, :k] = a.transpose(1, 2)
    out = torch.empty((B, 2, n), dtype=torch.int32, device=a.device)
    cp = _lib.c_params(params)
    L = _lib.load()
    ws = torch.empty(max(1, (L.hwb_pack_ks_workspace_bytes(ctypes.byref(cp), B) + 3) // 4),
                     dtype=torch.int32, device=a.device)
    g = params.gadget_pks
    _lib.check(L.hwb_pack_ks(ctypes.byref(cp), g.levels, g.base_log, _ptr(ksk.spectra()), _ptr(apolys),
                             _ptr(bp), _ptr(out), B, _ptr(ws), _stream()))
    return _wrap(a_stacks, out)


def packing_key_switch(cs: Sequence[LweCiphertext], ksk: PackingKeySwitchKey) -> RlweCiphertext:
    """hw/tfhe.py:373-387: pack <= N extracted-LWE ciphertexts into one RLWE whose
    coefficient i decrypts to message i (also accepts packed (N+1,) rows)."""
    params = ksk.params
    n = params.n
    if len(cs) > n:
        raise TfheError(f"cannot pack {len(cs)} > N = {n} ciphertexts")
    if len(cs) == 0:
        return RlweCiphertext(params, np.zeros((2, n), dtype=U32))
    out_rows = []
    for c in cs:
        if isinstance(c, LweCiphertext):
            _check_params(c.params, params)
            out_rows.append(c.row())
        else:
            out_rows.append(np.asarray(c if isinstance(c, np.ndarray) else to_host(c), dtype=U32))
    rows = np.stack(out_rows)
    b = np.zeros(n, dtype=U32)
    b[: len(rows)] = rows[:, n]
    out = pack_batch(rows[None, :, :n], b[None], ksk)[0]
    return RlweCiphertext(ksk.params, out)


def _encode(m, params: HeParams) -> np.ndarray:
    """hw/tfhe.py:181-190."""
    n = params.n
    m = np.atleast_1d(np.asarray(m, dtype=np.int64))
    if m.size > n:
        raise EncodingError(f"message longer than ring dimension {n}")
    if np.any(m < 0) or np.any(m >= params.p):
        raise EncodingError(f"message coefficients must lie in [0, {params.p})")
    mu = np.zeros(n, dtype=U32)
    mu[: m.size] = (m * params.delta) & MASK32
    return mu


def trivial_rlwe(m, params: HeParams) -> RlweCiphertext:
    """hw/tfhe.py:193-197."""
    data = np.zeros((2, params.n), dtype=U32)
    data[1] = _encode(m, params)
    return RlweCiphertext(params, data)


def enc_rlwe_raw(mu, key: SecretKey, rng) -> RlweCiphertext:
    """hw/tfhe.py:200-206."""
    n = key.params.n
    a = uniform_u32(rng, (n,))
    e = gaussian_u32(rng, key.params.sigma, (n,))
    b = key._key_mul(a) + np.asarray(mu, dtype=U32) + e
    return RlweCiphertext(key.params, np.stack([a, b.astype(U32)]))


def enc_rlwe(m, key: SecretKey, rng) -> RlweCiphertext:
    return enc_rlwe_raw(_encode(m, key.params), key, rng)


def phase_rlwe(ct: RlweCiphertext, key: SecretKey) -> np.ndarray:
    data = ct.data if isinstance(ct.data, np.ndarray) else to_host(ct.data)
    return (data[1] - key._key_mul(data[0])).astype(U32)


def decode_phase(phase, params: HeParams) -> np.ndarray:
    """hw/tfhe.py:223-225."""
    half = U64(params.delta // 2)
    ph = np.asarray(phase).astype(U64)
    return (((ph + half) & U64(MASK32)) >> U64(Q_BITS - params.p.bit_length() + 1)).astype(np.int64)


def dec_rlwe(ct: RlweCiphertext, key: SecretKey) -> np.ndarray:
    return decode_phase(phase_rlwe(ct, key), ct.params)


def enc_rgsw_batch(ms, key: SecretKey, rng) -> list[RgswCiphertext]:
    """hw/tfhe.py:246-263: one batched key product; a drawn before e."""
    ms = np.asarray(ms, dtype=np.int64)
    if ms.size == 0:
        return []
    if np.any((ms != 0) & (ms != 1)):
        raise EncodingError("RGSW messages are bits")
    params = key.params
    g = params.gadget
    rows = 2 * g.levels
    a = uniform_u32(rng, (len(ms), rows, params.n))
    e = gaussian_u32(rng, params.sigma, (len(ms), rows, params.n))
    b = (key._key_mul(a) + e).astype(U32)
    data = np.stack([a, b], axis=2)
    for t in range(g.levels):
        data[:, t, 1, 0] += ms.astype(U32) * U32(g.power(t))
        data[:, g.levels + t, 0, 0] += ms.astype(U32) * U32(g.power(t))
    return [RgswCiphertext(params, data[i]) for i in range(len(ms))]


def enc_rgsw(m: int, key: SecretKey, rng) -> RgswCiphertext:
    """hw/tfhe.py:228-243."""
    if m not in (0, 1):
        raise EncodingError("RGSW messages are bits")
    return enc_rgsw_batch([m], key, rng)[0]


def trivial_rgsw(m: int, params: HeParams) -> RgswCiphertext:
    """hw/tfhe.py:266-275."""
    if m not in (0, 1):
        raise EncodingError("RGSW messages are bits")
    g = params.gadget
    data = np.zeros((2 * g.levels, 2, params.n), dtype=U32)
    if m:
        for t in range(g.levels):
            data[t, 1, 0] += U32(g.power(t))
            data[g.levels + t, 0, 0] += U32(g.power(t))
    return RgswCiphertext(params, data)


def dec_rgsw(ct: RgswCiphertext, key: SecretKey) -> int:
    """hw/tfhe.py:278-283."""
    phase = ct.data[0, 1] - key._key_mul(ct.data[0, 0])
    g = ct.params.gadget
    val = ((int(phase[0]) + g.power(0) // 2) & MASK32) >> (Q_BITS - g.base_log)
    return val % g.base


def enc_lwe_batch(mu, key: LweSecretKey, rng) -> np.ndarray:
    """NEW: LWE_{s0}(mu) rows (B, n+1), b last; a (B, n) drawn before e (B,)."""
    mu = np.asarray(mu, dtype=np.int64)
    s0 = key.s
    B, n = len(mu), len(s0)
    a = uniform_u32(rng, (B, n))
    e = gaussian_u32(rng, key.params.lwe_sigma, (B,))
    dot = (a.astype(U64) * s0.astype(U64)).sum(axis=-1, dtype=U64)
    b = (dot + e.astype(U64) + (mu & MASK32).astype(U64)) & U64(MASK32)
    return np.concatenate([a, b.astype(U32)[:, None]], axis=1)


def phase_lwe_batch(lwe, s: np.ndarray) -> np.ndarray:
    """hw/tfhe.py:364-366 on (B, n+1) rows (b last) under key coefficients s."""
    lwe = lwe if isinstance(lwe, np.ndarray) else to_host(lwe)
    lwe = np.asarray(lwe, dtype=U32)
    dot = (lwe[..., :-1].astype(U64) * np.asarray(s, dtype=U64)).sum(axis=-1, dtype=U64)
    return ((lwe[..., -1].astype(U64) - dot) & U64(MASK32)).astype(U32)


def dec_lwe_batch(lwe, key, params: HeParams | None = None) -> np.ndarray:
    """hw/tfhe.py:369-370 batched; key is an LweSecretKey or SecretKey."""
    params = params or key.params
    return decode_phase(phase_lwe_batch(lwe, key.s), params)


@dataclass
class NoiseBudget:
    """Measured error against the nearest Z_p codeword (hw/tfhe.py:446-456)."""

    max_abs: int
    rms: float
    margin: int

    @property
    def ok(self) -> bool:
        return self.max_abs < self.margin


def measure_noise(ct, key, params: HeParams | None = None) -> NoiseBudget:
    """hw/tfhe.py:459-473 for an RlweCiphertext, or LWE rows (..., n+1) under
    `key` (LweSecretKey or SecretKey)."""
    if isinstance(ct, RlweCiphertext):
        params = ct.params
        phase = phase_rlwe(ct, key).astype(np.int64)
    elif isinstance(ct, LweCiphertext):
        params = ct.params
        phase = np.array([int(phase_lwe(ct, key))], dtype=np.int64)
    else:
        params = params or key.params
        phase = phase_lwe_batch(ct, key.s).astype(np.int64)
    delta = params.delta
    err = (phase + delta // 2) % delta - delta // 2
    return NoiseBudget(int(np.abs(err).max()), float(np.sqrt(np.mean(err.astype(np.float64) ** 2))), delta // 2)


# ---------------------------------------------------------------------------
# device: NTT-domain GGSWs


def ntt_supported(params: HeParams) -> bool:
    """The exact two-prime NTT applies (2l N beta/2 2^31 < p0 p1 / 2); the
    FP64 FFT ladders cover full-precision gadgets beyond it."""
    cp = _lib.c_params(params)
    null = ctypes.c_void_p(0)
    return _lib.load().hwb_ggsw_to_ntt(ctypes.byref(cp), null, null, 0, null) == 0


def _fft_level(params: HeParams, fft: "GgswFft", idx, cur: torch.Tensor, inverse: bool) -> torch.Tensor:
    """One FFT-path IVP (CDEMUX) or VP (CMUX) level with m = 1 (hwb_ivp/vp_level_fft):
    cur (B, 2 or 1, 2, N) -> (B, 1 or 2, 2, N)."""
    B = cur.shape[0]
    nxt = torch.empty((B, 2 if inverse else 1, 2, params.n), dtype=torch.int32, device=cur.device)
    fn = _lib.load().hwb_ivp_level_fft if inverse else _lib.load().hwb_vp_level_fft
    cp = _lib.c_params(params)
    _lib.check(fn(ctypes.byref(cp), _ptr(fft.data), _ptr(idx), _ptr(cur.contiguous()), _ptr(nxt), 1, B, _stream()))
    return nxt


def _fft_rep(params: HeParams, rep) -> "GgswFft":
    if isinstance(rep, GgswFft):
        return rep
    if isinstance(rep, RgswCiphertext):
        rep = rep.data
    arr = rep if isinstance(rep, torch.Tensor) else np.asarray(rep)
    if arr.ndim == 3:
        arr = arr[None]
    return rgsw_to_fft(params, arr)


def _fft_idx(count: int, B: int, idx, dev) -> torch.Tensor:
    if idx is not None:
        it = torch.as_tensor(np.asarray(idx) if not isinstance(idx, torch.Tensor) else idx, dtype=torch.int32)
        if it.numel() != B:
            raise TfheError("GGSW index vector length differs from the batch")
        return it.to(dev).contiguous()
    if count == 1:
        return torch.zeros(B, dtype=torch.int32, device=dev)
    if count != B:
        raise TfheError(f"rgsw batch {count} does not match ciphertext batch {B}")
    return torch.arange(B, dtype=torch.int32, device=dev)


def rgsw_to_ntt(params: HeParams, ggsw) -> GgswNtt:
    """Forward-transform (count, 2l, 2, N) GGSWs into the NTT domain on the GPU."""
    g = ggsw
    if isinstance(g, np.ndarray) and g.ndim == 3:
        g = g[np.newaxis]
    t = to_device(g)
    if t.dim() != 4 or t.shape[1:] != (2 * params.gadget.levels, 2, params.n):
        raise TfheError(f"GGSW batch must be (count, {2 * params.gadget.levels}, 2, {params.n}), "
                        f"got {tuple(t.shape)}")
    cp = _lib.c_params(params)
    words = _lib.load().hwb_ggsw_ntt_words(ctypes.byref(cp))
    out = torch.empty((t.shape[0], words), dtype=torch.int32, device=t.device)
    _lib.check(_lib.load().hwb_ggsw_to_ntt(ctypes.byref(cp), _ptr(t), _ptr(out), t.shape[0], _stream()))
    return GgswNtt(params, out)


def rgsw_rep(ct: RgswCiphertext) -> GgswNtt:
    """Representation used by the batched external product (hw/tfhe.py:322-324)."""
    return ct.spectra()


def _as_ntt(params: HeParams, rep) -> GgswNtt:
    if isinstance(rep, GgswNtt):
        return rep
    if isinstance(rep, RgswCiphertext):
        return rep.spectra()
    arr = rep if isinstance(rep, torch.Tensor) else np.asarray(rep)
    if arr.ndim == 3:
        arr = arr[None]
    return rgsw_to_ntt(params, arr)


def _check_cts(params: HeParams, t: torch.Tensor, what="ciphertext batch"):
    if t.dim() != 3 or t.shape[1:] != (2, params.n):
        raise TfheError(f"{what} must be (B, 2, {params.n}), got {tuple(t.shape)}")


def _gidx(ntt: GgswNtt, B: int, idx=None):
    if idx is not None:
        it = torch.as_tensor(np.asarray(idx) if not isinstance(idx, torch.Tensor) else idx,
                             dtype=torch.int32).to(ntt.data.device).contiguous()
        if it.numel() != B:
            raise TfheError("GGSW index vector length differs from the batch")
        return it
    if ntt.count == 1:
        return None
    if ntt.count != B:
        raise TfheError(f"rgsw batch {ntt.count} does not match ciphertext batch {B}")
    return torch.arange(B, dtype=torch.int32, device=ntt.data.device)


def ext_product_batch(params: HeParams, rgsw_rep, cts, idx=None):
    """hw/tfhe.py:301-319: rep (B|1, 2l, 2, N) (or GgswNtt), cts (B, 2, N) -> (B, 2, N)."""
    if not ntt_supported(params) and not isinstance(rgsw_rep, GgswNtt):
        # full-precision gadgets: the product is the hi half of a one-level CDEMUX (FFT path)
        t = to_device(cts)
        _check_cts(params, t)
        fft = _fft_rep(params, rgsw_rep)
        nxt = _fft_level(params, fft, _fft_idx(fft.count, t.shape[0], idx, t.device), t.unsqueeze(1), True)
        return _wrap(cts, nxt[:, 1].contiguous())
    ntt = _as_ntt(params, rgsw_rep)
    t = to_device(cts)
    _check_cts(params, t)
    B = t.shape[0]
    gi = _gidx(ntt, B, idx)
    out = torch.empty_like(t)
    cp = _lib.c_params(params)
    _lib.check(_lib.load().hwb_ext_product(ctypes.byref(cp), _ptr(ntt.data), _ptr(gi), _ptr(t),
                                           _ptr(out), B, _stream()))
    return _wrap(cts, out)


def external_product(C: RgswCiphertext, c: RlweCiphertext) -> RlweCiphertext:
    """hw/tfhe.py:327-331."""
    _check_params(C.params, c.params)
    out = ext_product_batch(c.params, C.spectra(), c.data[np.newaxis] if isinstance(c.data, np.ndarray)
                            else c.data.unsqueeze(0))
    return RlweCiphertext(c.params, out[0])


def cmux_batch(params: HeParams, rgsw_rep, c1, c0, idx=None, rot=None):
    """hw/lut.py:200-206 / hw/tfhe.py:334-337 batched: c0 + C (*) (c1 - c0).
    With c1 None, c1 = c0 * X^rot[b] per item (the rotated branch)."""
    if not ntt_supported(params) and not isinstance(rgsw_rep, GgswNtt):
        # full-precision gadgets: a one-level VP CMUX on the FFT path
        t0 = to_device(c0)
        _check_cts(params, t0)
        if c1 is not None:
            t1 = to_device(c1)
            _check_cts(params, t1)
        else:
            if rot is None:
                raise TfheError("cmux needs c1 or a rotation vector")
            from .lut import monomial_gather
            t1 = monomial_gather(params, t0, rot)
        fft = _fft_rep(params, rgsw_rep)
        nxt = _fft_level(params, fft, _fft_idx(fft.count, t0.shape[0], idx, t0.device),
                         torch.stack([t0, t1], dim=1), False)
        return _wrap(c0, nxt[:, 0].contiguous())
    ntt = _as_ntt(params, rgsw_rep)
    t0 = to_device(c0)
    _check_cts(params, t0)
    B = t0.shape[0]
    t1 = None
    rt = None
    if c1 is not None:
        t1 = to_device(c1)
        _check_cts(params, t1)
    else:
        if rot is None:
            raise TfheError("cmux needs c1 or a rotation vector")
        rt = torch.as_tensor(np.asarray(rot, dtype=np.int64) if not isinstance(rot, torch.Tensor) else rot)
        rt = (rt % (2 * params.n)).to(torch.int32).to(t0.device).contiguous()
        if rt.numel() != B:
            raise TfheError("rotation vector length differs from the batch")
    gi = _gidx(ntt, B, idx)
    out = torch.empty_like(t0)
    cp = _lib.c_params(params)
    _lib.check(_lib.load().hwb_cmux(ctypes.byref(cp), _ptr(ntt.data), _ptr(gi), _ptr(t1), _ptr(t0),
                                    _ptr(rt), _ptr(out), B, _stream()))
    return _wrap(c0, out)


def cdemux_batch(params: HeParams, rgsw_rep, d, idx=None):
    """hw/lut.py:113-119 batched: (d - C (*) d, C (*) d)."""
    if not ntt_supported(params) and not isinstance(rgsw_rep, GgswNtt):
        t = to_device(d)
        _check_cts(params, t)
        fft = _fft_rep(params, rgsw_rep)
        nxt = _fft_level(params, fft, _fft_idx(fft.count, t.shape[0], idx, t.device), t.unsqueeze(1), True)
        return _wrap(d, nxt[:, 0].contiguous()), _wrap(d, nxt[:, 1].contiguous())
    ntt = _as_ntt(params, rgsw_rep)
    t = to_device(d)
    _check_cts(params, t)
    B = t.shape[0]
    gi = _gidx(ntt, B, idx)
    lo, hi = torch.empty_like(t), torch.empty_like(t)
    cp = _lib.c_params(params)
    _lib.check(_lib.load().hwb_cdemux(ctypes.byref(cp), _ptr(ntt.data), _ptr(gi), _ptr(t), _ptr(lo),
                                      _ptr(hi), B, _stream()))
    return _wrap(d, lo), _wrap(d, hi)


def cmux(C: RgswCiphertext, c1: RlweCiphertext, c2: RlweCiphertext) -> RlweCiphertext:
    """hw/tfhe.py:334-337: select c1 if the RGSW bit is 1, else c2."""
    _check_params(c1.params, c2.params)
    out = cmux_batch(c1.params, C.spectra(), np.asarray(c1.data)[None], np.asarray(c2.data)[None])
    return RlweCiphertext(c1.params, out[0])


def blind_rotate_batch(params: HeParams, acc, ggsw, exps):
    """Fused hw/tfhe.py:340-349 over a batch: acc (B, 2, N), ggsw L GGSWs shared by
    the batch (GgswNtt or (L, 2l, 2, N)), exps (B, L) the I values."""
    wide = not ntt_supported(params) and not isinstance(ggsw, GgswNtt)
    rep = _fft_rep(params, ggsw) if wide else _as_ntt(params, ggsw)
    t = to_device(acc).clone()
    _check_cts(params, t, "accumulator batch")
    B = t.shape[0]
    e = torch.as_tensor(np.asarray(exps, dtype=np.int64) if not isinstance(exps, torch.Tensor) else exps)
    e = (e % (2 * params.n)).to(torch.int32)
    if e.dim() == 1:
        e = e.unsqueeze(0).expand(B, -1)
    if e.shape[0] != B or e.shape[1] != rep.count:
        raise TfheError("selector/exponent length mismatch")
    e = e.to(t.device).contiguous()
    cp = _lib.c_params(params)
    fn = _lib.load().hwb_blind_rotate_fft if wide else _lib.load().hwb_blind_rotate
    _lib.check(fn(ctypes.byref(cp), _ptr(rep.data), None, _ptr(e), _ptr(t), rep.count, B, _stream()))
    return _wrap(acc, t)


def blind_rotate(c: RlweCiphertext, C: Sequence[RgswCiphertext], I: Sequence[int]) -> RlweCiphertext:
    """hw/tfhe.py:340-349: v -> v * X^(-sum S_i I_i)."""
    if len(C) != len(I):
        raise TfheError("selector/exponent length mismatch")
    params = c.params
    if len(C) == 0:
        return c.copy()
    ggsw = np.stack([np.asarray(x.data) for x in C])
    out = blind_rotate_batch(params, np.asarray(c.data)[None], ggsw, np.asarray(I, dtype=np.int64)[None])
    return RlweCiphertext(params, out[0])


def sample_extract_batch(params: HeParams, rlwe, coeff: int = 0):
    """hw/tfhe.py:352-361 batched: (B, 2, N) -> (B, N+1), b last."""
    t = to_device(rlwe)
    _check_cts(params, t)
    B = t.shape[0]
    out = torch.empty((B, params.n + 1), dtype=torch.int32, device=t.device)
    cp = _lib.c_params(params)
    _lib.check(_lib.load().hwb_sample_extract(ctypes.byref(cp), _ptr(t), _ptr(out), B, int(coeff),
                                              _stream()))
    return _wrap(rlwe, out)


def extract_lwe(c: RlweCiphertext, i: int = 0) -> LweCiphertext:
    """hw/tfhe.py:352-361: LWE of coefficient i under the coefficients of S1
    (a'[j] = a[i-j] for j <= i, -a[N+i-j] above; b' = b[i]) -- on the GPU."""
    n = c.params.n
    if not 0 <= i < n:
        raise TfheError(f"coefficient index {i} out of range [0, {n})")
    data = c.data[None] if isinstance(c.data, np.ndarray) else c.data.unsqueeze(0)
    return LweCiphertext.from_row(c.params, sample_extract_batch(c.params, data, i)[0])


def _key_coeffs(key) -> np.ndarray:
    # SecretKey.extracted (S1's coefficients, hw/tfhe.py:64-66) or LweSecretKey.s
    return np.asarray(key.extracted if hasattr(key, "extracted") else key.s, dtype=U64)


def phase_lwe(ct: LweCiphertext, key) -> np.uint32:
    """hw/tfhe.py:364-366: b - <a, s> mod 2^32 (key: SecretKey or LweSecretKey)."""
    dot = (np.asarray(ct.a, dtype=U64) * _key_coeffs(key)).sum(dtype=U64)
    return U32((int(ct.b) - int(dot)) & MASK32)


def dec_lwe(ct: LweCiphertext, key) -> int:
    """hw/tfhe.py:369-370."""
    return int(decode_phase(np.array([phase_lwe(ct, key)], dtype=U32), ct.params)[0])


# ---------------------------------------------------------------------------
# PBS (NEW composition)


def mod_switch(x, n_ring: int) -> np.ndarray:
    """NEW: round(x 2N / q) mod 2N with the rounding idiom of hw/ring.py:139-140."""
    logm = (2 * n_ring).bit_length() - 1
    x = np.asarray(x, dtype=U64)
    return (((x + U64(1 << (Q_BITS - logm - 1))) & U64(MASK32)) >> U64(Q_BITS - logm)).astype(np.int64)


def test_polynomial(f, params: HeParams, delta_out: int | None = None) -> np.ndarray:
    """NEW: trivial GLWE (0, TV) (cf. trivial_rlwe/encode_lut, hw/tfhe.py:193-197,
    hw/lut.py:86-97) evaluating m -> f(m) for m in [0, p/2); centred boxes of
    2N/p phase units; m in [p/2, p) gives -f(m - p/2) (negacyclic)."""
    p, n_ring = params.p, params.n
    if delta_out is None:
        delta_out = params.delta
    f = np.asarray(f, dtype=np.int64)
    if f.shape != (p // 2,):
        raise TfheError(f"LUT must have p/2 = {p // 2} entries")
    box = 2 * n_ring // p
    if box < 1:
        raise TfheError("plaintext modulus too large for the ring (2N/p < 1)")
    j = np.arange(n_ring)
    m = (j + box // 2) // box
    val = np.where(m < p // 2, f[np.minimum(m, p // 2 - 1)] * delta_out,
                   -f[np.clip(m - p // 2, 0, p // 2 - 1)] * delta_out)
    tv = np.zeros((2, n_ring), dtype=U32)
    tv[1] = (val & MASK32).astype(U32)
    return tv


def lwe_keyswitch(params: HeParams, lwe, ksk: LweKeySwitchKey, out=None, engine: str = "auto",
                  workspace: "PbsWorkspace | None" = None):
    """NEW LWE key switch (B, N+1) under s1 -> (B, n+1) under s0 (algebra of
    hw/tfhe.py:397-420).  engine: "auto" | "tc" (tcgen05 int8 GEMM) | "simt"."""
    t = to_device(lwe)
    if t.dim() != 2 or t.shape[1] != params.n + 1:
        raise TfheError(f"LWE batch must be (B, {params.n + 1})")
    B = t.shape[0]
    if out is None:
        out = torch.empty((B, params.lwe_n + 1), dtype=torch.int32, device=t.device)
    elif out.shape != (B, params.lwe_n + 1) or out.dtype != torch.int32 or not out.is_contiguous():
        raise TfheError(f"out must be a contiguous int32 (B, {params.lwe_n + 1}) tensor")
    cp = _lib.c_params(params)
    if _ks_engine(params, ksk, engine):
        ws = _ws(workspace).get(params, B, t.device, kind="ks_tc")
        _lib.check(_lib.load().hwb_keyswitch_tc(ctypes.byref(cp), _ptr(ksk.tensor_core_tiles()), _ptr(t),
                                                _ptr(out), B, _ptr(ws), _stream()))
    else:
        _lib.check(_lib.load().hwb_keyswitch(ctypes.byref(cp), _ptr(ksk.data), _ptr(t), _ptr(out), B,
                                             _stream()))
    return _wrap(lwe, out)


class PbsWorkspace:
    """Reusable device workspace for pbs_batch (avoids per-call allocation)."""

    def __init__(self):
        self.buf = None

    def get(self, params: HeParams, B: int, device, kind: str = "pbs") -> torch.Tensor:
        cp = _lib.c_params(params)
        L = _lib.load()
        if kind.startswith("pbs_fft"):
            nbytes = L.hwb_pbs_fft_workspace_bytes(ctypes.byref(cp), B, int(kind == "pbs_fft_ks"))
        else:
            size_fn = {"pbs": "hwb_pbs_workspace_bytes", "pbs_tc": "hwb_pbs_tc_workspace_bytes",
                       "ks_tc": "hwb_keyswitch_tc_workspace_bytes"}[kind]
            nbytes = getattr(L, size_fn)(ctypes.byref(cp), B)
        words = max(1, (nbytes + 3) // 4)
        if self.buf is None or self.buf.numel() < words or self.buf.device != device:
            self.buf = torch.empty(words, dtype=torch.int32, device=device)
        return self.buf


_default_ws: dict = {}
_default_ws_lock = threading.Lock()


def _ws(workspace: "PbsWorkspace | None") -> PbsWorkspace:
    """The caller's workspace, else a default one per (device, current stream): two
    threads or streams running PBS concurrently never share scratch memory, and a
    resize only frees a buffer last used on the same stream (the caching allocator
    orders its reuse after that stream's queued kernels)."""
    if workspace is not None:
        return workspace
    key = (torch.cuda.current_device(), torch.cuda.current_stream().cuda_stream)
    with _default_ws_lock:
        ws = _default_ws.get(key)
        if ws is None:
            ws = _default_ws[key] = PbsWorkspace()
    return ws


def _use_fft_ladder(bsk: BootstrapKey, B: int, ladder: str) -> bool:
    """"auto": the FP64 FFT ladders when their key exists -- the cluster latency
    ladder while the batch fits co-resident clusters (2l SMs per ciphertext), the
    throughput ladders above one CTA per SM -- and the NTT latency ladder in
    between; "fft" / "ntt" force one family (all ladders are bit-identical)."""
    if ladder not in ("auto", "fft", "ntt"):
        raise TfheError(f"unknown ladder {ladder!r}")
    if ladder == "ntt":
        if bsk.ntt is None:
            raise TfheError("no NTT bootstrapping key for these parameters (gadget beyond the two-prime range)")
        return False
    if bsk.ntt is None:
        return True
    if bsk.fft is None:
        if ladder == "fft":
            raise TfheError("no FFT bootstrapping key for these parameters (N = 1024 or 2048, narrow gadgets)")
        return False
    if ladder == "fft" or B > torch.cuda.get_device_properties(bsk.fft.device).multi_processor_count:
        return True
    L = _lib.load()
    cap = L.hwb_set_fft_cluster_batch(-2)          # query: values below -1 leave the setting
    if cap < 0:
        cp = _lib.c_params(bsk.params)
        cap = int(L.hwb_fft_cluster_capacity(ctypes.byref(cp)))
    return B <= cap


def pbs_batch(params: HeParams, lwe, tv, bsk: BootstrapKey, ksk: LweKeySwitchKey | None,
              out=None, workspace: PbsWorkspace | None = None, engine: str = "auto", ladder: str = "auto"):
    """Programmable bootstrapping of a batch: (B, n+1) -> (B, n+1) (or (B, N+1)
    without a key-switch key).  tv is (2, N) shared or (B, 2, N) per item.
    engine selects the key switch ("auto" | "tc" | "simt", see lwe_keyswitch),
    ladder the blind rotation ("auto" | "fft" | "ntt", see _use_fft_ladder)."""
    t = to_device(lwe)
    if t.dim() != 2 or t.shape[1] != params.lwe_n + 1:
        raise TfheError(f"LWE batch must be (B, {params.lwe_n + 1})")
    B = t.shape[0]
    tvt = to_device(tv)
    if tvt.dim() == 2:
        if tvt.shape != (2, params.n):
            raise TfheError(f"test polynomial must be (2, {params.n})")
        per_item = 0
    elif tvt.dim() == 3 and tvt.shape == (B, 2, params.n):
        per_item = 1
    else:
        raise TfheError("test polynomial must be (2, N) or (B, 2, N)")
    if bsk.count != params.lwe_n:
        raise TfheError(f"bootstrapping key has {bsk.count} GGSWs, params want {params.lwe_n}")
    width = params.lwe_n + 1 if ksk is not None else params.n + 1
    if out is None:
        out = torch.empty((B, width), dtype=torch.int32, device=t.device)
    cp = _lib.c_params(params)
    if _use_fft_ladder(bsk, B, ladder):
        ks_tc = _ks_engine(params, ksk, engine)
        if ksk is not None and not ks_tc:
            # the FFT ladder pairs with the tensor-core key switch; the integer-pipe
            # one runs as a separate pass
            ext = pbs_batch(params, t, tvt, bsk, None, workspace=workspace, ladder="fft")
            return _wrap(lwe, lwe_keyswitch(params, ext, ksk, out=out, engine=engine, workspace=workspace))
        ws = _ws(workspace).get(params, B, t.device, kind="pbs_fft_ks" if ks_tc else "pbs_fft")
        _lib.check(_lib.load().hwb_pbs_fft(ctypes.byref(cp), _ptr(bsk.fft),
                                           _ptr(ksk.tensor_core_tiles() if ks_tc else None), _ptr(tvt), per_item,
                                           _ptr(t), _ptr(out), B, _ptr(ws), _stream()))
    elif _ks_engine(params, ksk, engine):
        ws = _ws(workspace).get(params, B, t.device, kind="pbs_tc")
        _lib.check(_lib.load().hwb_pbs_tc(ctypes.byref(cp), _ptr(bsk.ntt.data), _ptr(ksk.tensor_core_tiles()),
                                          _ptr(tvt), per_item, _ptr(t), _ptr(out), B, _ptr(ws), _stream()))
    else:
        ws = _ws(workspace).get(params, B, t.device) if ksk is not None else None
        _lib.check(_lib.load().hwb_pbs(ctypes.byref(cp), _ptr(bsk.ntt.data), _ptr(ksk.data if ksk else None),
                                       _ptr(tvt), per_item, _ptr(t), _ptr(out), B, _ptr(ws), _stream()))
    return _wrap(lwe, out)
