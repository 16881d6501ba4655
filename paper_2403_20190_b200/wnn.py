"""WiSARD geometry, input encoding and the client-side scoring tail.

Mirrors the parts of the reference's `hewisard.wnn` (`pkg/src/hewisard/wnn.py`)
that encrypted training/inference and the client need: geometry
(`wnn.py:26-60`), the recorded-PRNG permutation (`wnn.py:189-196`), addresses
(`wnn.py:209-219`), thermometer encoding (`wnn.py:158-182`) and the activation /
balancing / argmax tail (`wnn.py:86-109, 241-293`), and the plaintext integer
trainer/evaluator (`wnn.py:222-238, 296-309`) that a decrypted model is checked
against.  The plaintext WiSARD is not part of the accelerated path.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from .tfhe import make_rng

DEFAULT_BLOG_BOUND = 4


class WnnError(ValueError):
    pass


@dataclass(frozen=True)
class WisardGeometry:
    """Shape of one WiSARD classifier (hw/wnn.py:26-60)."""

    s: int          # input bit size
    l: int          # class count
    a: int          # address size (bits per RAM)
    r: int          # permutation seed
    p: int          # counter modulus (power of two)

    def __post_init__(self):
        if self.l < 2:
            raise WnnError("need at least two classes")
        if self.s < 1 or self.a < 1:
            raise WnnError("input size and address size must be positive")
        if self.p < 2 or self.p & (self.p - 1):
            raise WnnError("counter modulus must be a power of two")

    @property
    def k0(self) -> int:
        return -(-self.s // self.a)

    @property
    def label_bits(self) -> int:
        return max(1, (self.l - 1).bit_length())

    @property
    def selector_bits(self) -> int:
        return self.label_bits + self.a

    @property
    def pad(self) -> int:
        return self.k0 * self.a - self.s


@dataclass
class ClassCounts:
    counts: np.ndarray

    @property
    def total(self) -> int:
        return int(self.counts.sum())


@dataclass(frozen=True)
class ActivationSpec:
    """RAM output activation (hw/wnn.py:86-109)."""

    kind: str
    thr: int = 0
    c: int = DEFAULT_BLOG_BOUND

    def __post_init__(self):
        if self.kind not in ("bin", "log", "b-log"):
            raise WnnError(f"unknown activation {self.kind!r}")
        if self.kind == "bin" and self.thr < 0:
            raise WnnError("bin threshold must be non-negative")
        if self.kind == "b-log" and self.c <= 0:
            raise WnnError("b-log bound must be positive")

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if self.kind == "bin":
            return (x > self.thr).astype(np.float64)
        y = np.log2(x + 1.0)
        if self.kind == "b-log":
            y = np.minimum(y, float(self.c))
        return y


def thermometer_thresholds(kind: str, size: int, value_range: int) -> np.ndarray:
    """hw/wnn.py:158-176."""
    if size < 1:
        raise WnnError("thermometer size must be positive")
    if kind == "lin":
        t = np.floor((np.arange(size) + 1) * value_range / (size + 1)).astype(np.int64)
    elif kind == "log":
        t = np.rint(np.power(float(value_range), np.arange(size) / size)).astype(np.int64)
    else:
        raise WnnError(f"unknown thermometer type {kind!r}")
    for i in range(1, size):
        if t[i] <= t[i - 1]:
            t[i] = t[i - 1] + 1
    return t


def thermometer_encode(v, thresholds: np.ndarray) -> np.ndarray:
    """hw/wnn.py:179-182: one bit per threshold, (..., f) -> (..., f, T)."""
    v = np.asarray(v)
    return (v[..., np.newaxis] >= thresholds).astype(np.uint8)


def encode_bits(values: np.ndarray, therm_size: int, value_range: int = 256, kind: str = "lin") -> np.ndarray:
    """Thermometer-encode integer features (n, f) -> bits (n, f*T) (hw/data.py:205-218
    with quant_kind "none")."""
    t = thermometer_thresholds(kind, therm_size, value_range)
    return thermometer_encode(values, t).reshape(len(values), -1)


def quantize_tabular(raw: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """hw/data.py:180-182: min-max scale to 8-bit integers."""
    span = np.where(hi > lo, hi - lo, 1.0)
    return np.clip((raw - lo) / span * 255, 0, 255).astype(np.int64)


@lru_cache(maxsize=64)
def _permutation_cached(r: int, s: int) -> np.ndarray:
    rng = make_rng(r)
    perm = np.arange(s)
    for i in range(s - 1, 0, -1):
        j = int(rng.integers(0, i + 1))
        perm[i], perm[j] = perm[j], perm[i]
    perm.setflags(write=False)
    return perm


def permutation(r: int, s: int) -> np.ndarray:
    """Deterministic Fisher-Yates shuffle of [0, s) from the recorded PRNG
    (hw/wnn.py:189-196); memoised per (r, s) -- the Python-level shuffle of a
    2352-bit input costs milliseconds and every selector build needs it."""
    return _permutation_cached(int(r), int(s)).copy()


def addresses(bits: np.ndarray, geometry: WisardGeometry) -> np.ndarray:
    """Permuted RAM addresses (n, s) -> (n, k0) (hw/wnn.py:209-219)."""
    bits = np.atleast_2d(bits)
    if bits.shape[-1] != geometry.s:
        raise WnnError(f"expected {geometry.s} input bits, got {bits.shape[-1]}")
    perm = permutation(geometry.r, geometry.s)
    px = bits[:, perm]
    if geometry.pad:
        px = np.hstack([px, np.zeros((len(px), geometry.pad), dtype=bits.dtype)])
    px = px.reshape(len(px), geometry.k0, geometry.a).astype(np.int64)
    return px @ (1 << np.arange(geometry.a, dtype=np.int64))


def train_integer(bits: np.ndarray, labels: np.ndarray, geometry: WisardGeometry):
    """Plaintext integer WiSARD (hw/wnn.py:222-238): counters (l, k0, 2^a) mod p
    and class counts -- what a correctly trained encrypted model decrypts to."""
    labels = np.asarray(labels, dtype=np.int64)
    counters = np.zeros((geometry.l, geometry.k0, 1 << geometry.a), dtype=np.int64)
    counts = ClassCounts(np.zeros(geometry.l, dtype=np.int64))
    if labels.size == 0:
        return counters, counts
    if labels.max() >= geometry.l:
        raise WnnError(f"label {labels.max()} out of range for {geometry.l} classes")
    addr = addresses(bits, geometry)
    rams = np.broadcast_to(np.arange(geometry.k0), addr.shape)
    lab = np.broadcast_to(labels[:, np.newaxis], addr.shape)
    np.add.at(counters, (lab, rams, addr), 1)
    counters &= geometry.p - 1
    counts.counts += np.bincount(labels, minlength=geometry.l)
    return counters, counts


def evaluate_dataset(counters: np.ndarray, geometry: WisardGeometry, bits: np.ndarray, spec: ActivationSpec,
                     counts: ClassCounts | None = None) -> np.ndarray:
    """Predicted classes for many samples (hw/wnn.py:296-309)."""
    x = counters.astype(np.float64)
    if counts is not None:
        x = x * rescale_factors(counts, geometry.l)[:, None, None]
    act_t = np.ascontiguousarray(spec.apply(x).transpose(1, 2, 0))          # (k0, 2^a, l)
    addr = addresses(bits, geometry)
    gathered = act_t[np.arange(geometry.k0)[None, :], addr, :]
    return np.argmax(gathered.sum(axis=1), axis=1)


def rescale_factors(counts: ClassCounts, l: int) -> np.ndarray:
    """hw/wnn.py:241-247."""
    c = counts.counts.astype(np.float64)
    if np.any(c <= 0):
        raise WnnError("balancing requires at least one sample of every class")
    return (c.sum() / l) / c


def scores_from_lookups(raw: np.ndarray, spec: ActivationSpec, counts: ClassCounts | None = None) -> np.ndarray:
    """hw/wnn.py:273-280."""
    x = raw.astype(np.float64)
    if counts is not None:
        x = x * rescale_factors(counts, raw.shape[0])[:, np.newaxis]
    return spec.apply(x).sum(axis=1)


def predict_from_lookups(raw: np.ndarray, spec: ActivationSpec, counts: ClassCounts | None = None) -> int:
    """hw/wnn.py:283-286 (argmax breaks ties at the lowest class)."""
    return int(np.argmax(scores_from_lookups(raw, spec, counts)))


__all__ = ["WnnError", "WisardGeometry", "ClassCounts", "ActivationSpec", "thermometer_thresholds",
           "thermometer_encode", "encode_bits", "quantize_tabular", "permutation", "addresses",
           "rescale_factors", "scores_from_lookups", "predict_from_lookups", "train_integer",
           "evaluate_dataset"]
