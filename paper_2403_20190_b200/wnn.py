"""Plaintext WiSARD glue needed around the encrypted path (NOT accelerated).

Semantics restated from the reference's `hewisard.wnn`
(`/root/reference/pkg/src/hewisard/wnn.py`; cited per item below) -- written
independently here because the reference package is not present on the GPU box.
Only what the encrypted pipeline and its client tail consume is kept:

* the geometry of a classifier and the seeded input permutation (selector
  construction of encrypted training/inference),
* the activation / balancing / argmax tail the client runs after decryption,
* the plaintext integer trainer and dataset evaluator, used only to CHECK that
  a decrypted encrypted model (and encrypted predictions) equal the plaintext
  semantics,
* thermometer encoding of the synthetic BASELINE workloads.

Everything else of `hewisard.wnn` (PreprocessSpec, f_comp, merge, CLI helpers)
is out of scope.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, field

import numpy as np

from .tfhe import make_rng

__all__ = ["WnnError", "WisardGeometry", "ClassCounts", "IntegerWisardModel", "ActivationSpec",
           "thermometer_thresholds", "thermometer_encode", "encode_bits", "quantize_tabular", "permutation",
           "addresses", "rescale_factors", "scores_from_lookups", "predict_from_lookups", "train_integer",
           "evaluate_dataset"]

BLOG_BOUND = 4          # default upper bound of the bounded-log activation (hw/wnn.py:19)


class WnnError(ValueError):
    """Geometry / encoding / label errors (the reference's WnnError, hw/wnn.py:22)."""


@dataclass(frozen=True)
class WisardGeometry:
    """s input bits, l classes, a address bits per RAM, permutation seed r,
    counter modulus p (hw/wnn.py:26-60)."""

    s: int
    l: int
    a: int
    r: int
    p: int

    def __post_init__(self):
        problems = []
        if self.l < 2:
            problems.append("a classifier needs two or more classes")
        if min(self.s, self.a) <= 0:
            problems.append("input and address sizes have to be >= 1")
        if self.p < 2 or bin(self.p).count("1") != 1:
            problems.append(f"counter modulus {self.p} is not a power of two >= 2")
        if problems:
            raise WnnError("; ".join(problems))

    @property
    def k0(self) -> int:                # RAMs per discriminator: ceil(s / a)
        return (self.s + self.a - 1) // self.a

    @property
    def label_bits(self) -> int:        # bits that index a class (at least one)
        return max(1, int(self.l - 1).bit_length())

    @property
    def selector_bits(self) -> int:     # selector of one (label, address) entry
        return self.a + self.label_bits

    @property
    def pad(self) -> int:               # zero bits appended to fill the last RAM
        return self.a * self.k0 - self.s


@dataclass
class ClassCounts:
    """Per-class sample counts (hw/wnn.py:63-72)."""

    counts: np.ndarray

    @property
    def total(self) -> int:
        return int(np.sum(self.counts))

    def __add__(self, other: "ClassCounts") -> "ClassCounts":
        return ClassCounts(np.asarray(self.counts) + np.asarray(other.counts))


@dataclass
class IntegerWisardModel:
    """Plaintext counters (l, k0, 2^a) mod p (hw/wnn.py:75-83): what
    `hewnn.decrypt_model` returns."""

    geometry: WisardGeometry
    counters: np.ndarray = field(default=None)

    @classmethod
    def zeros(cls, geometry: WisardGeometry) -> "IntegerWisardModel":
        return cls(geometry, np.zeros((geometry.l, geometry.k0, 2 ** geometry.a), dtype=np.int64))


@dataclass(frozen=True)
class ActivationSpec:
    """RAM output activation (hw/wnn.py:86-109): "bin" is 1 where x > thr,
    "log" is log2(x + 1), "b-log" the same clipped at c."""

    kind: str
    thr: int = 0
    c: int = BLOG_BOUND

    def __post_init__(self):
        if self.kind not in ("bin", "log", "b-log"):
            raise WnnError(f"activation kind {self.kind!r} is not one of bin, log, b-log")
        if self.kind == "bin" and self.thr < 0:
            raise WnnError("the bin activation needs a threshold >= 0")
        if self.kind == "b-log" and self.c <= 0:
            raise WnnError("the b-log activation needs a bound > 0")

    def apply(self, x) -> np.ndarray:
        v = np.asarray(x, dtype=np.float64)
        if self.kind == "bin":
            return np.greater(v, self.thr).astype(np.float64)
        out = np.log2(1.0 + v)
        return out if self.kind == "log" else np.minimum(out, float(self.c))


# ---------------------------------------------------------------------------
# input encoding (synthetic BASELINE workloads)


def thermometer_thresholds(kind: str, size: int, value_range: int) -> np.ndarray:
    """Strictly increasing thresholds (hw/wnn.py:158-176): "lin" splits
    [0, value_range) into size + 1 equal steps, "log" spaces them as
    value_range^(i/size); collisions are pushed up by one."""
    if size <= 0:
        raise WnnError("a thermometer needs at least one threshold")
    i = np.arange(size, dtype=np.float64)
    if kind == "lin":
        raw = np.floor(value_range * (i + 1.0) / (size + 1.0))
    elif kind == "log":
        raw = np.rint(float(value_range) ** (i / size))
    else:
        raise WnnError(f"thermometer kind {kind!r} is not lin or log")
    t = raw.astype(np.int64)
    # t_i = max(raw_i, t_{i-1} + 1), i.e. a running maximum of raw_i - i, shifted back
    return np.maximum.accumulate(t - np.arange(size)) + np.arange(size)


def thermometer_encode(v, thresholds: np.ndarray) -> np.ndarray:
    """(..., f) values -> (..., f, T) bits, bit t set when v >= threshold t (hw/wnn.py:179-182)."""
    return np.greater_equal(np.expand_dims(np.asarray(v), -1), thresholds).astype(np.uint8)


def encode_bits(values: np.ndarray, therm_size: int, value_range: int = 256, kind: str = "lin") -> np.ndarray:
    """Integer features (n, f) -> flattened thermometer bits (n, f * T) (hw/data.py:205-218)."""
    bits = thermometer_encode(values, thermometer_thresholds(kind, therm_size, value_range))
    return bits.reshape(bits.shape[0], -1)


def quantize_tabular(raw: np.ndarray, lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """Min-max scaling of real features to [0, 255] integers (hw/data.py:180-182)."""
    width = np.where(hi > lo, hi - lo, 1.0)
    return np.clip(255.0 * (raw - lo) / width, 0.0, 255.0).astype(np.int64)


# ---------------------------------------------------------------------------
# permutation and addressing


@functools.lru_cache(maxsize=64)
def _perm(r: int, s: int) -> np.ndarray:
    # Fisher-Yates driven by the recorded PRNG: position i (from the top down)
    # swaps with rng.integers(0, i + 1) -- the draw order of hw/wnn.py:189-196
    rng = make_rng(r)
    draws = [int(rng.integers(0, i + 1)) for i in range(s - 1, 0, -1)]
    out = list(range(s))
    for i, j in zip(range(s - 1, 0, -1), draws):
        out[i], out[j] = out[j], out[i]
    arr = np.array(out, dtype=np.int64)
    arr.setflags(write=False)
    return arr


def permutation(r: int, s: int) -> np.ndarray:
    """The input-bit permutation of seed r over s bits (memoised per (r, s))."""
    return np.array(_perm(int(r), int(s)))


def addresses(bits: np.ndarray, geometry: WisardGeometry) -> np.ndarray:
    """(n, s) bits -> (n, k0) RAM addresses: permute, zero-pad to k0 * a, read each
    a-bit group LSB first (hw/wnn.py:209-219)."""
    x = np.atleast_2d(np.asarray(bits))
    if x.shape[-1] != geometry.s:
        raise WnnError(f"samples have {x.shape[-1]} bits, the geometry expects {geometry.s}")
    x = np.pad(x[:, permutation(geometry.r, geometry.s)].astype(np.int64), ((0, 0), (0, geometry.pad)))
    groups = x.reshape(x.shape[0], geometry.k0, geometry.a)
    return np.left_shift(groups, np.arange(geometry.a)).sum(axis=-1)


# ---------------------------------------------------------------------------
# plaintext training / evaluation (the checker of decrypted models) and the client tail


def train_integer(bits: np.ndarray, labels: np.ndarray, geometry: WisardGeometry):
    """Counters (l, k0, 2^a) mod p and class counts of plaintext training
    (hw/wnn.py:222-238), as an (IntegerWisardModel, ClassCounts) pair."""
    y = np.asarray(labels, dtype=np.int64).reshape(-1)
    g = geometry
    if y.size and int(y.max()) >= g.l:
        raise WnnError(f"class label {int(y.max())} does not exist (l = {g.l})")
    model = IntegerWisardModel.zeros(g)
    counts = ClassCounts(np.bincount(y, minlength=g.l).astype(np.int64))
    if y.size:
        addr = addresses(bits, g)                                        # (n, k0)
        cells = (y[:, None] * g.k0 + np.arange(g.k0)[None, :]) * (1 << g.a) + addr
        hist = np.bincount(cells.reshape(-1), minlength=model.counters.size)
        model.counters[...] = (hist.reshape(model.counters.shape) % g.p)
    return model, counts


def rescale_factors(counts: ClassCounts, l: int) -> np.ndarray:
    """Class balancing weights (mean count) / count_c (hw/wnn.py:252-257)."""
    c = np.asarray(counts.counts, dtype=np.float64)
    if (c <= 0).any():
        raise WnnError("class balancing needs every class to have samples")
    return c.sum() / l / c


def scores_from_lookups(raw: np.ndarray, spec: ActivationSpec, counts: ClassCounts | None = None) -> np.ndarray:
    """(l, k0) counter lookups -> (l,) activated class scores (hw/wnn.py:275-281)."""
    x = np.asarray(raw, dtype=np.float64)
    if counts is not None:
        x = rescale_factors(counts, x.shape[0])[:, None] * x
    return spec.apply(x).sum(axis=-1)


def predict_from_lookups(raw: np.ndarray, spec: ActivationSpec, counts: ClassCounts | None = None) -> int:
    """Highest score wins; ties go to the lowest class (hw/wnn.py:284-287)."""
    return int(np.argmax(scores_from_lookups(raw, spec, counts)))


def evaluate_dataset(model, bits: np.ndarray, spec: ActivationSpec, counts: ClassCounts | None = None,
                     chunk: int = 1024, *, geometry: WisardGeometry | None = None) -> np.ndarray:
    """Predicted class of every sample (hw/wnn.py:296-309).  `model` is an
    IntegerWisardModel (reference signature) or a bare (l, k0, 2^a) counter array
    with `geometry` given."""
    if isinstance(model, IntegerWisardModel):
        g, counters = model.geometry, model.counters
    else:
        if geometry is None:
            raise WnnError("a bare counter array needs geometry=")
        g, counters = geometry, np.asarray(model)
    x = counters.astype(np.float64)
    if counts is not None:
        x = x * rescale_factors(counts, g.l)[:, None, None]
    table = np.moveaxis(spec.apply(x), 0, -1)                            # (k0, 2^a, l)
    bits = np.atleast_2d(bits)
    preds = np.empty(bits.shape[0], dtype=np.int64)
    for lo in range(0, bits.shape[0], chunk):
        addr = addresses(bits[lo: lo + chunk], g)                        # (m, k0)
        votes = table[np.arange(g.k0), addr].sum(axis=1)                 # (m, l)
        preds[lo: lo + addr.shape[0]] = votes.argmax(axis=1)
    return preds
