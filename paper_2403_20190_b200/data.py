"""Seeded synthetic datasets standing in for the BASELINE.json training configs.

MNIST/HAM10000 are absent; these generators reproduce the
shapes, sizes and value distributions BASELINE.json describes.  None of the
public datasets' items are reproduced.  Preprocessing follows the reference:
min-max 8-bit quantisation for tabular data (`hw/data.py:180-182`) and linear
thermometer encoding (`hw/wnn.py:158-182`).

  cfg1  2 classes, 64 samples x 30 features ~ N(+-1, 1), 4-bit thermometer -> 120 bits
  cfg3  28x28 grey, 10 classes, 3 Gaussian blobs per class prototype (amplitude 255),
        N(0, 30^2) noise, +-2 px shift, clip; 3-bit thermometer -> 2352 bits
  cfg4  as cfg3 (16384 train + 2048 test)
  cfg5  28x28x3 RGB, 7 classes with frequencies .67/.11/.11/.05/.03/.02/.01, per-class
        channel means U[60,200], 2-D sinusoid texture, N(0, 25^2); 2-bit thermometer
        per channel -> 4704 bits
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import wnn


@dataclass
class BitDataset:
    bits: np.ndarray        # (n, s) uint8
    labels: np.ndarray      # (n,) int64
    classes: int


def _blob_prototypes(rng, classes: int, size: int = 28) -> np.ndarray:
    yy, xx = np.mgrid[0:size, 0:size].astype(np.float64)
    protos = np.zeros((classes, size, size))
    for c in range(classes):
        for _ in range(3):
            mx, my = rng.uniform(6, size - 6, 2)
            sd = rng.uniform(2.0, 5.0)
            protos[c] += 255.0 * np.exp(-((xx - mx) ** 2 + (yy - my) ** 2) / (2 * sd * sd))
    return protos


def _shift(img: np.ndarray, dy: int, dx: int) -> np.ndarray:
    out = np.zeros_like(img)
    h, w = img.shape[:2]
    ys, yd = (slice(0, h - dy), slice(dy, h)) if dy >= 0 else (slice(-dy, h), slice(0, h + dy))
    xs, xd = (slice(0, w - dx), slice(dx, w)) if dx >= 0 else (slice(-dx, w), slice(0, w + dx))
    out[yd, xd] = img[ys, xs]
    return out


def grey_images(n: int, seed: int, classes: int = 10, proto_seed: int = 0):
    """cfg3/cfg4 generator: (n, 28, 28) uint8 images and labels."""
    protos = _blob_prototypes(np.random.default_rng(proto_seed), classes)
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, classes, n)
    imgs = np.empty((n, 28, 28), dtype=np.uint8)
    for i in range(n):
        dy, dx = rng.integers(-2, 3, 2)
        img = _shift(protos[labels[i]], int(dy), int(dx)) + rng.normal(0.0, 30.0, (28, 28))
        imgs[i] = np.clip(img, 0, 255).astype(np.uint8)
    return imgs, labels


def rgb_images(n: int, seed: int, proto_seed: int = 0):
    """cfg5 generator: (n, 28, 28, 3) uint8 images, skewed 7-class labels."""
    freqs = np.array([0.67, 0.11, 0.11, 0.05, 0.03, 0.02, 0.01])
    prng = np.random.default_rng(proto_seed)
    means = prng.uniform(60, 200, (7, 3))
    fx, fy = prng.uniform(0.1, 0.8, (2, 7))
    phase = prng.uniform(0, 2 * np.pi, 7)
    yy, xx = np.mgrid[0:28, 0:28].astype(np.float64)
    rng = np.random.default_rng(seed)
    labels = rng.choice(7, size=n, p=freqs / freqs.sum())
    imgs = np.empty((n, 28, 28, 3), dtype=np.uint8)
    for i in range(n):
        c = labels[i]
        tex = 40.0 * np.sin(fx[c] * xx + fy[c] * yy + phase[c])
        img = means[c][None, None, :] + tex[:, :, None] + rng.normal(0.0, 25.0, (28, 28, 3))
        imgs[i] = np.clip(img, 0, 255).astype(np.uint8)
    return imgs, labels


def tabular(n: int, seed: int, features: int = 30):
    """cfg1 generator: (n, features) float64, 2 classes with means +-1, sigma 1."""
    rng = np.random.default_rng(seed)
    labels = rng.integers(0, 2, n)
    x = rng.normal(0.0, 1.0, (n, features)) + np.where(labels[:, None] == 1, 1.0, -1.0)
    return x, labels


def config_dataset(cfg: int, split: str = "train", n: int | None = None, seed: int = 0) -> BitDataset:
    """Preprocessed bits for BASELINE config `cfg` (1, 3, 4, 5)."""
    test = split == "test"
    if cfg == 1:
        n = n or 64
        x, y = tabular(n, seed + (1 if test else 0))
        lo, hi = x.min(axis=0), x.max(axis=0)          # train bounds (hw/data.py:188-196)
        bits = wnn.encode_bits(wnn.quantize_tabular(x, lo, hi), 4)
        return BitDataset(bits, y, 2)
    if cfg in (3, 4):
        n = n or ({3: 1024, 4: 16384}[cfg] if not test else 2048)
        imgs, y = grey_images(n, seed + (7 if test else 0))
        bits = wnn.encode_bits(imgs.reshape(n, -1).astype(np.int64), 3)
        return BitDataset(bits, y, 10)
    if cfg == 5:
        n = n or (4096 if not test else 1024)
        imgs, y = rgb_images(n, seed + (7 if test else 0))
        bits = wnn.encode_bits(imgs.reshape(n, -1).astype(np.int64), 2)
        return BitDataset(bits, y, 7)
    raise ValueError(f"no synthetic generator for config {cfg}")


# WiSARD geometry (s, l, a, r, p) and parameter set of each training config
CONFIG_GEOMETRY = {
    1: ((120, 2, 4, 7, 16), "CFG1"),
    3: ((2352, 10, 12, 7, 256), "CFG3"),
    4: ((2352, 10, 16, 7, 4096), "CFG4"),
    5: ((4704, 7, 14, 7, 1024), "CFG5"),
}
