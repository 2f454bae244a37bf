"""Seeded synthetic inputs for the five BASELINE.json configs.

No public dataset is involved; every input is generated from a
fixed seed with the shapes, dtypes and value distributions BASELINE.json names.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BASE_SEED = 2411_07351


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    batch: int
    dtype: str          # input element type
    acc: str            # accumulator type
    quadrants: tuple    # quadrant names
    tolerance: str      # "bit-exact" or "1e-5*L1"
    description: str


ALL_Q = ("horiz_pos", "horiz_neg", "vert_pos", "vert_neg")

CONFIGS = {
    "c1": Config("c1", 1000, 1, "u8", "i32", ("vert_pos",), "bit-exact",
                 "single 1000x1000 u8 U{0..255}, one quadrant (mostly-vertical positive slope = fht2d(I^T))"),
    "c2": Config("c2", 1024, 1, "u8", "i32", ALL_Q, "bit-exact", "single 1024x1024 u8 U{0..255}, four quadrants"),
    "c3": Config("c3", 3001, 1, "f32", "f32", ALL_Q, "1e-5*L1", "single 3001x3001 f32 N(0,1), four quadrants"),
    "c4": Config("c4", 509, 256, "u8", "i32", ALL_Q, "bit-exact",
                 "256 binary 509x509 edge maps (2% ones + 20 border-to-border segments), four quadrants"),
    "c5": Config("c5", 8191, 1, "f32", "f32", ALL_Q, "1e-5*L1", "single 8191x8191 f32 U[0,1), four quadrants"),
}


def _rng(cfg: str, index: int = 0) -> np.random.Generator:
    return np.random.default_rng([BASE_SEED, int(cfg[1:]), index])


def _border_point(rng, n):
    side = rng.integers(4)
    p = int(rng.integers(n))
    return [(p, 0), (p, n - 1), (0, p), (n - 1, p)][side]


def edge_map(n: int, rng: np.random.Generator, density: float = 0.02, segments: int = 20) -> np.ndarray:
    """Binary u8 edge map: Bernoulli(density) ones plus `segments` one-pixel-wide
    8-connected segments between two uniformly random border points
    ("full-length": endpoints on the image border)."""
    img = (rng.random((n, n)) < density).astype(np.uint8)
    for _ in range(segments):
        (x0, y0), (x1, y1) = _border_point(rng, n), _border_point(rng, n)
        m = max(abs(x1 - x0), abs(y1 - y0)) + 1
        xs = np.rint(np.linspace(x0, x1, m)).astype(np.int64)
        ys = np.rint(np.linspace(y0, y1, m)).astype(np.int64)
        img[ys, xs] = 1
    return img


def make_images(cfg: str, count: int | None = None, offset: int = 0) -> np.ndarray:
    """Images [offset, offset+count) of config `cfg`, shape (count, n, n)."""
    c = CONFIGS[cfg]
    count = c.batch if count is None else count
    n = c.n
    if cfg == "c4":
        return np.stack([edge_map(n, _rng(cfg, offset + i)) for i in range(count)])
    out = []
    for i in range(count):
        rng = _rng(cfg, offset + i)
        if cfg in ("c1", "c2"):
            out.append(rng.integers(0, 256, (n, n), dtype=np.uint8))
        elif cfg == "c3":
            out.append(rng.standard_normal((n, n), dtype=np.float32))
        else:
            out.append(rng.random((n, n), dtype=np.float32))
    return np.stack(out)


def nominal_sums(cfg: str, images: int | None = None) -> int:
    """BASELINE.json's Gsums denominator: Q * imgs * n^2 * ceil(log2 n)."""
    c = CONFIGS[cfg]
    imgs = c.batch if images is None else images
    return len(c.quadrants) * imgs * c.n * c.n * int(np.ceil(np.log2(c.n)))
