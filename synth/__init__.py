"""Seeded synthetic workloads for the five BASELINE.json configs.

This module holds NONE of the method's arithmetic: it only draws images. Both the
oracle (`oracle/`) and the CUDA path (through `paper_1811_06378_b200`) consume
these arrays; neither imports the other.

Recipe: every image is drawn from
``numpy.random.Generator(PCG64(SeedSequence([BASE_SEED, config_id, image_index])))``.
The paper uses no public dataset (PAPER.md has no experiments), so
these synthetic images stand in for its figures' example images.
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 1811063780

# id -> (description, batch, h, w, dtype, mode)
CONFIGS = {
    1: dict(name="c1_quadrant_u8_256", batch=1, h=256, w=256, dtype="u8", mode="quadrant"),
    2: dict(name="c2_full_f32_1024", batch=1, h=1024, w=1024, dtype="f32", mode="full"),
    3: dict(name="c3_full_u8_64x512", batch=64, h=512, w=512, dtype="u8", mode="full"),
    4: dict(name="c4_range_f32_4096", batch=1, h=4096, w=4096, dtype="f32", mode="range",
             theta_min=-15.0, theta_max=15.0),
    5: dict(name="c5_full_f32_16x2048", batch=16, h=2048, w=2048, dtype="f32", mode="full"),
}


def rng_for(config_id: int, image_index: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, config_id, image_index])))


def _border_point(t: float, P: int) -> tuple[float, float]:
    """Point at perimeter parameter t in [0, 4(P-1)) walking the border clockwise."""
    L = P - 1
    if t < L:
        return t, 0.0
    if t < 2 * L:
        return float(L), t - L
    if t < 3 * L:
        return L - (t - 2 * L), float(L)
    return 0.0, L - (t - 3 * L)


def _dda(x0: float, y0: float, x1: float, y1: float):
    n = int(max(abs(x1 - x0), abs(y1 - y0))) + 1
    ts = np.linspace(0.0, 1.0, n) if n > 1 else np.zeros(1)
    xs = np.floor(x0 + (x1 - x0) * ts + 0.5).astype(np.int64)
    ys = np.floor(y0 + (y1 - y0) * ts + 0.5).astype(np.int64)
    return xs, ys


def image_c1(index: int = 0) -> np.ndarray:
    """C1: 256x256 uint8, i.i.d. uniform [0,255]."""
    return rng_for(1, index).integers(0, 256, size=(256, 256), dtype=np.uint8)


def image_c2(P: int = 1024, index: int = 0) -> np.ndarray:
    """C2: N(0, 0.1) noise plus 50 rasterised lines of intensity 1.0, endpoints uniform on the border."""
    g = rng_for(2, index)
    img = g.normal(0.0, 0.1, size=(P, P))
    for _ in range(50):
        ta, tb = g.uniform(0, 4 * (P - 1), size=2)
        (xa, ya), (xb, yb) = _border_point(ta, P), _border_point(tb, P)
        xs, ys = _dda(xa, ya, xb, yb)
        ok = (xs >= 0) & (xs < P) & (ys >= 0) & (ys < P)
        np.add.at(img, (ys[ok], xs[ok]), 1.0)
    return img.astype(np.float32)


def image_c3(index: int, P: int = 512) -> np.ndarray:
    """C3: Bernoulli(0.05) edge map plus 3..8 near-horizontal lines (|angle| < 10 deg)."""
    g = rng_for(3, index)
    img = (g.random((P, P)) < 0.05).astype(np.uint8)
    for _ in range(int(g.integers(3, 9))):
        a = math.radians(g.uniform(-10.0, 10.0))
        y0 = g.uniform(0, P)
        xs = np.arange(P)
        ys = np.floor(y0 + xs * math.tan(a) + 0.5).astype(np.int64)
        ok = (ys >= 0) & (ys < P)
        img[ys[ok], xs[ok]] = 1
    return img


def image_c4(P: int = 4096, index: int = 0) -> np.ndarray:
    """C4: uniform [0,1) float32."""
    return rng_for(4, index).random((P, P), dtype=np.float32)


def image_c5(index: int, P: int = 2048) -> np.ndarray:
    """C5: sum of 20 Gaussian ellipses (phantom-like), normalised to max 1, float32.

    Evaluated in float64 row-blocks; each ellipse: centre U[0.1P,0.9P]^2, semi-axes
    U[P/64, P/4], angle U[0, pi), amplitude U[0.1, 1], value A*exp(-((u/a)^2+(v/b)^2)/2).
    """
    g = rng_for(5, index)
    params = []
    for _ in range(20):
        cx, cy = g.uniform(0.1 * P, 0.9 * P, size=2)
        a, b = g.uniform(P / 64, P / 4, size=2)
        th = g.uniform(0.0, math.pi)
        amp = g.uniform(0.1, 1.0)
        params.append((cx, cy, a, b, th, amp))
    img = np.zeros((P, P), dtype=np.float64)
    xs = np.arange(P, dtype=np.float64)[None, :]
    blk = 256
    for y0 in range(0, P, blk):
        ys = np.arange(y0, min(P, y0 + blk), dtype=np.float64)[:, None]
        acc = np.zeros((ys.shape[0], P))
        for cx, cy, a, b, th, amp in params:
            dx, dy = xs - cx, ys - cy
            c, s = math.cos(th), math.sin(th)
            u = (c * dx + s * dy) / a
            v = (-s * dx + c * dy) / b
            acc += amp * np.exp(-0.5 * (u * u + v * v))
        img[y0:y0 + blk] = acc
    return (img / img.max()).astype(np.float32)


def batch(config_id: int, count: int | None = None, first: int = 0) -> np.ndarray:
    """[B][h][w] array for a config: images first .. first+B-1 (B = the config's batch, or `count`).
    `first` selects another rank's images under weak scaling (paper_1811_06378_b200.sharding)."""
    cfg = CONFIGS[config_id]
    n = cfg["batch"] if count is None else min(count, cfg["batch"])
    idx = range(first, first + n)
    gen = {1: lambda i: image_c1(i), 2: lambda i: image_c2(index=i), 3: image_c3, 4: lambda i: image_c4(index=i),
           5: image_c5}
    if config_id not in gen:
        raise ValueError(config_id)
    return np.stack([gen[config_id](i) for i in idx])


def random_image(shape, dtype: str, seed: int, density: float | None = None, bound: int | None = None) -> np.ndarray:
    """Small seeded random image for unit/parity tests: u8 / i32 in [0,255], f32 N(0,1); "i32w": int32
    uniform in [-bound, bound] (signed, large magnitudes; the caller picks a bound its sums fit in)."""
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, 99, seed])))
    if dtype == "i32w":
        return g.integers(-bound, bound + 1, size=shape).astype(np.int32)
    if dtype == "u8":
        a = g.integers(0, 256, size=shape, dtype=np.uint8)
        if density is not None:
            a = (g.random(shape) < density).astype(np.uint8)
        return a
    if dtype == "i32":
        return g.integers(0, 256, size=shape).astype(np.int32)
    if dtype == "f32":
        return g.normal(0.0, 1.0, size=shape).astype(np.float32)
    raise ValueError(dtype)
