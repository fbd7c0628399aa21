"""Seeded synthetic colour images + impulsive noise (the paper's corpus stand-in).

This module is shared by the CPU oracle tests, the GPU parity tests and
``bench.py``.  It holds NO arithmetic of the filtering method itself (no
distances, criteria, approximants or argmin): it only produces uint8 RGB
inputs.  Both sides of every parity check consume the very same bytes.

Paper context
-------------
* PAPER.md §4 uses 100 internet RGB images, which are not available
  here; BASELINE.json configs 0..4 describe the synthetic stand-in
  (smooth gradients + random rectangles/edges), recipe fixed in DESIGN.md §3.
* Noise models: PAPER.md Eq. 10.
  - uncorrelated impulsive: each channel independently replaced by a uniform
    random value r_k in {0..255} with probability phi_k (= p for all k);
  - correlated impulsive with phi_1 = phi_2 = phi_3 = 0: the whole pixel is
    replaced by a uniform random RGB vector with probability phi (= p)
    (BASELINE.json configs 1 and 4: "whole pixel replaced by random RGB").
  - correlated impulsive with general phi_k (the paper used 0.25) is
    also provided (``noise="correlated_phik"``);
  - mixed ("Gaussian Noise + Correlated Impulsive Noise"): additive
    Gaussian noise of standard deviation ``sigma`` per channel (rounded half
    up, clamped to 0..255), then the correlated_phik model
    (``noise="mixed"``).  The paper never states sigma; 10 is SPEC.md's
    default (flagged S:403) and a parameter here.

RNG
---
Counter-based: every draw is ``mix64`` (the SplitMix64 finaliser) of a key
built from (seed, image_id, stream tag, element index).  Draws are therefore
independent of generation order and any row band of an image can be
generated on its own (the row-stripe partitioner relies on this).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import numpy as np

__all__ = [
    "ImageSpec", "CONFIGS", "config", "make_image", "make_batch", "mix64",
    "uniform01", "draw_u64", "expected_corrupt_fraction",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_TAGMUL = np.uint64(0xD1B54A32D192ED03)

# stream tags (one independent stream per purpose)
TAG_BG = 1          # corner colours
TAG_OBJ = 2         # object geometry + colours
TAG_NOISE_MASK = 3  # per-element corruption decision
TAG_NOISE_VAL = 4   # impulse values
TAG_PSEL = 5        # per-image noise probability choice (config 3)
TAG_PATTERN = 6     # correlated-phik pattern choice
TAG_GAUSS = 7       # mixed model: Gaussian noise (Box-Muller, two draws per element)


def mix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014), vectorised on uint64."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return x


def _stream_key(seed: int, image_id: int, tag: int) -> np.uint64:
    with np.errstate(over="ignore"):
        base = mix64(np.uint64(seed) * _GOLD + np.uint64(image_id))
        return mix64(base ^ (np.uint64(tag) * _TAGMUL))


def draw_u64(seed: int, image_id: int, tag: int, idx) -> np.ndarray:
    """64-bit draw number ``idx`` (array-like of non-negative ints) of a stream."""
    key = _stream_key(seed, image_id, tag)
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(key + (idx + np.uint64(1)) * _GOLD)


def uniform01(seed, image_id, tag, idx) -> np.ndarray:
    """Uniform doubles in [0, 1) with 53 random bits."""
    v = draw_u64(seed, image_id, tag, idx)
    return (v >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def uniform_byte(seed, image_id, tag, idx) -> np.ndarray:
    """Uniform integers in {0..255} (top byte of the draw)."""
    return (draw_u64(seed, image_id, tag, idx) >> np.uint64(56)).astype(np.uint8)


@dataclasses.dataclass(frozen=True)
class ImageSpec:
    """One synthetic workload (a BASELINE.json config)."""
    name: str
    H: int
    W: int
    batch: int
    window: Tuple[int, ...]
    n_objects: int
    rects_only: bool
    noise: str                       # "uncorrelated" | "correlated" | "correlated_phik" | "mixed"
    p: Optional[float]               # fixed corruption probability, or None
    p_choices: Tuple[float, ...] = ()  # per-image choice when p is None
    phi_k: Tuple[float, float, float] = (0.25, 0.25, 0.25)
    seed: int = 10090959
    sigma: float = 10.0              # mixed model only


# BASELINE.json "configs", restated ("768x512" read as
# W x H, reading R15).  Seeds: 1009_0959 + config index.
CONFIGS = {
    "C1": ImageSpec("C1", 64, 64, 1, (3,), 4, True, "uncorrelated", 0.10, seed=10090959 + 0),
    "C2": ImageSpec("C2", 512, 512, 1, (3,), 32, False, "correlated", 0.10, seed=10090959 + 1),
    "C3": ImageSpec("C3", 2048, 2048, 8, (5,), 32, False, "uncorrelated", 0.20, seed=10090959 + 2),
    "C4": ImageSpec("C4", 512, 768, 1024, (3,), 32, False, "uncorrelated", None,
                    p_choices=(0.05, 0.10, 0.20, 0.30), seed=10090959 + 3),
    "C5": ImageSpec("C5", 4320, 7680, 1, (3, 5), 32, False, "correlated", 0.15, seed=10090959 + 4),
}


def config(name: str) -> ImageSpec:
    return CONFIGS[name]


def image_p(spec: ImageSpec, image_id: int) -> float:
    """Corruption probability used for image ``image_id`` of a config."""
    if spec.p is not None:
        return float(spec.p)
    k = int(draw_u64(spec.seed, image_id, TAG_PSEL, 0) % np.uint64(len(spec.p_choices)))
    return float(spec.p_choices[k])


def _objects(spec: ImageSpec, image_id: int):
    """Object list: (kind, y0, x0, y1, x1, cy, cx, cos, sin, rgb)."""
    H, W = spec.H, spec.W
    objs = []
    for k in range(spec.n_objects):
        u = uniform01(spec.seed, image_id, TAG_OBJ, np.arange(k * 16, k * 16 + 8))
        col = uniform_byte(spec.seed, image_id, TAG_OBJ, np.arange(k * 16 + 8, k * 16 + 11))
        y0 = int(u[0] * H)
        x0 = int(u[1] * W)
        hmin, hmax = max(1, H // 16), max(1, H // 3)
        wmin, wmax = max(1, W // 16), max(1, W // 3)
        h = hmin + int(u[2] * (hmax - hmin + 1))
        w = wmin + int(u[3] * (wmax - wmin + 1))
        y1, x1 = min(H, y0 + h), min(W, x0 + w)
        edge = (not spec.rects_only) and (k % 2 == 1)
        theta = u[4] * np.pi
        objs.append(("edge" if edge else "rect", y0, x0, y1, x1,
                     0.5 * (y0 + y1 - 1), 0.5 * (x0 + x1 - 1),
                     float(np.cos(theta)), float(np.sin(theta)), col))
    return objs


def clean_rows(spec: ImageSpec, image_id: int, r0: int = 0, r1: Optional[int] = None) -> np.ndarray:
    """Noise-free rows [r0, r1) of image ``image_id`` as uint8 [r1-r0, W, 3]."""
    H, W = spec.H, spec.W
    r1 = H if r1 is None else r1
    assert 0 <= r0 <= r1 <= H
    corners = uniform_byte(spec.seed, image_id, TAG_BG, np.arange(12)).astype(np.float64).reshape(4, 3)
    ys = np.arange(r0, r1, dtype=np.float64)
    xs = np.arange(W, dtype=np.float64)
    fy = (ys / max(H - 1, 1))[:, None, None]
    fx = (xs / max(W - 1, 1))[None, :, None]
    c00, c01, c10, c11 = corners
    img = ((1 - fy) * (1 - fx) * c00 + (1 - fy) * fx * c01
           + fy * (1 - fx) * c10 + fy * fx * c11)
    img = np.floor(img + 0.5).clip(0, 255).astype(np.uint8)
    yy = np.arange(r0, r1)[:, None]
    xx = np.arange(W)[None, :]
    for kind, y0, x0, y1, x1, cy, cx, c, s, col in _objects(spec, image_id):
        lo, hi = max(y0, r0), min(y1, r1)
        if lo >= hi:
            continue
        sub = img[lo - r0:hi - r0, x0:x1]
        if kind == "rect":
            sub[...] = col
        else:
            ys_ = yy[lo - r0:hi - r0]
            xs_ = xx[:, x0:x1]
            m = (xs_ - cx) * c + (ys_ - cy) * s > 0
            sub[m] = col
    return img


def noisy_rows(spec: ImageSpec, image_id: int, clean: np.ndarray, r0: int = 0) -> np.ndarray:
    """Apply the config's impulsive noise (Eq. 10) to clean rows starting at r0."""
    rows, W = clean.shape[0], clean.shape[1]
    p = image_p(spec, image_id)
    pix = (np.arange(r0, r0 + rows, dtype=np.uint64)[:, None] * np.uint64(W)
           + np.arange(W, dtype=np.uint64)[None, :])
    out = clean.copy()
    if spec.noise == "uncorrelated":
        el = pix[..., None] * np.uint64(3) + np.arange(3, dtype=np.uint64)[None, None, :]
        m = uniform01(spec.seed, image_id, TAG_NOISE_MASK, el) < p
        v = uniform_byte(spec.seed, image_id, TAG_NOISE_VAL, el)
        out[m] = v[m]
    elif spec.noise == "correlated":
        m = uniform01(spec.seed, image_id, TAG_NOISE_MASK, pix) < p
        el = pix[..., None] * np.uint64(3) + np.arange(3, dtype=np.uint64)[None, None, :]
        v = uniform_byte(spec.seed, image_id, TAG_NOISE_VAL, el)
        out[m] = v[m]
    elif spec.noise in ("correlated_phik", "mixed"):
        if spec.noise == "mixed":
            el = pix[..., None] * np.uint64(3) + np.arange(3, dtype=np.uint64)[None, None, :]
            u1 = uniform01(spec.seed, image_id, TAG_GAUSS, el * np.uint64(2))
            u2 = uniform01(spec.seed, image_id, TAG_GAUSS, el * np.uint64(2) + np.uint64(1))
            g = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)    # N(0, 1), u1 in [0, 1)
            out = np.floor(out.astype(np.float64) + spec.sigma * g + 0.5).clip(0, 255).astype(np.uint8)
        m = uniform01(spec.seed, image_id, TAG_NOISE_MASK, pix) < p
        u = uniform01(spec.seed, image_id, TAG_PATTERN, pix)
        f1, f2, f3 = spec.phi_k
        pat = np.where(u < f1, 0, np.where(u < f1 + f2, 1, np.where(u < f1 + f2 + f3, 2, 3)))
        el = pix[..., None] * np.uint64(3) + np.arange(3, dtype=np.uint64)[None, None, :]
        v = uniform_byte(spec.seed, image_id, TAG_NOISE_VAL, el)
        ch = np.arange(3)[None, None, :]
        chm = (pat[..., None] == 3) | (pat[..., None] == ch)
        mm = m[..., None] & chm
        out[mm] = v[mm]
    else:
        raise ValueError(f"unknown noise model {spec.noise!r}")
    return out


def make_image(spec: ImageSpec, image_id: int = 0, r0: int = 0, r1: Optional[int] = None):
    """(clean, noisy) rows [r0, r1) of one image, each uint8 [rows, W, 3]."""
    c = clean_rows(spec, image_id, r0, r1)
    return c, noisy_rows(spec, image_id, c, r0)


def make_batch(spec: ImageSpec, ids=None) -> np.ndarray:
    """Noisy images ``ids`` (default: the whole batch) as uint8 [B, H, W, 3]."""
    ids = range(spec.batch) if ids is None else ids
    return np.stack([make_image(spec, i)[1] for i in ids])


def expected_corrupt_fraction(spec: ImageSpec, p: float) -> float:
    """Expected fraction of pixels that have at least one channel replaced
    (a replaced channel may keep its value by chance; that is ignored here)."""
    if spec.noise == "uncorrelated":
        return 1.0 - (1.0 - p) ** 3
    return p


def random_image(seed: int, H: int, W: int, image_id: int = 0) -> np.ndarray:
    """I.i.d. uniform uint8 RGB image (stress input for parity tests)."""
    idx = np.arange(H * W * 3, dtype=np.uint64)
    return uniform_byte(seed, image_id, 7, idx).reshape(H, W, 3)


def small_palette_image(seed: int, H: int, W: int, levels=(0, 1, 2, 127, 128, 255), image_id: int = 0) -> np.ndarray:
    """Image whose channels take few values: many duplicate samples, exact
    aggregate ties, parallel vectors, zero vectors and c = 0.5 branch points."""
    idx = np.arange(H * W * 3, dtype=np.uint64)
    k = (draw_u64(seed, image_id, 8, idx) % np.uint64(len(levels))).astype(np.int64)
    return np.asarray(levels, dtype=np.uint8)[k].reshape(H, W, 3)
