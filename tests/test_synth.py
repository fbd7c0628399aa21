"""Synthetic generator (vfsynth): determinism, row-addressability and the
noise statistics of Eq. 10."""
import dataclasses
import math

import numpy as np
import pytest

import vfsynth


def test_deterministic_and_seed_sensitive():
    s = vfsynth.config("C2")
    a = vfsynth.make_image(s, 0)[1]
    b = vfsynth.make_image(s, 0)[1]
    c = vfsynth.make_image(s, 1)[1]
    d = vfsynth.make_image(dataclasses.replace(s, seed=s.seed + 1), 0)[1]
    assert a.dtype == np.uint8 and a.shape == (512, 512, 3)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c) and not np.array_equal(a, d)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_row_bands_equal_full_image(name):
    s = vfsynth.config(name)
    if name == "C3":
        s = dataclasses.replace(s, H=256, W=200)
    c, x = vfsynth.make_image(s, 0)
    for r0, r1 in [(0, 7), (13, 51), (s.H - 9, s.H)]:
        cb, xb = vfsynth.make_image(s, 0, r0, r1)
        assert np.array_equal(cb, c[r0:r1]) and np.array_equal(xb, x[r0:r1])


def _sigma3(p, n):
    return 3 * math.sqrt(p * (1 - p) / n)


@pytest.mark.parametrize("p", [0.1, 0.2, 0.3, 0.4])
@pytest.mark.parametrize("model", ["uncorrelated", "correlated"])
def test_noise_rates_within_3_sigma(p, model):
    s = vfsynth.ImageSpec("t", 512, 512, 1, (3,), 8, False, model, p, seed=77)
    clean = vfsynth.clean_rows(s, 0)
    noisy = vfsynth.noisy_rows(s, 0, clean)
    n = 512 * 512
    if model == "uncorrelated":
        # channel replaced w.p. p; a replaced channel keeps its value w.p. 1/256
        q = p * (1 - 1 / 256)
        frac = (noisy != clean).mean()
        assert abs(frac - q) <= _sigma3(q, 3 * n)
    else:
        # whole pixel replaced w.p. p; unchanged only if all 3 draws hit (prob ~0)
        frac = (noisy != clean).any(-1).mean()
        q = p * (1 - 1 / 256 ** 3)
        assert abs(frac - q) <= _sigma3(q, n)
        # the 3 channels of a changed pixel are independent uniform bytes
        ch = noisy[(noisy != clean).any(-1)].astype(np.float64)
        assert abs(ch.mean() - 127.5) < 1.0


def test_phi_zero_is_identity():
    s = vfsynth.ImageSpec("t", 64, 64, 1, (3,), 4, True, "correlated", 0.0, seed=1)
    c, x = vfsynth.make_image(s, 0)
    assert np.array_equal(c, x)


def test_correlated_phik_patterns():
    """phi = 0.1, phi_k = 0.25: single-channel patterns each 0.25."""
    s = vfsynth.ImageSpec("t", 512, 512, 1, (3,), 8, False, "correlated_phik", 0.1, seed=5)
    c, x = vfsynth.make_image(s, 0)
    diff = x != c
    changed = diff.any(-1)
    frac = changed.mean()
    assert abs(frac - 0.1) <= 0.005 + 0.001
    ncorr = changed.sum()
    single = diff.sum(-1) == 1
    for k in range(3):
        f = (single & diff[..., k]).sum() / ncorr
        assert abs(f - 0.25) <= 0.02


def test_c4_probabilities_drawn_from_choices():
    s = vfsynth.config("C4")
    ps = [vfsynth.image_p(s, i) for i in range(1024)]
    assert set(ps) == {0.05, 0.10, 0.20, 0.30}
    counts = np.array([ps.count(v) for v in (0.05, 0.10, 0.20, 0.30)])
    assert np.all(np.abs(counts - 256) <= 3 * math.sqrt(1024 * 0.25 * 0.75))


def test_c1_rectangles_only_and_smooth_background():
    s = vfsynth.config("C1")
    c, _ = vfsynth.make_image(s, 0)
    # bilinear background: neighbouring background pixels differ by at most
    # a few levels; objects are flat
    d = np.abs(np.diff(c.astype(int), axis=1)).max(-1)
    assert np.median(d) <= 4
    assert all(o[0] == "rect" for o in vfsynth._objects(s, 0))


def test_mixed_model_gaussian_then_correlated():
    """P:263 mixed model: Gaussian (sigma per channel, rounded, clamped) then
    correlated impulsive with phi_k.  sigma = 0 equals the correlated_phik
    image bit for bit; without impulses the residual of a
    mid-grey image is N(0, sigma^2) rounded (mean ~0, std ~sigma, symmetric)."""
    base = dict(H=256, W=256, batch=1, window=(3,), n_objects=0, rects_only=True, p=0.1, seed=9)
    s0 = vfsynth.ImageSpec("t", noise="mixed", sigma=0.0, **base)
    sc = vfsynth.ImageSpec("t", noise="correlated_phik", **base)
    assert np.array_equal(vfsynth.make_image(s0, 0)[1], vfsynth.make_image(sc, 0)[1])
    sg = vfsynth.ImageSpec("t", noise="mixed", sigma=10.0, **dict(base, p=0.0))
    c, x = vfsynth.make_image(sg, 0)
    interior = (c > 40) & (c < 215)             # away from the clamps
    r = (x.astype(np.float64) - c)[interior]
    assert abs(r.mean()) < 0.1
    assert abs(r.std() - math.sqrt(100.0 + 1.0 / 12.0)) < 0.15   # rounding adds 1/12
    assert abs(np.mean(r > 0) - np.mean(r < 0)) < 0.01
    # row bands of the mixed model equal the full image (counter-based RNG)
    sm = vfsynth.ImageSpec("t", noise="mixed", **base)
    full = vfsynth.make_image(sm, 0)[1]
    assert np.array_equal(vfsynth.make_image(sm, 0, 100, 180)[1], full[100:180])
