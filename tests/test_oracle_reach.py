"""Pins for the SURVEY.md 8(f4) variant VF_MINIMAX_REACH: minimax polynomials
re-derived by the Remez exchange for the criterion values on the
arguments the criteria can reach (z <= z*_25, u <= 1 - 1/e).

The coefficients are data (tests/golden/remez_reach.txt, written by
tools/remez_reach.py); what pins them is mathematics, not the tool:
  * the error against the function (50-digit mpmath, independent of numpy's
    expm1/log1p) has deg + 2 alternating extrema of equal size -- the
    Chebyshev alternation theorem, so no polynomial of that degree does better;
  * that level equals the survey's independent Remez run (App. A11:
    7.9e-8 for exp degree 5, 3.0e-7 for s ln s degree 7);
  * the oracle's C constants are the golden strings, and re-running the tool
    reproduces them;
  * on random windows the reach aggregates stay within (n - 1) eps of the
    exact variant's (the approximation bound applied at the right argument).
"""
import math
import os
import sys

import mpmath as mp
import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
mp.mp.dps = 50
Z_MAX = mp.mpf(25) ** (1 + mp.mpf("0.33") / 3) / 48
U_MAX = 1 - mp.exp(-1)
FUNCS = {
    "exp_reach": (lambda z: 1 - mp.exp(-z), Z_MAX, 5, 7.9e-8),
    "log_reach": (lambda u: -(1 - u) * mp.log(1 - u), U_MAX, 7, 3.0e-7),
}


def _err_grid(name, coeffs, npts):
    f, b, _, _ = FUNCS[name]
    c = [mp.mpf(v) for v in coeffs]
    zs = [b * k / (npts - 1) for k in range(npts)]
    out = []
    for z in zs:
        p = mp.mpf(0)
        for a in reversed(c):
            p = p * z + a
        out.append(float(f(z) - p))
    return np.array([float(z) for z in zs]), np.array(out)


@pytest.mark.parametrize("name", ["exp_reach", "log_reach"])
def test_golden_matches_oracle_constants(name, remez_reach):
    vals = np.array([float(v) for v in remez_reach[name]])
    assert np.array_equal(oracle.coeffs(name), vals)
    assert len(vals) == FUNCS[name][2] + 1


@pytest.mark.parametrize("name", ["exp_reach", "log_reach"])
def test_equioscillation_in_mpmath(name, remez_reach):
    """Chebyshev alternation: deg + 2 extrema of alternating sign and equal
    size (level spread <= 1e-5 relative) -> the best uniform approximation."""
    _, b, deg, survey_eps = FUNCS[name]
    z, e = _err_grid(name, remez_reach[name], 6001)
    s = np.sign(e)
    s[s == 0] = 1
    cuts = np.flatnonzero(np.diff(s) != 0) + 1
    starts, ends = np.concatenate([[0], cuts]), np.concatenate([cuts, [len(e)]])
    ext = np.array([np.abs(e[a:c]).max() for a, c in zip(starts, ends)])
    assert len(ext) == deg + 2
    # refine each extremum's level on a finer local grid is unnecessary: the
    # interior extrema are flat, so a 6001-point grid samples them to 1e-6
    assert (ext.max() - ext.min()) / ext.max() < 1e-5
    eps = float(remez_reach[name + "_eps"][0])
    assert ext.max() == pytest.approx(eps, rel=1e-5)
    assert abs(eps - survey_eps) <= 0.05 * 10 ** math.floor(math.log10(survey_eps))   # App. A11 prints 2 digits
    # the ends of the interval are extrema (Remez endpoints)
    assert abs(e[0]) == pytest.approx(eps, rel=1e-5) and abs(e[-1]) == pytest.approx(eps, rel=1e-5)


@pytest.mark.parametrize("name", ["exp_reach", "log_reach"])
def test_oracle_scalar_eval(name, remez_reach):
    """The oracle's Horner evaluation vs 50-digit mpmath of the same polynomial."""
    f, b, _, _ = FUNCS[name]
    zs = np.linspace(0, float(b), 257)
    got = oracle.eval_fn(name, zs)
    c = [mp.mpf(v) for v in remez_reach[name]]
    for z, g in zip(zs, got):
        p = mp.mpf(0)
        for a in reversed(c):
            p = p * mp.mpf(z) + a
        assert g == pytest.approx(float(p), rel=1e-14, abs=1e-22)
        assert abs(g - float(f(mp.mpf(z)))) <= float(remez_reach[name + "_eps"][0]) * (1 + 1e-6)


def test_tool_reproduces_golden(remez_reach):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import remez_reach as rr  # noqa: E402
    (ce, ee, _), (cl, el, _) = rr.fits()
    np.testing.assert_allclose(ce, [float(v) for v in remez_reach["exp_reach"]], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(cl, [float(v) for v in remez_reach["log_reach"]], rtol=1e-9, atol=1e-15)
    assert float(remez_reach["exp_reach_interval"][1]) == pytest.approx(float(Z_MAX), rel=1e-15)
    assert float(remez_reach["log_reach_interval"][1]) == pytest.approx(float(U_MAX), rel=1e-15)


@pytest.mark.parametrize("n", [9, 25])
@pytest.mark.parametrize("crit", ["exp", "log"])
def test_reach_aggregates_within_bound_of_exact(n, crit, remez_reach):
    """|R_reach - R_exact| <= (n - 1) eps on every window: each of the n - 1
    terms of R_i is the polynomial at the exact variant's argument."""
    eps = float(remez_reach[("exp" if crit == "exp" else "log") + "_reach_eps"][0])
    rng = np.random.default_rng(5 + n)
    for t in range(150):
        s = rng.integers(0, 256, size=(n, 3)).astype(np.uint8)
        if t % 2:
            s[rng.random(n) < 0.6] = s[0]
        _, Re, _ = oracle.window(s, crit, "exact")
        _, Rr, Dr = oracle.window(s, crit, "reach")
        if np.all(Re == 0):
            assert np.all(Rr == 0)        # flat window (R18)
            continue
        assert np.max(np.abs(Rr - Re)) <= (n - 1) * eps * (1 + 1e-9)
        assert np.array_equal(Dr, Dr.T)
