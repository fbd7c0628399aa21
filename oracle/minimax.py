"""Minimax tooling (TEST INFRASTRUCTURE): dense-grid certification, the Remez
exchange algorithm and an equioscillation check.

PAPER.md section 2: the minimax error is
    eps = max_{z in [a,b]} |f(z) - P(z)|                (Eq. 1)
and the polynomials of Tables 1-2 were computed with the Remez exchange
algorithm ("an iterative method that uses Lagrangian interpolation to
systematically minimize the maximum absolute difference").  The
certification criterion is the measured max error on a
dense uniform grid compared with the paper's printed eps.

Only numpy is used; all evaluation is in double precision, which is ample
for errors of 1e-7 .. 1e-1.
"""
from __future__ import annotations

from typing import Callable, Sequence, Tuple

import numpy as np


def polyval(coeffs: Sequence[float], z: np.ndarray) -> np.ndarray:
    """Horner evaluation of a_0 + a_1 z + ...."""
    z = np.asarray(z, dtype=np.float64)
    r = np.full_like(z, coeffs[-1], dtype=np.float64)
    for a in reversed(coeffs[:-1]):
        r = r * z + a
    return r


def certify(approx: Callable[[np.ndarray], np.ndarray], f: Callable[[np.ndarray], np.ndarray],
            a: float, b: float, npts: int = 2_000_001) -> Tuple[float, float]:
    """Max |f - approx| on a uniform grid of ``npts`` points of [a, b]
    (Eq. 1).  Returns (eps, argmax z)."""
    z = np.linspace(a, b, npts)
    e = np.abs(f(z) - approx(z))
    i = int(np.argmax(e))
    return float(e[i]), float(z[i])


def _alternating_extrema(z: np.ndarray, e: np.ndarray):
    """Indices of the largest |e| on every maximal run of constant sign."""
    s = np.sign(e)
    s[s == 0] = 1
    cuts = np.flatnonzero(np.diff(s) != 0) + 1
    starts = np.concatenate([[0], cuts])
    ends = np.concatenate([cuts, [len(e)]])
    return np.array([st + int(np.argmax(np.abs(e[st:en]))) for st, en in zip(starts, ends)])


def extrema(coeffs: Sequence[float], f: Callable, a: float, b: float, npts: int = 400_001):
    """Alternating error extrema (z_i, e_i) of f - P on [a, b]."""
    z = np.linspace(a, b, npts)
    e = f(z) - polyval(coeffs, z)
    idx = _alternating_extrema(z, e)
    return z[idx], e[idx]


def remez(f: Callable[[np.ndarray], np.ndarray], deg: int, a: float, b: float,
          tol: float = 1e-9, max_iter: int = 60, npts: int = 400_001):
    """Best uniform polynomial approximation of degree ``deg`` on [a, b].

    Classic multi-point exchange (SPEC S:161-166 design): start from the
    deg+2 Chebyshev extreme points, solve the levelled system
        sum_j c_j x_i^j + (-1)^i E = f(x_i),  i = 0..deg+1,
    then replace the reference with the deg+2 alternating extrema of the
    error on a dense grid, until the extrema levels agree within ``tol``.
    Returns (coeffs, eps, iterations).
    """
    m = deg + 2
    k = np.arange(m)
    x = 0.5 * (a + b) - 0.5 * (b - a) * np.cos(np.pi * k / (m - 1))
    grid = np.linspace(a, b, npts)
    fg = f(grid)
    c = None
    for it in range(1, max_iter + 1):
        A = np.hstack([np.vander(x, deg + 1, increasing=True),
                       ((-1.0) ** k)[:, None]])
        sol = np.linalg.solve(A, f(x))
        c = sol[:-1]
        e = fg - polyval(c, grid)
        idx = _alternating_extrema(grid, e)
        while len(idx) > m:
            if abs(e[idx[0]]) < abs(e[idx[-1]]):
                idx = idx[1:]
            else:
                idx = idx[:-1]
        emax = float(np.max(np.abs(e)))
        if len(idx) == m:
            lv = np.abs(e[idx])
            x = grid[idx]
            if (lv.max() - lv.min()) / lv.max() <= tol:
                return c, emax, it
        else:  # degenerate (should not happen): keep reference, report
            break
    return c, float(np.max(np.abs(fg - polyval(c, grid)))), max_iter
