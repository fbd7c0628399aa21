"""Re-derive minimax polynomials on the arguments the criteria can actually
reach with the oracle's Remez exchange (oracle/minimax.py,
the algorithm of), and write tests/golden/remez_reach.txt.

Reachable intervals (proved in DESIGN.md section 2, tested on the oracle):
  exp criterion  D_E = 1 - exp(-z),          z in [0, z*_25],  z*_n = n^(1+kappa/3) / (2(n-1))
  log criterion  D_L = -(1 - u) ln(1 - u),   u in [0, 1 - 1/e] (u = 1 - s, s the ENT argument)
Both are fitted directly as the criterion value (minimax in the absolute
error of Eq. 1 is invariant under D = 1 - E and under the affine change
s = 1 - u), so a kernel evaluates one Horner polynomial and no division.

Usage: python tools/remez_reach.py [--write]
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import minimax  # noqa: E402

KAPPA = 0.33
Z_MAX = 25 ** (1 + KAPPA / 3) / (2 * 24)          # z*_25 = 0.7421166...
U_MAX = 1 - math.exp(-1.0)
DEG_EXP, DEG_LOG = 5, 7
OUT = os.path.join(ROOT, "tests", "golden", "remez_reach.txt")


def g_exp(z):
    return -np.expm1(-np.asarray(z, dtype=np.float64))


def g_log(u):
    u = np.asarray(u, dtype=np.float64)
    return -(1.0 - u) * np.log1p(-u)


def fits():
    ce, ee, ie = minimax.remez(g_exp, DEG_EXP, 0.0, Z_MAX, tol=1e-7, npts=800_001)
    cl, el, il = minimax.remez(g_log, DEG_LOG, 0.0, U_MAX, tol=1e-7, npts=800_001)
    return (ce, ee, ie), (cl, el, il)


def main():
    (ce, ee, ie), (cl, el, il) = fits()
    lines = [
        "# Minimax polynomials on the reachable arguments (SURVEY.md 8(f4)), written by",
        "# tools/remez_reach.py with oracle/minimax.remez (Remez exchange, P:70).  17 significant digits.",
        f"# exp: D_E(z) = 1 - exp(-z) on [0, {Z_MAX!r}] (z*_25), degree {DEG_EXP}, eps {ee:.6e} ({ie} iterations)",
        "exp_reach " + " ".join(f"{c:.17g}" for c in ce),
        f"exp_reach_eps {ee:.17g}",
        f"exp_reach_interval 0 {Z_MAX!r}",
        f"# log: D_L(u) = -(1 - u) ln(1 - u) on [0, 1 - 1/e], degree {DEG_LOG}, eps {el:.6e} ({il} iterations)",
        "log_reach " + " ".join(f"{c:.17g}" for c in cl),
        f"log_reach_eps {el:.17g}",
        f"log_reach_interval 0 {U_MAX!r}",
    ]
    text = "\n".join(lines) + "\n"
    print(text)
    if "--write" in sys.argv:
        with open(OUT, "w") as fh:
            fh.write(text)
        print("wrote", OUT)


if __name__ == "__main__":
    main()
