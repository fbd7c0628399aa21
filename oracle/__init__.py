"""CPU oracle for the minimax order-statistics vector filters (TEST INFRASTRUCTURE).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_1009_0959_b200``) never touches it.  It shares no code
with the CUDA path; see ``vf_oracle.c`` for the definitions and their
PAPER.md citations, and DESIGN.md section 4 for how each function is pinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "vf_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

ANGULAR, EXP, LOG = 0, 1, 2
EXACT, MINIMAX, MINIMAX_POLY4, MINIMAX_REACH = 0, 1, 2, 3
AMNFE, AMNFG, EVMF = 3, 4, 5
CRITERIA = {"angular": ANGULAR, "exp": EXP, "log": LOG}
FILTERS = {"amnfe": AMNFE, "amnfg": AMNFG, "evmf": EVMF}
VARIANTS = {"exact": EXACT, "minimax": MINIMAX, "poly4": MINIMAX_POLY4, "reach": MINIMAX_REACH}

FN = dict(arccos_exact=0, arccos_mm=1, p_arccos=2, p_arcsin=3, exp_exact=4,
          exp_rational=5, exp_poly2=6, exp_poly3=7, exp_poly4=8, ent_exact=9, ent_mm=10,
          exp_reach=11, log_reach=12)
TABLES = dict(arcsin=0, arccos=1, exp_p2=2, exp_p3=3, exp_p4=4, exp_num=5, exp_den=6,
              ent_num=7, ent_den=8, constants=9, exp_reach=10, log_reach=11)

_lib = None


def build(force: bool = False) -> str:
    """Compile vf_oracle.c with gcc (-O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + ".tmp%d" % os.getpid()
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
               "-fno-fast-math", "-Wall", "-Wextra", "-o", tmp, SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int
        L.oracle_filter.argtypes = [P, I, I, I, I, I, P, P, P, I]
        L.oracle_filter.restype = I
        L.oracle_filter_pixels.argtypes = [P, I, I, I, I, I, P, P, ctypes.c_int64, P, P, P, I]
        L.oracle_filter_pixels.restype = I
        L.oracle_window.argtypes = [P, I, I, I, P, P]
        L.oracle_window.restype = I
        L.oracle_gather_window.argtypes = [P, I, I, I, I, I, P]
        L.oracle_gather_window.restype = I
        L.oracle_pair_angular.argtypes = [P, P, I]
        L.oracle_pair_angular.restype = ctypes.c_double
        L.oracle_eval.argtypes = [I, P, ctypes.c_int64, P]
        L.oracle_eval.restype = I
        L.oracle_coeffs.argtypes = [I, P]
        L.oracle_coeffs.restype = I
        L.oracle_paper_window.argtypes = [P, I, I, I, P, P]
        L.oracle_paper_window.restype = I
        L.oracle_paper_filter.argtypes = [P, I, I, I, I, I, P, P, ctypes.c_int64, P, P, P, I]
        L.oracle_paper_filter.restype = I
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = I
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def _cv(c):
    return CRITERIA[c] if isinstance(c, str) else int(c)


def _vv(v):
    return VARIANTS[v] if isinstance(v, str) else int(v)


def filter_image(img: np.ndarray, window: int, criterion, variant, want_index=True,
                 want_agg=False, nthreads: int = 0):
    """Filter a uint8 [H, W, 3] image.  Returns (out, index|None, agg|None)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape[:2]
    n = window * window
    out = np.empty_like(img)
    idx = np.empty((H, W), np.uint8) if want_index else None
    agg = np.empty((H, W, n), np.float64) if want_agg else None
    rc = lib().oracle_filter(_ptr(img), H, W, window, _cv(criterion), _vv(variant),
                             _ptr(out), _ptr(idx), _ptr(agg), nthreads)
    if rc != 0:
        raise ValueError("oracle_filter: invalid arguments")
    return out, idx, agg


def filter_pixels(img: np.ndarray, window: int, criterion, variant, ys, xs,
                  want_agg=True, nthreads: int = 0):
    """Filter only the listed pixels.  Returns (out[npix,3], index[npix], agg[npix,n]|None)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape[:2]
    ys = np.ascontiguousarray(ys, dtype=np.int32)
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    npix = ys.shape[0]
    n = window * window
    out = np.zeros((npix, 3), np.uint8)
    idx = np.zeros((npix,), np.uint8)
    agg = np.zeros((npix, n), np.float64) if want_agg else None
    rc = lib().oracle_filter_pixels(_ptr(img), H, W, window, _cv(criterion), _vv(variant),
                                    _ptr(ys), _ptr(xs), npix, _ptr(out), _ptr(idx), _ptr(agg),
                                    nthreads)
    if rc != 0:
        raise ValueError("oracle_filter_pixels: invalid arguments")
    return out, idx, agg


def window(samples: np.ndarray, criterion, variant):
    """One window of n samples (uint8 [n, 3]).  Returns (k*, R[n], D[n, n])."""
    s = np.ascontiguousarray(samples, dtype=np.uint8).reshape(-1, 3)
    n = s.shape[0]
    R = np.empty(n, np.float64)
    Dm = np.empty((n, n), np.float64)
    k = lib().oracle_window(_ptr(s), n, _cv(criterion), _vv(variant), _ptr(R), _ptr(Dm))
    if k < 0:
        raise ValueError("oracle_window: invalid arguments")
    return k, R, Dm


def gather_window(img: np.ndarray, window_side: int, y: int, x: int) -> np.ndarray:
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape[:2]
    s = np.empty((window_side * window_side, 3), np.uint8)
    if lib().oracle_gather_window(_ptr(img), H, W, window_side, y, x, _ptr(s)) != 0:
        raise ValueError("bad window")
    return s


def pair_angular(a, b, variant) -> float:
    a = np.ascontiguousarray(a, dtype=np.uint8)
    b = np.ascontiguousarray(b, dtype=np.uint8)
    return float(lib().oracle_pair_angular(_ptr(a), _ptr(b), _vv(variant)))


def eval_fn(name: str, z) -> np.ndarray:
    z = np.ascontiguousarray(np.atleast_1d(np.asarray(z, dtype=np.float64)))
    out = np.empty_like(z)
    if lib().oracle_eval(FN[name], _ptr(z), z.shape[0], _ptr(out)) != 0:
        raise ValueError(name)
    return out


def coeffs(table: str) -> np.ndarray:
    out = np.zeros(8, np.float64)
    m = lib().oracle_coeffs(TABLES[table], _ptr(out))
    return out[:m].copy()


def _fv(f):
    return FILTERS[f] if isinstance(f, str) else int(f)


def paper_window(samples, filt, variant):
    """AMNF (Eq. 8) / EVMF (Eq. 9) on one window of n samples (uint8 [n, 3]).
    Returns (selected index, out[3], aux[n + 3]) -- see vf_oracle.c."""
    s = np.ascontiguousarray(samples, dtype=np.uint8).reshape(-1, 3)
    n = s.shape[0]
    out = np.zeros(3, np.uint8)
    aux = np.zeros(n + 3, np.float64)
    k = lib().oracle_paper_window(_ptr(s), n, _fv(filt), _vv(variant), _ptr(out), _ptr(aux))
    if k < 0:
        raise ValueError("oracle_paper_window: invalid arguments")
    return k, out, aux


def paper_filter(img, window: int, filt, variant, ys=None, xs=None, want_aux=True, nthreads: int = 0):
    """AMNF / EVMF over a full image (ys = xs = None: outputs [H, W, ...]) or at
    sampled pixels ([npix, ...]).  Returns (out, index, aux | None)."""
    img = np.ascontiguousarray(img, dtype=np.uint8)
    H, W = img.shape[:2]
    n = window * window
    if ys is None:
        npix = H * W
        yp = xp = None
    else:
        yp = np.ascontiguousarray(ys, dtype=np.int32)
        xp = np.ascontiguousarray(xs, dtype=np.int32)
        npix = yp.shape[0]
    out = np.zeros((npix, 3), np.uint8)
    idx = np.zeros((npix,), np.uint8)
    aux = np.zeros((npix, n + 3), np.float64) if want_aux else None
    rc = lib().oracle_paper_filter(_ptr(img), H, W, window, _fv(filt), _vv(variant), _ptr(yp), _ptr(xp), npix,
                                   _ptr(out), _ptr(idx), _ptr(aux), nthreads)
    if rc != 0:
        raise ValueError("oracle_paper_filter: invalid arguments")
    if ys is None:
        out = out.reshape(H, W, 3)
        idx = idx.reshape(H, W)
        aux = None if aux is None else aux.reshape(H, W, n + 3)
    return out, idx, aux


def max_threads() -> int:
    return int(lib().oracle_max_threads())
