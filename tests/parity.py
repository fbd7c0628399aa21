"""Parity acceptance rule, GPU vs oracle (BASELINE.json
north_star):

* aggregates: |R_gpu - R_oracle| <= 1e-5 |R_oracle| + 1e-12 for every sample;
* selected index g: accepted iff x_g equals the oracle's output vector x_k*,
  or R^o_g - R^o_k* <= 1e-5 max(|R^o_g|, |R^o_k*|) + 1e-12 (the oracle's top
  candidates are within 1e-5 relative, so either is correct);
* the output pixel must be the window sample at g (bit-exact).
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-5
ATOL = 1e-12


def windows_at(img: np.ndarray, w: int, ys: np.ndarray, xs: np.ndarray) -> np.ndarray:
    """Window samples [npix, n, 3] at the given pixels (replicate padding)."""
    H, W = img.shape[:2]
    r = w // 2
    dy, dx = np.meshgrid(np.arange(w) - r, np.arange(w) - r, indexing="ij")
    yy = np.clip(ys[:, None] + dy.ravel()[None, :], 0, H - 1)
    xx = np.clip(xs[:, None] + dx.ravel()[None, :], 0, W - 1)
    return img[yy, xx]


def check_parity(img, w, g_out, g_idx, g_agg, o_idx, o_agg, ys=None, xs=None,
                 rtol: float = RTOL, atol: float = ATOL) -> dict:
    """img: uint8 [H, W, 3].  Full-image arrays ([H, W, ...]) when ys/xs are
    None, else per-sample arrays ([npix, ...]) for pixels (ys, xs)."""
    H, W = img.shape[:2]
    if ys is None:
        yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        ys, xs = yy.ravel(), xx.ravel()
        g_out = g_out.reshape(-1, 3)
        g_idx = g_idx.reshape(-1)
        o_idx = o_idx.reshape(-1)
        if g_agg is not None:
            g_agg = g_agg.reshape(ys.shape[0], -1)
        o_agg = o_agg.reshape(ys.shape[0], -1)
    ys = np.asarray(ys)
    xs = np.asarray(xs)
    S = windows_at(img, w, ys, xs)
    ar = np.arange(ys.shape[0])
    g_idx = g_idx.astype(np.int64)
    o_idx = o_idx.astype(np.int64)
    rep = dict(npix=int(ys.shape[0]))
    if g_agg is not None:
        err = np.abs(g_agg.astype(np.float64) - o_agg)
        lim = rtol * np.abs(o_agg) + atol
        bad = err > lim
        rep["agg_bad"] = int(bad.sum())
        with np.errstate(divide="ignore", invalid="ignore"):
            rel = np.where(o_agg != 0, err / np.abs(o_agg), np.where(err > 0, np.inf, 0.0))
        rep["agg_max_rel"] = float(rel.max()) if rel.size else 0.0
        rep["agg_exact_zero_violations"] = int(((o_agg == 0) & (g_agg != 0)).sum())
    else:
        rep["agg_bad"] = 0
    Rg = o_agg[ar, g_idx]
    Rk = o_agg[ar, o_idx]
    same_vec = np.all(S[ar, g_idx] == S[ar, o_idx], axis=-1)
    near = (Rg - Rk) <= rtol * np.maximum(np.abs(Rg), np.abs(Rk)) + atol
    idx_ok = same_vec | near
    rep["idx_bad"] = int((~idx_ok).sum())
    rep["idx_differs_accepted"] = int(((g_idx != o_idx) & idx_ok).sum())
    rep["vec_differs_accepted"] = int((~same_vec & idx_ok).sum())
    out_ok = np.all(g_out.reshape(-1, 3) == S[ar, g_idx], axis=-1)
    rep["out_bad"] = int((~out_ok).sum())
    rep["ok"] = rep["agg_bad"] == 0 and rep["idx_bad"] == 0 and rep["out_bad"] == 0 \
        and rep.get("agg_exact_zero_violations", 0) == 0
    return rep
