"""Image quality criteria of PAPER.md section 4, numpy float64
(TEST INFRASTRUCTURE: the oracle for the GPU stats kernel).

MAE(X, Y) = 1/(3MN) sum ||x - y||_1
MSE(X, Y) = 1/(3MN) sum ||x - y||_2^2
NCD(X, Y) = sum ||x_Lab - y_Lab||_2 / sum ||x_Lab||_2
CIELAB via sRGB (IEC 61966-2-1 transfer), BT.709 primaries, D65 white.
"""
import numpy as np

_M = np.array([[0.4124564, 0.3575761, 0.1804375],
               [0.2126729, 0.7151522, 0.0721750],
               [0.0193339, 0.1191920, 0.9503041]])
_WHITE = np.array([0.95047, 1.0, 1.08883])


def mae(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).sum() / a.size)


def mse(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(((a - b) ** 2).sum() / a.size)


def rgb_to_lab(rgb):
    c = np.asarray(rgb, np.float64) / 255.0
    lin = np.where(c <= 0.04045, c / 12.92, ((c + 0.055) / 1.055) ** 2.4)
    xyz = lin @ _M.T / _WHITE
    d = 6.0 / 29.0
    f = np.where(xyz > d ** 3, np.cbrt(xyz), xyz / (3 * d * d) + 4.0 / 29.0)
    L = 116.0 * f[..., 1] - 16.0
    A = 500.0 * (f[..., 0] - f[..., 1])
    B = 200.0 * (f[..., 1] - f[..., 2])
    return np.stack([L, A, B], -1)


def ncd(a, b):
    la, lb = rgb_to_lab(a), rgb_to_lab(b)
    den = np.linalg.norm(la, axis=-1).sum()
    if den == 0:
        raise ValueError("NCD undefined for an all-black reference")
    return float(np.linalg.norm(la - lb, axis=-1).sum() / den)


def psnr(a, b):
    m = mse(a, b)
    return float("inf") if m == 0 else 10.0 * np.log10(255.0 ** 2 / m)
