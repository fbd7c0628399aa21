"""CPU-only checks: the metric oracle against SPEC examples, and
the C-ABI library: it loads without a GPU, exports every symbol include/vf.h
declares, and rejects invalid arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import metrics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_mae_mse_spec_examples():
    a = np.array([[[0, 0, 0]]], np.uint8)
    assert metrics.mae(a, np.array([[[3, 6, 0]]], np.uint8)) == 3.0
    assert metrics.mse(a, np.array([[[3, 4, 0]]], np.uint8)) == pytest.approx(25 / 3)
    rng = np.random.default_rng(0)
    x = rng.integers(0, 256, (8, 8, 3))
    y = rng.integers(0, 256, (8, 8, 3))
    s = 0.0
    for i in range(8):
        for j in range(8):
            for k in range(3):
                s += abs(int(x[i, j, k]) - int(y[i, j, k]))
    assert metrics.mae(x, y) == pytest.approx(s / 192, rel=1e-12)


def test_lab_spec_examples():
    L, A, B = metrics.rgb_to_lab(np.array([255, 255, 255]))
    assert L == pytest.approx(100, abs=1e-3) and abs(A) <= 0.01 and abs(B) <= 0.01
    assert np.allclose(metrics.rgb_to_lab(np.array([0, 0, 0])), 0)
    L, A, B = metrics.rgb_to_lab(np.array([255, 0, 0]))
    assert (L, A, B) == (pytest.approx(53.24, abs=0.1), pytest.approx(80.09, abs=0.1),
                         pytest.approx(67.20, abs=0.1))


def test_ncd_properties():
    rng = np.random.default_rng(1)
    x = rng.integers(0, 256, (8, 8, 3))
    assert metrics.ncd(x, x) == 0.0
    with pytest.raises(ValueError):
        metrics.ncd(np.zeros((2, 2, 3)), x[:2, :2])


# ------------------------------------------------------------------ the C ABI
def _header_symbols():
    src = open(os.path.join(ROOT, "include", "vf.h")).read()
    return sorted(set(re.findall(r"VF_API\s+[\w\s\*]*?\b(vf_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_1009_0959_b200 import build, vf
    build.build()
    return vf.load_library()


def test_library_exports_every_declared_symbol(lib):
    syms = _header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    from paper_1009_0959_b200 import vf
    assert sorted(vf.EXPORTS) == syms


def test_status_strings_and_version(lib):
    from paper_1009_0959_b200 import vf
    assert vf.vf_version() == 105
    assert vf.vf_status_string(0) == "VF_OK"
    assert "invalid" in vf.vf_status_string(-1)
    assert "compiled" in vf.vf_status_string(-2)
    assert "CUDA" in vf.vf_status_string(-3)


def test_invalid_arguments_rejected_before_any_device_work(lib):
    """Validation happens on the host before any CUDA call (NULL pointers are
    never dereferenced), so these run without a GPU."""
    f = lib.vf_filter
    p = ctypes.c_void_p(16)      # never dereferenced
    q = ctypes.c_void_p(1 << 40)
    assert f(p, 16, 16, 4, 0, 0, q, None, None, None) == -1          # even window
    assert f(p, 16, 16, 1, 0, 0, q, None, None, None) == -1          # window < 3
    assert f(p, 16, 16, 7, 0, 0, q, None, None, None) == -2          # valid, not compiled
    assert f(p, 2, 16, 3, 0, 0, q, None, None, None) == -1           # window > H
    assert f(p, 16, 16, 3, 6, 0, q, None, None, None) == -1          # criterion
    assert f(p, 16, 16, 3, 1, 4, q, None, None, None) == -1          # variant
    assert f(p, 16, 16, 3, 0, 3, q, None, None, None) == -1          # REACH only for exp / log
    assert f(p, 16, 16, 3, 0, 2, q, None, None, None) == -1          # POLY4 only for the EXP filters
    assert f(p, 16, 16, 3, 5, 2, q, None, None, None) == -1          # (EVMF uses ENT, not EXP)
    assert f(None, 16, 16, 3, 0, 0, q, None, None, None) == -1       # NULL input
    assert f(p, 16, 16, 3, 0, 0, p, None, None, None) == -1          # aliasing
    assert b"overlap" in lib.vf_last_error()
    assert lib.vf_filter_batch(p, 0, 16, 16, 3, 0, 0, q, None, None, None) == -1   # B < 1
    # stripe band that misses a halo row
    assert lib.vf_filter_rows(p, 5, 8, 40, 16, 5, 5, 3, 0, 1, q, None, None, None) == -1
    assert lib.vf_host_workspace_bytes(1, 10, 10) >= 600
    # plans validate every filter before creating anything
    h = ctypes.c_void_p()
    crit = (ctypes.c_int * 2)(0, 1)
    var = (ctypes.c_int * 2)(1, 2)
    outs = (ctypes.c_void_p * 2)(1 << 40, 1 << 41)
    assert lib.vf_plan_create(ctypes.byref(h), 1, 16, 16, 3, 2, crit, (ctypes.c_int * 2)(1, 4), p, outs, None,
                              None) == -1
    assert lib.vf_plan_create(ctypes.byref(h), 1, 16, 16, 3, 0, crit, var, p, outs, None, None) == -1
    assert lib.vf_plan_create(ctypes.byref(h), 1, 16, 16, 4, 2, crit, var, p, outs, None, None) == -1
    assert h.value is None
    assert lib.vf_plan_launch(None, None) == -1
    assert lib.vf_plan_destroy(None) == 0
