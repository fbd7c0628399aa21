"""Run every kernel variant on small ragged inputs with the debug build
(libvf_debug.so: device-side VF_CHECK bounds checks on every staged global
read, shared-memory pair-map index and output store).  A violated check traps
the kernel and the driver process fails.  (compute-sanitizer is closed on the
GPU pool; this is the substitute.)"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEBUG_LIB = os.path.join(ROOT, "paper_1009_0959_b200", "libvf_debug.so")


def test_all_kernels_under_bounds_checks():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(DEBUG_LIB):
        from paper_1009_0959_b200 import build
        build.build(debug=True)
    env = dict(os.environ, VF_LIB=DEBUG_LIB, VF_FORCE_TMA="1")   # stripes and "auto" through the TMA kernel too
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_driver.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "sanitize driver done" in r.stdout
    assert "VF_CHECK failed" not in r.stdout + r.stderr
