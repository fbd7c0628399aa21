"""GPU: the VF_EXACT_LIBM=1 build (libvf_paperlibm.so: the exact exp / log
variants as the paper's expf / logf instead of the survey's expm1f / log1pf,
DESIGN.md reading R26) meets the same parity rule against the float64
oracle: full C1 / C2 images, 3x3 and 5x5, and a fused 7-filter plan.  Run in
a child process (VF_LIB selects the library once per process)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1009_0959_b200", "libvf_paperlibm.so")

CHILD = r'''
import dataclasses, numpy as np, torch, oracle, vfsynth, paper_1009_0959_b200 as vfb
from tests.parity import check_parity
assert vfb.vf.LIB_PATH.endswith("libvf_paperlibm.so")
worst = 0.0
for cfg in ("C1", "C2"):
    _, img = vfsynth.make_image(vfsynth.config(cfg), 0)
    x = torch.from_numpy(img).cuda()
    for w in (3, 5):
        for crit in ("exp", "log"):
            out, idx, agg = vfb.filter(x, w, crit, "exact", want_index=True, want_agg=True)
            torch.cuda.synchronize()
            _, o_idx, o_agg = oracle.filter_image(img, w, crit, "exact", want_agg=True)
            rep = check_parity(img, w, out.cpu().numpy(), idx.cpu().numpy(), agg.cpu().numpy(), o_idx, o_agg)
            assert rep["ok"], (cfg, w, crit, rep)
            worst = max(worst, rep["agg_max_rel"])
# the fused plan (pair-major exp/log node) against the single-filter kernels of the same build
spec = dataclasses.replace(vfsynth.config("C4"), batch=8)
xb = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
combos = [("angular", "exact"), ("angular", "minimax"), ("exp", "exact"), ("exp", "minimax"),
          ("exp", "poly4"), ("log", "exact"), ("log", "minimax")]
outs = [torch.empty_like(xb) for _ in combos]
vfb.Plan(xb, outs, 3, combos).launch()
torch.cuda.synchronize()
for c, o in zip(combos, outs):
    assert torch.equal(o, vfb.filter(xb, 3, *c)[0]), c
print("paperlibm ok worst %.3e" % worst)
'''


def test_paper_libm_build_parity():
    if not os.path.exists(LIB):
        from paper_1009_0959_b200 import build
        build.build(True, False, False, *build.PAPER_LIBM)
    r = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, env=dict(os.environ, VF_LIB=LIB),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "paperlibm ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    worst = float(r.stdout.split("worst")[-1])
    assert worst < 1e-5
