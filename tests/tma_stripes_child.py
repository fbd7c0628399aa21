"""Child process of test_tma_path_borders_batches_stripes: with VF_FORCE_TMA=1
every exp/log launch with 16-byte aligned rows uses the TMA-staged kernel, so
row stripes (band-relative tensor map rows) run through it; their outputs
must be bit-identical to the full image on the plain-load kernel."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402

assert os.environ.get("VF_FORCE_TMA") == "1"
x = vfsynth.random_image(51, 77, 144)
H, W = x.shape[:2]
for crit, var in [("exp", "exact"), ("exp", "minimax"), ("exp", "poly4"), ("log", "exact"), ("log", "minimax"),
                  ("exp", "reach"), ("log", "reach")]:
    for w in (3, 5):
        xt = torch.from_numpy(x).cuda()
        full, fidx, fagg = vfb.filter(xt, w, crit, var, algo="auto+notma", want_index=True, want_agg=True)
        r = w // 2
        for k in (2, 3, 5):
            bounds = np.linspace(0, H, k + 1).astype(int)
            for a, b in zip(bounds[:-1], bounds[1:]):
                lo, hi = max(0, a - r), min(H, b + r)
                band = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
                idx = torch.empty((b - a, W), dtype=torch.uint8, device="cuda")
                agg = torch.empty((b - a, W, w * w), dtype=torch.float32, device="cuda")
                out = vfb.vf_filter_rows(band, lo, H, a, b - a, w, crit, var, index=idx, aggregates=agg)
                torch.cuda.synchronize()
                assert torch.equal(out, full[a:b]), (crit, var, w, k, a)
                assert torch.equal(idx, fidx[a:b]), (crit, var, w, k, a)
                assert torch.equal(agg, fagg[a:b]), (crit, var, w, k, a)
print("tma stripes ok")
