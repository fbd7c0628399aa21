"""Largest aggregate error (relative to the float64 oracle) of the exact
exp / log variants on full images: C2 (3x3, 5x5) and a C3-like 512^2 crop
with 20% uncorrelated impulses (5x5).  VF_LIB selects the library build."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402
from tests.parity import check_parity  # noqa: E402

imgs = [("C2", vfsynth.make_image(vfsynth.config("C2"), 0)[1]),
        ("C3crop", vfsynth.make_image(dataclasses.replace(vfsynth.config("C3"), H=512, W=512), 0)[1])]
tag = os.path.basename(os.environ.get("VF_LIB", "libvf.so"))
for name, img in imgs:
    x = torch.from_numpy(np.ascontiguousarray(img)).cuda()
    for w in (3, 5):
        for crit in ("exp", "log"):
            out, idx, agg = vfb.filter(x, w, crit, "exact", want_index=True, want_agg=True)
            torch.cuda.synchronize()
            _, o_idx, o_agg = oracle.filter_image(img, w, crit, "exact", want_agg=True)
            rep = check_parity(img, w, out.cpu().numpy(), idx.cpu().numpy(), agg.cpu().numpy(), o_idx, o_agg)
            print(f"{tag} {name} {w}x{w} {crit}/exact agg_max_rel {rep['agg_max_rel']:.3e} ok {rep['ok']} "
                  f"idx_differs_accepted {rep['idx_differs_accepted']}", flush=True)
