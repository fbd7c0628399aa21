"""Child process of test_el_block_shapes_bit_identical: with the exp/log 3x3
block shape forced by VF_EL_TY / VF_EL_OPT (read once per process), print a
digest of the outputs, indices and aggregates of every non-libm variant on a
ragged 2-image batch above the large-launch threshold.  The parent compares
the digests with the default configuration's: every tile shape must give
bit-identical results (deterministic accumulation)."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402

COMBOS = [("exp", "minimax"), ("exp", "poly4"), ("exp", "reach"), ("log", "minimax"), ("log", "reach")]


def digests():
    x = np.stack([vfsynth.random_image(70 + b, 1031, 1029) for b in range(2)])   # 2.1 M px, ragged tiles
    xt = torch.from_numpy(x).cuda()
    res = {}
    for c in COMBOS:
        out, idx, agg = vfb.filter(xt, 3, *c, want_index=True, want_agg=True)
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for t in (out, idx, agg):
            h.update(t.cpu().numpy().tobytes())
        res[f"{c[0]}/{c[1]}"] = h.hexdigest()
    return res


if __name__ == "__main__":
    for k, v in digests().items():
        print(k, v)
