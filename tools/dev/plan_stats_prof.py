"""One launch each of the exp/log fused node without and with epilogue
statistics (C4, 64 images), for an ncu capture (tools/dev)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

n = int(os.environ.get("AB_IMAGES", "64"))
x = torch.from_numpy(bench.gen_batch("C4", range(n))).cuda()
EL = [("exp", "exact"), ("exp", "minimax"), ("exp", "poly4"), ("log", "exact"), ("log", "minimax")]
for refs in (None, [-1, 0, 0, -1, 3]):
    outs = [torch.empty_like(x) for _ in EL]
    st = None if refs is None else torch.empty((3, n, 8), dtype=torch.float64, device="cuda")
    p = vfb.Plan(x, outs, 3, EL, refs=refs, stats=st)
    p.launch()
    torch.cuda.synchronize()
    p.close()
print("done")
