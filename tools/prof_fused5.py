"""One launch of the bench's exp/log plan node (pair-major fused kernel) on 64
C4 images, for an `ncu --set full -k regex:fused5` capture."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

x = torch.from_numpy(bench.gen_batch("C4", range(int(os.environ.get("PROF_IMAGES", "64"))))).cuda()
gcs = [c for c in bench.COMBOS if c[0] in ("exp", "log")]
outs = [torch.empty_like(x) for _ in gcs]
plan = vfb.Plan(x, outs, 3, gcs)
assert plan.kernels() == 1, plan.kernels()
plan.launch()
torch.cuda.synchronize()
print("fused5 done")
