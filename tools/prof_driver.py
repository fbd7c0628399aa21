"""Small driver for ncu captures: runs every criterion x variant filter of a
config twice (the first round warms up; profile the second with
`ncu -k regex:vf_ -s 7 -c 7 ...`)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--algo", default="auto")
a = ap.parse_args()
spec, w = bench.workload(a.config)
x = torch.from_numpy(bench.make_input(spec, 0)).cuda()
out = torch.empty_like(x)
for _ in range(a.rounds):
    for crit, var in bench.COMBOS:
        vfb.vf_filter_batch_algo(x, w, crit, var, a.algo, out=out)
torch.cuda.synchronize()
print("done", a.config, tuple(x.shape))
