"""Run one filter (config, criterion, variant) twice for a targeted ncu capture."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1009_0959_b200 as vfb
import bench
cfg, crit, var = sys.argv[1], sys.argv[2], sys.argv[3]
algo = sys.argv[4] if len(sys.argv) > 4 else "auto"
spec, w = bench.workload(cfg)
x = torch.from_numpy(bench.make_input(spec, 0)).cuda()
out = torch.empty_like(x)
for _ in range(2):
    vfb.vf_filter_batch_algo(x, w, crit, var, algo, out=out)
torch.cuda.synchronize()
print("done")
