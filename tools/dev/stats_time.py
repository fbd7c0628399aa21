"""Time vf_image_stats at the C4 slice (16 x 512x768) against the filter time."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_1009_0959_b200 as vfb
spec, w = bench.workload("C4")
x = torch.from_numpy(bench.make_input(spec, 0)).cuda()
a = vfb.vf_filter_batch(x, w, "angular", "exact")
b = vfb.vf_filter_batch(x, w, "exp", "minimax")
for name, (p, q) in {"ref_vs_other": (a, b), "ref_vs_self": (a, a), "input_vs_out": (x, a)}.items():
    for _ in range(3):
        vfb.vf_image_stats(p, q)
    ts = []
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); vfb.vf_image_stats(p, q); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(name, "%.1f us" % (1e3 * statistics.median(ts)), "px/s %.1f G" % (x.numel() / 3 / statistics.median(ts) / 1e6))
