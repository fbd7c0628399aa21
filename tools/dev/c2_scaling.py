"""Per-kernel time vs batch size at the C2 image size (fixed launch/ramp cost
vs throughput): python tools/dev/c2_scaling.py [--noflush]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
spec, w = bench.workload("C2")
x1 = torch.from_numpy(bench.make_input(spec, 0)).cuda()
noflush = "--noflush" in sys.argv
spin = "--spin" in sys.argv   # no flush; a 100 us sleep kernel hides the CPU launch latency
scratch = torch.zeros(1, device="cuda")
ts = []
for _ in range(15):
    if spin:
        torch.cuda._sleep(200000)
    elif not noflush:
        flush.fill_(1)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    scratch.add_(1)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"empty kernel {statistics.median(ts)*1e3:.1f} us", flush=True)
for B in (1, 2, 4, 8, 16):
    x = x1.expand(B, *x1.shape[-3:]).contiguous() if x1.dim() == 4 else x1.unsqueeze(0).expand(B, *x1.shape).contiguous()
    out = torch.empty_like(x)
    line = [f"B={B:2d}"]
    for c in bench.COMBOS:
        for _ in range(3):
            vfb.vf_filter_batch_algo(x, w, *c, "auto", out=out)
        ts = []
        for _ in range(15):
            if spin:
                torch.cuda._sleep(200000)
            elif not noflush:
                flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            vfb.vf_filter_batch_algo(x, w, *c, "auto", out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        line.append(f"{c[0][:3]}/{c[1][:3]} {statistics.median(ts)*1e3:7.1f}")
    print(" | ".join(line), flush=True)
