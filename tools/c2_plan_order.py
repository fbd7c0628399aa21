"""C2 (one 512x512 image, 7 filters) step time for different plan node orders
and shapes -- the bench's C2 step (L2 flushed outside the events, one graph
launch between CUDA events), averaged over --steps:

    python tools/c2_plan_order.py [--steps 200]

VF_LIB / VF_* environment knobs apply as usual (read once per process)."""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=200)
a = ap.parse_args()
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
x = torch.from_numpy(bench.gen_batch("C2", [0])).to(dev)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)


def step_us(combos):
    outs = [torch.empty_like(x) for _ in combos]
    plan = vfb.Plan(x, outs, 3, combos)
    for _ in range(10):
        plan.launch(stream)
    evs = [bench.ev_pair(torch) for _ in range(a.steps)]
    torch.cuda.synchronize()
    for k in range(a.steps):
        flush.fill_(k & 0xFF)
        evs[k][0].record(stream)
        plan.launch(stream)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    t = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
    plan.close()
    return sum(t) / len(t), t[len(t) // 2], plan_kernels(combos)


def plan_kernels(combos):
    outs = [torch.empty_like(x) for _ in combos]
    p = vfb.Plan(x, outs, 3, combos)
    n = p.kernels()
    p.close()
    return n


work = {c: 0.0 for c in bench.COMBOS}     # single-kernel C2 times (isolated, L2 warm) as the work estimate
for c in bench.COMBOS:
    out = torch.empty_like(x)
    work[c] = bench.kernel_avg_ms(torch, dev, stream, lambda c=c: vfb.vf_filter_batch(x, 3, *c, out=out, stream=stream),
                                  50) * 1e3
print("single kernels (us):", {f"{c[0]}/{c[1]}": round(v, 1) for c, v in work.items()}, flush=True)
orders = {"bench": bench.COMBOS,
          "longest first": sorted(bench.COMBOS, key=lambda c: -work[c]),
          "shortest first": sorted(bench.COMBOS, key=lambda c: work[c])}
for name, combos in orders.items():
    mean, med, nk = step_us(combos)
    print(f"{name:16s} nodes {nk}  mean {mean:6.1f} us  median {med:6.1f} us", flush=True)
# a few random permutations
for i, perm in enumerate(itertools.islice(itertools.permutations(bench.COMBOS), 0, 5040, 997)):
    mean, med, nk = step_us(list(perm))
    print(f"perm {i:2d}          nodes {nk}  mean {mean:6.1f} us  median {med:6.1f} us", flush=True)
