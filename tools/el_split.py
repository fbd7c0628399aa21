"""exp/log node variants on C4 images (CUDA events, back-to-back launches):
the pair-major 5-filter node vs splits of the five filters into smaller plans.

    python tools/el_split.py [--images 256]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--images", type=int, default=256)
a = ap.parse_args()
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
x = torch.from_numpy(bench.gen_batch("C4", range(a.images))).to(dev)
EL = [c for c in bench.COMBOS if c[0] in ("exp", "log")]
outs = {c: torch.empty_like(x) for c in EL}


def plan_ms(cs):
    p = vfb.Plan(x, [outs[c] for c in cs], 3, cs)
    ms = bench.kernel_avg_ms(torch, dev, stream, lambda: p.launch(stream), 5)
    n = p.kernels()
    p.close()
    return ms, n


tag = os.path.basename(os.environ.get("VF_LIB", "libvf.so"))
for name, groups in (("all5", [EL]),
                     ("exact|minimax", [[c for c in EL if c[1] == "exact"], [c for c in EL if c[1] != "exact"]]),
                     ("exp|log", [[c for c in EL if c[0] == "exp"], [c for c in EL if c[0] == "log"]]),
                     ("singles", [[c] for c in EL])):
    r = [plan_ms(g) for g in groups]
    print(f"{tag} {name:14s} " + " + ".join(f"{ms:.3f}({n})" for ms, n in r) + f" = {sum(ms for ms, _ in r):.3f} ms",
          flush=True)
