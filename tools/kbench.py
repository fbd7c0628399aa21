"""Quick per-kernel timing for tuning iterations (CUDA events over back-to-back
launches on inputs larger than L2):

    python tools/kbench.py [--images 128] [--only angular/minimax] [--algo auto] [--c3] [--reps 5]

VF_LIB=path/to/libvf_variant.so selects a library build (A/B comparisons)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--images", type=int, default=128)
ap.add_argument("--only", default=None)
ap.add_argument("--algo", default="auto")
ap.add_argument("--c3", action="store_true")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda")
stream = torch.cuda.current_stream()
peak = 2 * 128 * 148 * 1.965e9 / 1e12
tag = os.path.basename(os.environ.get("VF_LIB", "libvf.so"))
for cfg, w, ids in (("C4", 3, range(a.images)),) + ((("C3", 5, range(8)),) if a.c3 else ()):
    x = torch.from_numpy(bench.gen_batch(cfg, ids)).to(dev)
    npix = x.numel() // 3
    out = torch.empty_like(x)
    n = w * w
    pairs = n * (n - 1) // 2
    line = [f"{tag} {cfg}({w}x{w},{npix / 1e6:.0f}Mpx)"]
    for c in bench.COMBOS + bench.REACH_COMBOS:
        if a.only and a.only not in f"{c[0]}/{c[1]}":
            continue
        ms = bench.kernel_avg_ms(torch, dev, stream,
                                 lambda c=c: vfb.vf_filter_batch_algo(x, w, *c, a.algo, out=out, stream=stream), a.reps)
        frac = bench.FLOPS_PER_PAIR[c] * pairs * npix / (ms / 1e3) / 1e12 / peak
        line.append(f"{c[0][:3]}/{c[1][:3]} {ms * 1e3:8.1f}us {frac * 100:4.1f}%")
    print(" | ".join(line), flush=True)
