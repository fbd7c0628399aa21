"""Small driver for compute-sanitizer: every kernel of libvf.so once on small
images (ragged sizes, both windows, batch, stripes, plans, stats)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402

combos = [("angular", "exact"), ("angular", "minimax"), ("exp", "exact"), ("exp", "minimax"), ("exp", "poly4"),
          ("log", "exact"), ("log", "minimax"), ("exp", "reach"), ("log", "reach"), ("amnfe", "minimax"), ("amnfg", "exact"), ("amnfe", "poly4"),
          ("evmf", "exact"), ("evmf", "minimax")]
for H, W in [(37, 45), (64, 64), (5, 70), (77, 144), (300, 96)]:   # 3W % 16 == 0: TMA path
    x = torch.from_numpy(vfsynth.random_image(1, H, W)).cuda()
    for w in (3, 5):
        if w > min(H, W):
            continue
        for c in combos:
            algos = (["stream", "window", "shared", "shared:1", "shared:2", "shared:3", "role", "role:1", "role:2",
                      "role:3"] if c[0] == "angular" else
                     ["auto:1", "auto:2", "auto:3", "auto:1+notma", "auto:2+notma", "auto:3+notma"])
            for a in algos:
                vfb.filter(x, w, *c, algo=a, want_index=True, want_agg=True)
        # stripes
        for lo, hi in [(0, H // 2), (H // 2, H)]:
            blo, bhi = max(0, lo - w // 2), min(H, hi + w // 2)
            for c in (("angular", "minimax"), ("exp", "minimax"), ("log", "exact")):
                vfb.vf_filter_rows(x[blo:bhi].contiguous(), blo, H, lo, hi - lo, w, *c)
xb = torch.from_numpy(vfsynth.make_batch(vfsynth.ImageSpec("t", 40, 56, 3, (3,), 4, False, "uncorrelated", 0.2))).cuda()
outs = [torch.empty_like(xb) for _ in combos]
plan = vfb.Plan(xb, outs, 3, combos)
plan.launch()
vfb.vf_image_stats(xb, outs[0])
# a fused plan (>= 2^21 pixels: the exp/log filters in one node), ragged width
xl = torch.from_numpy(vfsynth.make_batch(vfsynth.ImageSpec("t", 300, 1201, 6, (3,), 4, False, "uncorrelated", 0.2))).cuda()
louts = [torch.empty_like(xl) for _ in combos[:9]]
lplan = vfb.Plan(xl, louts, 3, combos[:9])
assert lplan.kernels() < 9
lplan.launch()
# the bench's 7-filter plan (pair-major exp/log node, fused angular node) with
# its statistics nodes, on noisy images and on a constant batch (flat windows:
# S1 = 0, z = u = 0 -- the edges of the ranges the libm calls are told,
# checked here by VF_ASSUME_RANGE -> VF_CHECK)
for xs in (xl, torch.full_like(xl, 77)):
    pouts = [torch.empty_like(xs) for _ in combos[:7]]
    st = torch.empty((4, xs.shape[0], 8), dtype=torch.float64, device="cuda")
    pplan = vfb.Plan(xs, pouts, 3, combos[:7], refs=[-1, 0, -1, 2, 2, -1, 5], stats=st)
    pplan.launch()
    for w in (3, 5):
        for c in (("exp", "exact"), ("log", "exact")):
            vfb.filter(xs[:1].contiguous(), w, *c)
# lone impulses in flat images: the windows holding one reach the largest
# arguments the criteria can take (z = z*_n: 0.716 / 0.742, u = 1 - 1/e; the
# bounds the libm calls are told), checked by VF_ASSUME_RANGE -> VF_CHECK
flat = torch.full((2, 96, 160, 3), 90, dtype=torch.uint8, device="cuda")
flat[0, 40, 70] = torch.tensor([255, 0, 0], dtype=torch.uint8)
flat[1, 0, 0] = torch.tensor([0, 255, 255], dtype=torch.uint8)
flat[1, 95, 159] = torch.tensor([255, 255, 255], dtype=torch.uint8)
for w in (3, 5):
    for c in (("exp", "exact"), ("log", "exact"), ("exp", "minimax"), ("log", "minimax")):
        vfb.filter(flat, w, *c, want_index=True, want_agg=True)
fouts = [torch.empty_like(flat) for _ in combos[:7]]
vfb.Plan(flat, fouts, 3, combos[:7]).launch()
torch.cuda.synchronize()
print("sanitize driver done")
