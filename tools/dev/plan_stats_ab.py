"""A/B: plans with and without fidelity statistics nodes (C4, 256 images)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402

n = int(os.environ.get("AB_IMAGES", "256"))
x = torch.from_numpy(bench.gen_batch("C4", range(n))).cuda()
stream = torch.cuda.current_stream()
EL = [("exp", "exact"), ("exp", "minimax"), ("exp", "poly4"), ("log", "exact"), ("log", "minimax")]
ANG = [("angular", "exact"), ("angular", "minimax")]
cases = [("el plain", EL, None), ("el stats", EL, [-1, 0, 0, -1, 3]), ("el stats exp-only", EL, [-1, 0, -1, -1, -1]),
         ("ang plain", ANG, None), ("ang stats", ANG, [-1, 0]),
         ("all plain", bench.COMBOS, None), ("all stats", bench.COMBOS, bench.FIDELITY_REFS)]
for name, combos, refs in cases:
    outs = [torch.empty_like(x) for _ in combos]
    st = None
    if refs is not None:
        st = torch.empty((sum(r >= 0 for r in refs), n, 8), dtype=torch.float64, device="cuda")
    p = vfb.Plan(x, outs, 3, combos, refs=refs, stats=st)
    ms = bench.kernel_avg_ms(torch, x.device, stream, lambda: p.launch(stream), 5)
    print(f"{name:20s} {ms:8.3f} ms  kernels {p.kernels()}", flush=True)
    p.close()
