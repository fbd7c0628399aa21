"""Child process for tests/test_gpu_parity.py::test_stream_kernel_paths (run
with VF_ANG3_STREAM=1: the streamed 3x3 angular kernels at every size): row
stripes, batches and misaligned bases through the streamed kernels must equal
the whole-image streamed result bit for bit, and the whole image must pass the
oracle parity check."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_1009_0959_b200 as vfb  # noqa: E402
import vfsynth  # noqa: E402
from tests.parity import check_parity  # noqa: E402

assert os.environ.get("VF_ANG3_STREAM") == "1"
for var in ("minimax", "exact"):
    x = vfsynth.random_image(77, 53, 131)                     # 3W = 393: odd row stride
    H, W = x.shape[:2]
    xt = torch.from_numpy(x).cuda()
    info = vfb.vf_kernel_info(1, H, W, 3, "angular", var)
    assert "stream" in info["name"], info
    full, fidx, fagg = vfb.filter(xt, 3, "angular", var, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    _, o_idx, o_agg = oracle.filter_image(x, 3, "angular", var, want_agg=True)
    rep = check_parity(x, 3, full.cpu().numpy(), fidx.cpu().numpy(), fagg.cpu().numpy(), o_idx, o_agg)
    assert rep["ok"], (var, rep)
    for k in (2, 3, 5):
        bounds = np.linspace(0, H, k + 1).astype(int)
        for a, b in zip(bounds[:-1], bounds[1:]):
            lo, hi = max(0, a - 1), min(H, b + 1)
            band = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
            idx = torch.empty((b - a, W), dtype=torch.uint8, device="cuda")
            agg = torch.empty((b - a, W, 9), dtype=torch.float32, device="cuda")
            out = vfb.vf_filter_rows(band, lo, H, a, b - a, 3, "angular", var, index=idx, aggregates=agg)
            torch.cuda.synchronize()
            assert torch.equal(out, full[a:b]) and torch.equal(idx, fidx[a:b]) and torch.equal(agg, fagg[a:b]), (var, k, a)
    xb = np.stack([vfsynth.random_image(90 + i, 41, 101) for i in range(3)])      # odd image stride
    ob, ib, ab = vfb.filter(torch.from_numpy(xb).cuda(), 3, "angular", var, want_index=True, want_agg=True)
    buf = torch.zeros(xb.size + 1, dtype=torch.uint8, device="cuda")             # base at byte 1
    xv = buf[1:].view(xb.shape)
    xv.copy_(torch.from_numpy(xb))
    ob2 = vfb.filter(xv, 3, "angular", var)[0]
    torch.cuda.synchronize()
    assert torch.equal(ob, ob2), var
    for i in range(3):
        e_out, e_idx, e_agg = vfb.filter(torch.from_numpy(xb[i]).cuda(), 3, "angular", var, want_index=True,
                                         want_agg=True)
        torch.cuda.synchronize()
        assert torch.equal(ob[i], e_out) and torch.equal(ib[i], e_idx) and torch.equal(ab[i], e_agg), (var, i)
    # half-warp remainder strips (batches with W - 62 (S - 1) <= 30): the last
    # strip of images 2z, 2z + 1 on the two halves of one warp, a ghost half for
    # odd batches; must equal the one-image calls (full-warp strips) bit for bit
    for (nb, hh, ww) in ((2, 29, 80), (3, 23, 92), (3, 19, 63), (2, 17, 155), (5, 21, 142)):
        xb = np.stack([vfsynth.random_image(300 + 7 * i + ww, hh, ww) for i in range(nb)])
        xbt = torch.from_numpy(xb).cuda()
        ob, ib, ab = vfb.filter(xbt, 3, "angular", var, want_index=True, want_agg=True)
        pout = torch.empty_like(xbt)
        plan = vfb.Plan(xbt, [pout], 3, [("angular", var)])
        half = ww - 62 * ((ww + 61) // 62 - 1) <= 30
        assert plan.kernels() == (2 if half else 1), (ww, plan.kernels())
        plan.launch()
        torch.cuda.synchronize()
        assert torch.equal(pout, ob), (var, ww)
        plan.close()
        for i in range(nb):
            e_out, e_idx, e_agg = vfb.filter(torch.from_numpy(xb[i]).cuda(), 3, "angular", var, want_index=True,
                                             want_agg=True)
            torch.cuda.synchronize()
            assert torch.equal(ob[i], e_out) and torch.equal(ib[i], e_idx) and torch.equal(ab[i], e_agg), (var, ww, i)
        _, o_idx, o_agg = oracle.filter_image(xb[nb - 1], 3, "angular", var, want_agg=True)
        rep = check_parity(xb[nb - 1], 3, ob[nb - 1].cpu().numpy(), ib[nb - 1].cpu().numpy(),
                           ab[nb - 1].cpu().numpy(), o_idx, o_agg)
        assert rep["ok"], (var, ww, rep)
print("stream paths ok")
