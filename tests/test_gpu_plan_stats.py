"""GPU: plans with fidelity statistics (vf_plan_create_ex).  The statistics a
plan computes -- one statistics node per reference, after the nodes writing
its inputs, then a finalize node -- must be bit-identical to
vf_image_stats_multi over the plan's own outputs (per-pixel fixed-point sums
do not depend on how the outputs are grouped, include/vf.h), on every launch,
and the outputs must be those of a plan without statistics.
vf_image_stats_multi itself is checked against the float64 metrics oracle in
test_gpu_parity.py."""
import dataclasses

import pytest

import vfsynth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1009_0959_b200 as vfb  # noqa: E402

CV7 = [("angular", "exact"), ("angular", "minimax"), ("exp", "exact"), ("exp", "minimax"),
       ("exp", "poly4"), ("log", "exact"), ("log", "minimax")]
PAPER_REFS = [-1, 0, -1, 2, 2, -1, 5]          # each approximant against its exact filter (the bench's step)
STRESS_REFS = [1, 0, 5, 2, 5, 3, 4]            # every filter compared, many differing pixels, both directions


def expected_stats(outs, refs):
    rows = []
    for i, r in enumerate(refs):
        if r >= 0:
            rows.append(vfb.vf_image_stats_multi(outs[r], [outs[i]])[0])
    return torch.stack(rows)


def run_plan(x, combos, refs, w=3, launches=2):
    outs = [torch.empty_like(x) for _ in combos]
    ncmp = sum(1 for r in refs if r >= 0)
    st = torch.full((ncmp, x.shape[0], 8), float("nan"), dtype=torch.float64, device=x.device)
    plan = vfb.Plan(x, outs, w, combos, refs=refs, stats=st)
    got = []
    for _ in range(launches):
        plan.launch()
        torch.cuda.synchronize()
        got.append(st.clone())
    return plan, outs, got


@pytest.mark.parametrize("refs", [PAPER_REFS, STRESS_REFS], ids=["paper", "stress"])
def test_plan_stats_fused_nodes_bit_identical(refs):
    """C4-shaped batch (both fusions apply); statistics nodes depend on fused
    nodes."""
    spec = dataclasses.replace(vfsynth.config("C4"), batch=32)
    x = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
    plan, outs, got = run_plan(x, CV7, refs)
    # exp/log node, angular node + remainder strips, one statistics node per reference, finalize
    assert plan.kernels() == 3 + len(set(r for r in refs if r >= 0)) + 1
    want = expected_stats(outs, refs)
    for g in got:                                  # every launch re-zeroes and recomputes
        assert torch.equal(g, want)
    assert float(want[:, :, 4].min()) > 0          # reference norms present
    if refs is STRESS_REFS:
        assert float(want[:, :, 0].sum()) > 1e4    # the diff path (atomics) is exercised
    # outputs are those of a plan without statistics
    plain = [torch.empty_like(x) for _ in CV7]
    vfb.Plan(x, plain, 3, CV7).launch()
    torch.cuda.synchronize()
    for a, b in zip(outs, plain):
        assert torch.equal(a, b)


def test_plan_stats_ragged_tiles():
    """500 x 700 images (ragged tiles, half-warp remainder strips 700 = 11 x 62
    + 18, an odd batch) and an image size that is not a multiple of 4 pixels
    (the statistics pass's one-pixel path)."""
    spec = dataclasses.replace(vfsynth.config("C4"), batch=33, H=500, W=700)
    x = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
    plan, outs, got = run_plan(x, CV7, STRESS_REFS, launches=1)
    assert plan.kernels() == 3 + 6 + 1
    assert torch.equal(got[0], expected_stats(outs, STRESS_REFS))
    spec = dataclasses.replace(vfsynth.config("C4"), batch=3, H=61, W=97)      # 5917 px per image
    x = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
    plan, outs, got = run_plan(x, CV7, STRESS_REFS, launches=1)
    assert torch.equal(got[0], expected_stats(outs, STRESS_REFS))


@pytest.mark.parametrize("w", [3, 5])
def test_plan_stats_nodes_small_and_cross(w):
    """One C2 image (no fusion: one statistics node per reference) and
    cross-criterion references."""
    _, img = vfsynth.make_image(vfsynth.config("C2"), 0)
    x = torch.from_numpy(img).cuda().unsqueeze(0).contiguous()
    refs = [-1, 0, 0, 2, 1, 3, 2]
    plan, outs, got = run_plan(x, CV7, refs)
    want = expected_stats(outs, refs)
    for g in got:
        assert torch.equal(g, want)


def test_plan_stats_cross_node_in_fused_plan():
    """A fused plan with comparisons across its nodes (log minimax against
    angular exact, angular minimax against exp exact): each statistics node
    depends on both producers."""
    spec = dataclasses.replace(vfsynth.config("C4"), batch=32)
    x = torch.from_numpy(vfsynth.make_batch(spec)).cuda()
    refs = [-1, 2, -1, 2, 2, -1, 0]
    plan, outs, got = run_plan(x, CV7, refs)
    assert plan.kernels() == 3 + 2 + 1             # + a statistics node per reference + finalize
    assert torch.equal(got[-1], expected_stats(outs, refs))


def test_plan_stats_argument_errors():
    x = torch.zeros((1, 16, 16, 3), dtype=torch.uint8, device="cuda")
    outs = [torch.empty_like(x) for _ in CV7[:2]]
    st = torch.zeros((1, 1, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(vfb.VFError):
        vfb.Plan(x, outs, 3, CV7[:2], refs=[0, -1], stats=st)          # self-reference
    with pytest.raises(vfb.VFError):
        vfb.Plan(x, outs, 3, CV7[:2], refs=[-1, 5], stats=st)          # out of range
    with pytest.raises(ValueError):
        vfb.Plan(x, outs, 3, CV7[:2], refs=[-1, 0], stats=st[:, :, :4])   # wrong size
    with pytest.raises(ValueError):
        vfb.Plan(x, outs, 3, CV7[:2], refs=[-1, 0], stats=None)
    # refs all -1: a plain plan, no statistics buffer needed
    p = vfb.Plan(x, outs, 3, CV7[:2], refs=[-1, -1])
    p.launch()
    torch.cuda.synchronize()
