"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs, with the acceptance rule of tests/parity.py (aggregates
within 1e-5 relative, selected index exact unless the oracle's candidates are
within 1e-5 relative, output = the window sample at the selected index)."""
import dataclasses
import os

import numpy as np
import pytest

import oracle
import vfsynth
from tests.parity import check_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1009_0959_b200 as vfb  # noqa: E402

CV = [("angular", "exact"), ("angular", "minimax"), ("exp", "exact"), ("exp", "minimax"),
      ("exp", "poly4"), ("log", "exact"), ("log", "minimax"), ("exp", "reach"), ("log", "reach")]


def gpu_full(img_np, w, crit, var, algo="auto"):
    x = torch.from_numpy(np.ascontiguousarray(img_np)).cuda()
    out, idx, agg = vfb.filter(x, w, crit, var, algo=algo, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    return out.cpu().numpy(), idx.cpu().numpy(), agg.cpu().numpy()


def full_parity(img_np, w, crit, var, algo=None):
    """Every kernel variant is checked unless `algo` is given: angular default
    (3x3 minimax: the warp-streamed kernel), per-window and pair-sharing with
    each region height (1..3 pixels per thread); exp/log with 1 and (3x3) 2
    output rows per thread."""
    if algo:
        algos = [algo]
    elif crit == "angular":
        algos = ["auto", "stream", "window", "shared", "shared:1", "shared:2", "shared:3", "role", "role:1",
                 "role:2", "role:3"]
    else:
        # tile bits force the TMA-staged kernel where the rows allow it (3W % 16 == 0);
        # "+notma" the plain-load one
        algos = ["auto", "auto:1", "auto:2", "auto:3"] if w == 3 else ["auto", "auto:1"]
        algos += [a + "+notma" for a in algos[1:]]
    _, o_idx, o_agg = oracle.filter_image(img_np, w, crit, var, want_agg=True)
    for a in algos:
        g_out, g_idx, g_agg = gpu_full(img_np, w, crit, var, a)
        rep = check_parity(img_np, w, g_out, g_idx, g_agg, o_idx, o_agg)
        assert rep["ok"], (a, rep)
    return rep


# ------------------------------------------------------------- config images
@pytest.mark.parametrize("var", ["exact", "minimax"])
def test_c1_angular(var):
    _, x = vfsynth.make_image(vfsynth.config("C1"), 0)
    full_parity(x, 3, "angular", var)


@pytest.mark.parametrize("crit,var", CV)
def test_c2_all_criteria(crit, var):
    _, x = vfsynth.make_image(vfsynth.config("C2"), 0)
    full_parity(x, 3, crit, var)


@pytest.mark.parametrize("crit,var", CV)
def test_5x5_midsize(crit, var):
    spec = dataclasses.replace(vfsynth.config("C3"), H=203, W=301)   # several tiles + ragged tail
    _, x = vfsynth.make_image(spec, 0)
    full_parity(x, 5, crit, var)


# ------------------------------------------------------------- edge cases
RAGGED = [(3, 3), (5, 5), (3, 37), (37, 3), (9, 200), (41, 33), (8, 32), (17, 65)]


@pytest.mark.parametrize("crit,var", CV)
@pytest.mark.parametrize("w", [3, 5])
def test_ragged_sizes(crit, var, w):
    for H, W in RAGGED:
        if w > min(H, W):
            continue
        x = vfsynth.random_image(11 + H, H, W)
        full_parity(x, w, crit, var)


@pytest.mark.parametrize("crit,var", CV)
@pytest.mark.parametrize("w", [3, 5])
def test_misaligned_rows_and_image_bases(crit, var, w):
    """Interior tiles are staged as whole 32-bit words: cover row strides that
    are not a multiple of 4 bytes (W = 131, 3W = 393), batches whose images
    start at odd byte offsets (H*W*3 odd), and an input starting at byte 1 of
    its allocation -- against the oracle and bit-exact between layouts."""
    x = vfsynth.random_image(31, 75, 131)
    full_parity(x, w, crit, var)
    g_out, g_idx, g_agg = gpu_full(x, w, crit, var)
    buf = torch.zeros(x.size + 1, dtype=torch.uint8, device="cuda")
    xv = buf[1:].view(x.shape)
    xv.copy_(torch.from_numpy(x))
    out, idx, agg = vfb.filter(xv, w, crit, var, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), g_out)
    assert np.array_equal(idx.cpu().numpy(), g_idx)
    assert np.array_equal(agg.cpu().numpy(), g_agg)
    xb = np.stack([vfsynth.random_image(40 + b, 41, 101) for b in range(3)])   # 41*101*3 = 12423 (odd)
    ob, ib, ab = vfb.filter(torch.from_numpy(xb).cuda(), w, crit, var, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    for b in range(3):
        e_out, e_idx, e_agg = gpu_full(xb[b], w, crit, var)
        assert np.array_equal(ob[b].cpu().numpy(), e_out)
        assert np.array_equal(ib[b].cpu().numpy(), e_idx)
        assert np.array_equal(ab[b].cpu().numpy(), e_agg)


@pytest.mark.parametrize("crit,var", [c for c in CV if c[0] != "angular"])
@pytest.mark.parametrize("w", [3, 5])
def test_tma_path_borders_batches_stripes(crit, var, w):
    """The persistent TMA-staged exp/log kernel (3W % 16 == 0): ragged tile
    tails in both directions, border tiles (zero-filled box + replicate
    clamp), a batch (3-D tensor map), row stripes (band-relative rows) -- all
    bit-identical to the plain-load kernel, and the image against the oracle."""
    x = vfsynth.random_image(51, 77, 144)            # 3*144 = 432 = 27*16
    full_parity(x, w, crit, var)
    for a in (["auto:1", "auto:2", "auto:3"] if w == 3 else ["auto:1"]):
        t = gpu_full(x, w, crit, var, a)
        n = gpu_full(x, w, crit, var, a + "+notma")
        for u, v in zip(t, n):
            assert np.array_equal(u, v), a
    xb = np.stack([vfsynth.random_image(60 + b, 45, 96) for b in range(3)])
    ob, ib, ab = vfb.filter(torch.from_numpy(xb).cuda(), w, crit, var, algo="auto:1", want_index=True,
                            want_agg=True)
    torch.cuda.synchronize()
    for b in range(3):
        e_out, e_idx, e_agg = gpu_full(xb[b], w, crit, var, "auto:1+notma")
        assert np.array_equal(ob[b].cpu().numpy(), e_out)
        assert np.array_equal(ib[b].cpu().numpy(), e_idx)
        assert np.array_equal(ab[b].cpu().numpy(), e_agg)


def test_tma_path_row_stripes():
    """Row stripes through the TMA-staged kernel (forced in a child process)
    equal the full image on the plain-load kernel, bit for bit."""
    import subprocess
    import sys
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tma_stripes_child.py")
    r = subprocess.run([sys.executable, child], env=dict(os.environ, VF_FORCE_TMA="1"), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "tma stripes ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_stream_kernel_paths():
    """The streamed 3x3 angular kernels (forced at every size in a child
    process, VF_ANG3_STREAM=1): oracle parity, row stripes, batches, odd
    strides and a misaligned base are bit-identical to the whole-image call."""
    import subprocess
    import sys
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)), "stream_paths_child.py")
    r = subprocess.run([sys.executable, child], env=dict(os.environ, VF_ANG3_STREAM="1"), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "stream paths ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


def test_el_block_shapes_bit_identical():
    """exp/log 3x3 large launches: the default 4-warp x 4-row blocks, the
    8-warp blocks with 4 or 2 rows and 4-warp x 2-row blocks give bit-identical
    outputs, indices and aggregates (child processes: the shape knobs are read
    once per process)."""
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    import el_blocks_child
    ref = el_blocks_child.digests()
    child = os.path.join(here, "el_blocks_child.py")
    for env in ({"VF_EL_TY": "8", "VF_EL_OPT": "4"}, {"VF_EL_TY": "8", "VF_EL_OPT": "2"},
                {"VF_EL_TY": "4", "VF_EL_OPT": "2"}):
        r = subprocess.run([sys.executable, child], env=dict(os.environ, **env), capture_output=True, text=True,
                           timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        got = dict(line.split() for line in r.stdout.strip().splitlines())
        assert got == ref, (env, got, ref)


@pytest.mark.parametrize("crit,var", CV)
@pytest.mark.parametrize("w", [3, 5])
def test_palette_ties_zero_vectors_branch_points(crit, var, w):
    """Few channel levels: duplicate samples (exact ties), parallel vectors,
    black pixels (zero-vector rule S:342) and cos = 0.5 pairs."""
    x = vfsynth.small_palette_image(5, 67, 71)
    full_parity(x, w, crit, var)
    x2 = vfsynth.small_palette_image(6, 40, 50, levels=(0, 0, 0, 60, 120))   # many black pixels
    full_parity(x2, w, crit, var)


@pytest.mark.parametrize("crit,var", CV)
def test_constant_and_black_images(crit, var):
    for val in [(0, 0, 0), (255, 255, 255), (12, 200, 7)]:
        x = np.empty((19, 45, 3), np.uint8)
        x[...] = val
        for w in (3, 5):
            g_out, g_idx, g_agg = gpu_full(x, w, crit, var)
            assert np.array_equal(g_out, x)
            assert np.all(g_idx == 0)
            full_parity(x, w, crit, var)


@pytest.mark.parametrize("crit,var", CV)
def test_branch_point_image(crit, var):
    """Every pixel is one of (v,v,0), (0,v,v), (v,0,v): all cross pairs sit
    exactly on cos = 0.5, where the two Table 1 rows differ by 3.1e-5."""
    rng = np.random.default_rng(3)
    v = rng.integers(1, 256, size=(30, 40))
    k = rng.integers(0, 3, size=(30, 40))
    x = np.zeros((30, 40, 3), np.uint8)
    for c in range(3):
        x[..., c] = np.where((k == c) | (k == (c + 1) % 3), v, 0)
    full_parity(x, 3, crit, var)
    full_parity(x, 5, crit, var)


# ------------------------------------------------------------- batch / rows / host API
@pytest.mark.parametrize("crit,var", [("angular", "minimax"), ("exp", "minimax"), ("log", "exact")])
def test_batch_matches_per_image(crit, var):
    spec = dataclasses.replace(vfsynth.config("C4"), H=64, W=96, batch=3)
    xb = vfsynth.make_batch(spec)
    xt = torch.from_numpy(xb).cuda()
    out, idx, agg = vfb.filter(xt, 3, crit, var, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    for b in range(3):
        _, o_idx, o_agg = oracle.filter_image(xb[b], 3, crit, var, want_agg=True)
        rep = check_parity(xb[b], 3, out[b].cpu().numpy(), idx[b].cpu().numpy(), agg[b].cpu().numpy(),
                           o_idx, o_agg)
        assert rep["ok"], (b, rep)


@pytest.mark.parametrize("w", [3, 5])
@pytest.mark.parametrize("crit,var", [("angular", "minimax"), ("angular", "exact"), ("log", "minimax")])
def test_row_stripes_equal_full_image(w, crit, var):
    """Stripes with w//2 halo rows, clamped at the global border, reproduce the
    full-image result bit-exactly (the per-pixel computation does not depend
    on the partition)."""
    x = vfsynth.random_image(21, 53, 70)
    H, W = x.shape[:2]
    full, fidx, fagg = gpu_full(x, w, crit, var)
    r = w // 2
    for k in (1, 2, 3, 4, 7):
        bounds = np.linspace(0, H, k + 1).astype(int)
        for a, b in zip(bounds[:-1], bounds[1:]):
            lo, hi = max(0, a - r), min(H, b + r)
            band = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
            idx = torch.empty((b - a, W), dtype=torch.uint8, device="cuda")
            agg = torch.empty((b - a, W, w * w), dtype=torch.float32, device="cuda")
            out = vfb.vf_filter_rows(band, lo, H, a, b - a, w, crit, var, index=idx, aggregates=agg)
            torch.cuda.synchronize()
            assert np.array_equal(out.cpu().numpy(), full[a:b])
            assert np.array_equal(idx.cpu().numpy(), fidx[a:b])
            assert np.array_equal(agg.cpu().numpy(), fagg[a:b])


def test_rows_invalid_band_rejected():
    x = torch.zeros((20, 30, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(vfb.VFError) as e:
        vfb.vf_filter_rows(x[2:10].contiguous(), 2, 40, 5, 5, 5, "angular", "minimax")   # needs rows 3..11
    assert e.value.status == -1


def test_host_api_matches_device_api():
    _, x = vfsynth.make_image(vfsynth.config("C2"), 0)
    h = torch.from_numpy(x).pin_memory()
    ho = torch.empty_like(h).pin_memory()
    ws = torch.empty(vfb.vf_host_workspace_bytes(1, 512, 512), dtype=torch.uint8, device="cuda")
    for crit, var in CV:
        vfb.vf_filter_host(h, 3, crit, var, ho, ws)
        torch.cuda.synchronize()
        d, _, _ = gpu_full(x, 3, crit, var)
        assert np.array_equal(ho.numpy(), d), (crit, var)


def test_invalid_arguments_return_status():
    x = torch.zeros((16, 16, 3), dtype=torch.uint8, device="cuda")
    for w, c, v, st in [(4, "angular", "exact", -1), (7, "angular", "exact", -2), (3, "angular", "poly4", -1),
                        (3, 6, 0, -1), (3, 0, 9, -1), (3, "evmf", "poly4", -1), (17, "exp", "exact", -1),
                        (3, "angular", "reach", -1), (3, "amnfe", "reach", -1)]:
        with pytest.raises(vfb.VFError) as e:
            vfb.filter(x, w, c, v)
        assert e.value.status == st, (w, c, v)
    with pytest.raises(vfb.VFError):
        vfb.vf_filter_batch_algo(x, 3, "angular", "exact", out=x)    # aliasing


# ------------------------------------------------------------- stats kernel
def test_image_stats_against_numpy_metrics():
    from oracle import metrics
    rng = np.random.default_rng(0)
    a = rng.integers(0, 256, size=(2, 33, 47, 3)).astype(np.uint8)
    b = a.copy()
    m = rng.random(a.shape) < 0.1
    b[m] = rng.integers(0, 256, size=m.sum())
    s = vfb.vf_image_stats(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()).cpu().numpy()
    for i in range(2):
        npix = 33 * 47
        assert s[i, 0] == (a[i] != b[i]).any(-1).sum()
        assert s[i, 1] / (3 * npix) == pytest.approx(metrics.mae(a[i], b[i]), rel=1e-12)
        assert s[i, 2] / (3 * npix) == pytest.approx(metrics.mse(a[i], b[i]), rel=1e-12)
        assert s[i, 3] / s[i, 4] == pytest.approx(metrics.ncd(a[i], b[i]), rel=2e-6)   # fp32 Lab per pixel
        assert s[i, 5] == np.abs(a[i].astype(int) - b[i]).max()


def test_image_stats_without_reference_norm():
    """vf_image_stats_ex(VF_STATS_NO_REF_NORM): every column but 4 equals the
    full statistics (bit-exact: same per-pixel fp32 values, same summation),
    column 4 is 0; unknown flags are rejected."""
    rng = np.random.default_rng(1)
    a = rng.integers(0, 256, size=(3, 41, 37, 3)).astype(np.uint8)
    b = a.copy()
    m = rng.random(a.shape[:3]) < 0.3
    b[m] = rng.integers(0, 256, size=(m.sum(), 3))
    ta, tb = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    full = vfb.vf_image_stats(ta, tb).cpu().numpy()
    part = vfb.vf_image_stats(ta, tb, ref_norm=False).cpu().numpy()
    for k in (0, 1, 2, 5):
        assert np.array_equal(full[:, k], part[:, k])
    assert np.allclose(part[:, 3], full[:, 3], rtol=1e-6, atol=0)
    assert np.all(part[:, 4] == 0) and np.all(full[:, 4] > 0)
    from paper_1009_0959_b200 import vf as vfm
    L = vfm.load_library()
    st = torch.empty((3, 8), dtype=torch.float64, device="cuda")
    rc = L.vf_image_stats_ex(ta.data_ptr(), tb.data_ptr(), 3, 41, 37, st.data_ptr(), 2, None)
    assert rc == vfm.VF_EINVAL


def test_image_stats_multi_one_pass():
    """vf_image_stats_multi(a, [b_0..b_6]): row k is bit-identical to
    vf_image_stats(a, b_k) (same per-pixel values, same fixed-point sums),
    the statistics are bit-reproducible run to run, and each row matches the
    numpy metrics oracle; nb outside [1, 8] is rejected."""
    from oracle import metrics
    rng = np.random.default_rng(2)
    B, H, W = 3, 57, 83
    a = rng.integers(0, 256, size=(B, H, W, 3)).astype(np.uint8)
    bs = []
    for k in range(7):
        b = a.copy()
        m = rng.random(a.shape[:3]) < 0.05 * k
        b[m] = rng.integers(0, 256, size=(m.sum(), 3))
        bs.append(b)
    ta = torch.from_numpy(a).cuda()
    tbs = [torch.from_numpy(b).cuda() for b in bs]
    multi = vfb.vf_image_stats_multi(ta, tbs).cpu().numpy()
    again = vfb.vf_image_stats_multi(ta, tbs).cpu().numpy()
    assert multi.shape == (7, B, 8) and np.array_equal(multi, again)
    for k in range(7):
        single = vfb.vf_image_stats(ta, tbs[k]).cpu().numpy()
        assert np.array_equal(multi[k], single), k
        for i in range(B):
            npix = H * W
            assert multi[k, i, 0] == (a[i] != bs[k][i]).any(-1).sum()
            assert multi[k, i, 1] / (3 * npix) == pytest.approx(metrics.mae(a[i], bs[k][i]), rel=1e-12, abs=0)
            assert multi[k, i, 2] / (3 * npix) == pytest.approx(metrics.mse(a[i], bs[k][i]), rel=1e-12, abs=0)
            if k:
                assert multi[k, i, 3] / multi[k, i, 4] == pytest.approx(metrics.ncd(a[i], bs[k][i]), rel=2e-6)
    assert np.all(multi[0, :, [0, 1, 2, 3, 5]] == 0)               # b_0 == a
    nr = vfb.vf_image_stats_multi(ta, tbs, ref_norm=False).cpu().numpy()
    assert np.all(nr[:, :, 4] == 0) and np.array_equal(nr[:, :, [0, 1, 2, 5]], multi[:, :, [0, 1, 2, 5]])
    with pytest.raises(ValueError):
        vfb.vf_image_stats_multi(ta, tbs + tbs)
    with pytest.raises(ValueError):
        vfb.vf_image_stats_multi(ta, [tbs[0][:, :10]])


# ------------------------------------------------------------- full-size configs (sampled)
def _sample_pixels(H, W, n, seed):
    rng = np.random.default_rng(seed)
    ys = rng.integers(0, H, size=n)
    xs = rng.integers(0, W, size=n)
    # all four borders too
    by = np.concatenate([np.zeros(W, int), np.full(W, H - 1), np.arange(H), np.arange(H)])
    bx = np.concatenate([np.arange(W), np.arange(W), np.zeros(H, int), np.full(H, W - 1)])
    sel = np.random.default_rng(seed + 1).permutation(by.shape[0])[:4000]
    return np.concatenate([ys, by[sel]]), np.concatenate([xs, bx[sel]])


def sampled_parity(img_np, w, crit, var, g_out, g_idx, g_agg, nsample=20000, seed=0):
    H, W = img_np.shape[:2]
    ys, xs = _sample_pixels(H, W, nsample, seed)
    _, o_idx, o_agg = oracle.filter_pixels(img_np, w, crit, var, ys, xs)
    rep = check_parity(img_np, w, g_out[ys, xs], g_idx[ys, xs], g_agg[ys, xs], o_idx, o_agg, ys=ys, xs=xs)
    assert rep["ok"], rep
    return rep


@pytest.mark.parametrize("crit,var", CV)
def test_c3_full_size_sampled(crit, var):
    """C3: 8 x 2048 x 2048, 5x5, the bench's launch configuration (whole batch
    in one call); sampled pixels of images 0 and 7 against the oracle."""
    spec = vfsynth.config("C3")
    xb = vfsynth.make_batch(spec, ids=range(8))
    xt = torch.from_numpy(xb).cuda()
    out, idx, agg = vfb.filter(xt, 5, crit, var, want_index=True, want_agg=True)
    torch.cuda.synchronize()
    for b in (0, 7):
        sampled_parity(xb[b], 5, crit, var, out[b].cpu().numpy(), idx[b].cpu().numpy(), agg[b].cpu().numpy(),
                       nsample=4000, seed=b)


@pytest.mark.parametrize("w", [3, 5])
def test_c5_full_size_sampled(w):
    """C5: one 4320 x 7680 image, minimax angular."""
    _, x = vfsynth.make_image(vfsynth.config("C5"), 0)
    xt = torch.from_numpy(x).cuda()
    out, idx, agg = vfb.filter(xt, w, "angular", "minimax", want_index=True, want_agg=True)
    torch.cuda.synchronize()
    sampled_parity(x, w, "angular", "minimax", out.cpu().numpy(), idx.cpu().numpy(), agg.cpu().numpy(),
                   nsample=20000 if w == 3 else 5000)


@pytest.mark.parametrize("crit,var", CV)
def test_c4_full_batch_sampled(crit, var):
    """C4: 1024 x 512 x 768 in one batched call; sampled pixels of 3 images."""
    spec = vfsynth.config("C4")
    ids = [0, 511, 1023]
    xb = vfsynth.make_batch(spec, ids=ids)
    full = torch.empty((1024, 512, 768, 3), dtype=torch.uint8, device="cuda")
    full.random_(0, 256, generator=torch.Generator(device="cuda").manual_seed(1))
    for j, b in enumerate(ids):
        full[b] = torch.from_numpy(xb[j]).cuda()
    out, idx, _ = vfb.filter(full, 3, crit, var, want_index=True)
    torch.cuda.synchronize()
    # the per-image call must use the batched call's kernel (the angular
    # default depends on the launch size: streamed for the batch; the exp/log
    # kernels of different tile shapes are bit-identical by construction)
    algo = "stream" if crit == "angular" else "auto"
    if crit == "angular":
        assert vfb.vf_kernel_info(1024, 512, 768, 3, crit, var)["name"] == \
            vfb.vf_kernel_info(1, 512, 768, 3, crit, var, algo)["name"]
    for j, b in enumerate(ids):
        sub = full[b:b + 1]
        o2, i2, a2 = vfb.filter(sub.contiguous(), 3, crit, var, algo=algo, want_index=True, want_agg=True)
        assert torch.equal(o2[0], out[b]) and torch.equal(i2[0], idx[b])
        sampled_parity(xb[j], 3, crit, var, o2[0].cpu().numpy(), i2[0].cpu().numpy(), a2[0].cpu().numpy(),
                       nsample=5000, seed=b)


def test_c4_bench_plan_sampled():
    """The bench's timed launch configuration: the 7-filter plan over the full
    1024 x 512 x 768 batch (3 kernel nodes: pair-major exp/log, fused angular,
    angular remainder strips).  For 3 images (first, middle, last) every
    filter's plan output equals the one-image call bit for bit, and that
    call's sampled pixels pass the oracle parity check."""
    import bench
    spec = vfsynth.config("C4")
    ids = [0, 511, 1023]
    xb = vfsynth.make_batch(spec, ids=ids)
    full = torch.empty((1024, 512, 768, 3), dtype=torch.uint8, device="cuda")
    full.random_(0, 256, generator=torch.Generator(device="cuda").manual_seed(2))
    for j, b in enumerate(ids):
        full[b] = torch.from_numpy(xb[j]).cuda()
    outs = [torch.empty_like(full) for _ in bench.COMBOS]
    plan = vfb.Plan(full, outs, 3, bench.COMBOS)
    assert plan.kernels() == 3
    plan.launch()
    torch.cuda.synchronize()
    for (crit, var), o in zip(bench.COMBOS, outs):
        algo = "stream" if crit == "angular" else "auto"
        for j, b in enumerate(ids):
            o2, i2, a2 = vfb.filter(full[b:b + 1].contiguous(), 3, crit, var, algo=algo, want_index=True,
                                    want_agg=True)
            torch.cuda.synchronize()
            assert torch.equal(o2[0], o[b]), (crit, var, b)
            sampled_parity(xb[j], 3, crit, var, o2[0].cpu().numpy(), i2[0].cpu().numpy(), a2[0].cpu().numpy(),
                           nsample=1500, seed=100 + b)
    plan.close()
    del outs, full
    torch.cuda.empty_cache()


# ------------------------------------------------------------- plan (CUDA-graph executor)
def test_fused_plan_large_batch():
    """A plan of >= 2^21 pixels fuses its exp/log filters into one kernel node
    (shared staging and S1) and its angular exact + minimax into another (one
    geometry evaluation; plus the half-warp remainder-strip node): 3 kernel
    nodes for the 7 filters, outputs
    bit-identical to each filter's own kernel, and to VF_PLAN_FUSE=0 plans
    (the single-filter nodes)."""
    spec = dataclasses.replace(vfsynth.config("C4"), batch=32)
    xb = torch.from_numpy(vfsynth.make_batch(spec)).cuda()          # 32 x 512 x 768: both fusions apply
    combos = CV[:7]
    outs = [torch.empty_like(xb) for _ in combos]
    plan = vfb.Plan(xb, outs, 3, combos)
    assert plan.kernels() == 3                  # exp/log node + angular node + its remainder strips (768 = 12 x 62 + 24)
    plan.launch()
    torch.cuda.synchronize()
    for (crit, var), o in zip(combos, outs):
        ref = vfb.filter(xb, 3, crit, var)[0]
        torch.cuda.synchronize()
        assert torch.equal(o, ref), (crit, var)
    small = vfb.Plan(xb[:1].contiguous(), [torch.empty_like(xb[:1]) for _ in combos], 3, combos)
    assert small.kernels() == 7
    mid = vfb.Plan(xb[:6].contiguous(), [torch.empty_like(xb[:6]) for _ in combos], 3, combos)
    assert mid.kernels() == 4       # exp/log fused; angular exact block kernel, minimax streamed (+ remainder strips)



@pytest.mark.parametrize("w", [3, 5])
def test_plan_matches_individual_filters(w):
    """A plan runs the 7 filters as independent graph nodes; outputs must be
    bit-identical to launching each filter alone, on every replay."""
    _, x = vfsynth.make_image(vfsynth.config("C2"), 0)
    xt = torch.from_numpy(x).cuda()
    outs = [torch.empty_like(xt) for _ in CV]
    plan = vfb.Plan(xt, outs, w, CV)
    for rep in range(3):
        for o in outs:
            o.zero_()
        plan.launch()
        torch.cuda.synchronize()
        for (crit, var), o in zip(CV, outs):
            ref, _, _ = vfb.filter(xt, w, crit, var)
            assert torch.equal(o, ref), (rep, crit, var)
    plan.close()


def test_host_plan_copies_inside_graph():
    spec = dataclasses.replace(vfsynth.config("C4"), H=96, W=128, batch=2)
    xb = vfsynth.make_batch(spec)
    h_in = torch.from_numpy(xb).pin_memory()
    h_outs = [torch.zeros_like(h_in).pin_memory() for _ in CV]
    d_in = torch.empty(h_in.shape, dtype=torch.uint8, device="cuda")
    d_outs = [torch.empty_like(d_in) for _ in CV]
    plan = vfb.Plan(d_in, d_outs, 3, CV, h_in=h_in, h_outs=h_outs)
    plan.launch()
    torch.cuda.synchronize()
    xt = torch.from_numpy(xb).cuda()
    for (crit, var), ho in zip(CV, h_outs):
        ref, _, _ = vfb.filter(xt, 3, crit, var)
        assert torch.equal(ho, ref.cpu()), (crit, var)
    # new host data is picked up by the next launch (pointers are bound, not data)
    h_in.copy_(torch.from_numpy(xb[::-1].copy()))
    plan.launch()
    torch.cuda.synchronize()
    ref, _, _ = vfb.filter(xt.flip(0).contiguous(), 3, *CV[1])
    assert torch.equal(h_outs[1], ref.cpu())
    plan.close()


def test_plan_rejects_bad_arguments():
    x = torch.zeros((16, 16, 3), dtype=torch.uint8, device="cuda")
    with pytest.raises(vfb.VFError):
        vfb.Plan(x, [x], 3, [("angular", "minimax")])                   # output aliases input
    o = torch.empty_like(x)
    with pytest.raises(vfb.VFError):
        vfb.Plan(x, [o, o], 3, [("angular", "minimax"), ("exp", "exact")])   # outputs overlap
    with pytest.raises(vfb.VFError):
        vfb.Plan(x, [o], 3, [("log", "poly4")])
