"""Multi-process (gloo, CPU) tests of the partitioner's host logic: partitions,
halo bands, the stats all_gather and the stripe gather.  The per-rank compute
is the CPU oracle (tests may use it), so results must equal the single-process
oracle bit-exactly for every world size."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1009_0959_b200 import parallel as par


def test_shard_range_partitions():
    for n in [0, 1, 5, 8, 17, 1024]:
        for world in [1, 2, 3, 4, 8]:
            parts = [par.shard_range(n, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts, parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_stripe_bounds_halo_and_clamp():
    H = 4320
    for w in (3, 5):
        r = w // 2
        for world in (1, 2, 4, 8):
            rows = []
            for rank in range(world):
                o0, on, b0, bn = par.stripe_bounds(H, world, rank, w)
                rows.extend(range(o0, o0 + on))
                assert b0 == max(0, o0 - r) and b0 + bn == min(H, o0 + on + r)
            assert rows == list(range(H))


# ---------------------------------------------------------------- multi-process
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_filter_batch(imgs, window, crit, var):
    import oracle
    x = imgs.numpy()
    return torch.from_numpy(np.stack([oracle.filter_image(x[b], window, crit, var, want_index=False)[0]
                                      for b in range(x.shape[0])]))


def _numpy_stats_multi(a, bs):
    return torch.stack([_numpy_stats(a, b) for b in bs])


def _numpy_stats(a, b):
    from oracle import metrics
    a, b = a.numpy(), b.numpy()
    out = np.zeros((a.shape[0], 8))
    for i in range(a.shape[0]):
        ai, bi = a[i].astype(np.int64), b[i].astype(np.int64)
        out[i, 0] = (ai != bi).any(-1).sum()
        out[i, 1] = np.abs(ai - bi).sum()
        out[i, 2] = ((ai - bi) ** 2).sum()
        la, lb = metrics.rgb_to_lab(a[i]), metrics.rgb_to_lab(b[i])
        out[i, 3] = np.linalg.norm(la - lb, axis=-1).sum()
        out[i, 4] = np.linalg.norm(la, axis=-1).sum()
        out[i, 5] = np.abs(ai - bi).max()
    return torch.from_numpy(out)


def _oracle_filter_rows(band, band_row0, H, out_row0, out_rows, window, crit, var, out=None):
    """Stripe filter from the band only: rows outside the band are garbage
    (255) in the scratch image, so a wrong halo shows up as a mismatch."""
    import oracle
    b = band.numpy()
    W = b.shape[1]
    scratch = np.full((H, W, 3), 255, np.uint8)
    scratch[band_row0:band_row0 + b.shape[0]] = b
    ys, xs = np.meshgrid(np.arange(out_row0, out_row0 + out_rows), np.arange(W), indexing="ij")
    o, _, _ = oracle.filter_pixels(scratch, window, crit, var, ys.ravel(), xs.ravel(), want_agg=False)
    res = torch.from_numpy(o.reshape(out_rows, W, 3))
    if out is not None:
        out.copy_(res)
        return out
    return res


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import vfsynth
        # ---- batch sharding (C4-like, small)
        spec = vfsynth.ImageSpec("t", 24, 40, 5, (3,), 4, False, "uncorrelated", None,
                                 p_choices=(0.05, 0.3), seed=99)
        B = spec.batch
        lo, hi = par.shard_range(B, world, rank)
        local = torch.from_numpy(vfsynth.make_batch(spec, ids=range(lo, hi)))
        combos = [("angular", "exact"), ("angular", "minimax"), ("log", "minimax")]
        outs, stats = par.run_batch_sharded(local, B, 3, combos, filter_fn=_oracle_filter_batch,
                                            stats_fn=_numpy_stats_multi)
        # ---- stripes (C5-like, small): band generated locally, row-addressable
        spec5 = vfsynth.ImageSpec("t5", 37, 29, 1, (3, 5), 4, False, "correlated", 0.15, seed=7)
        res = {}
        for w in (3, 5):
            o0, on, b0, bn = par.stripe_bounds(spec5.H, world, rank, w)
            band = torch.from_numpy(vfsynth.make_image(spec5, 0, b0, b0 + bn)[1])
            stripe, full = par.run_stripes(band, spec5.H, w, "angular", "minimax", filter_fn=_oracle_filter_rows)
            res[w] = full.numpy()
        q.put((rank, {k: v.numpy() for k, v in stats.items()}, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multiprocess_batch_and_stripes(world):
    import oracle
    import vfsynth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process references
    spec = vfsynth.ImageSpec("t", 24, 40, 5, (3,), 4, False, "uncorrelated", None, p_choices=(0.05, 0.3), seed=99)
    full_b = torch.from_numpy(vfsynth.make_batch(spec))
    combos = [("angular", "exact"), ("angular", "minimax"), ("log", "minimax")]
    ref_out = {c: _oracle_filter_batch(full_b, 3, *c) for c in combos}
    ref_stats = {c: _numpy_stats(ref_out[combos[0]], ref_out[c]).numpy() for c in combos}
    spec5 = vfsynth.ImageSpec("t5", 37, 29, 1, (3, 5), 4, False, "correlated", 0.15, seed=7)
    img5 = vfsynth.make_image(spec5, 0)[1]
    for rank, stats, res in results:
        for c in combos:
            assert np.array_equal(stats[c], ref_stats[c]), (rank, c)
        for w in (3, 5):
            ref = oracle.filter_image(img5, w, "angular", "minimax", want_index=False)[0]
            assert np.array_equal(res[w], ref), (rank, w)
    # a filter against itself: no differing pixel, zero error (column 4 is the NCD denominator)
    z = ref_stats[("angular", "exact")]
    assert np.all(z[:, [0, 1, 2, 3, 5]] == 0) and np.all(z[:, 4] > 0)


# ---------------------------------------------------------------- C5 stripe bounds, world 4 / 8, empty shards
def _box_filter_rows(band, band_row0, H, out_row0, out_rows, window, crit, var, out=None):
    """A stand-in stripe filter that depends on every halo row: the
    per-channel max over the clamped (2r+1)-row vertical neighbourhood.  A
    wrong band, halo or clamp changes the result."""
    r = window // 2
    b = band.numpy()
    res = np.empty((out_rows, b.shape[1], 3), np.uint8)
    for i in range(out_rows):
        y = out_row0 + i
        rows = [min(max(y + d, 0), H - 1) - band_row0 for d in range(-r, r + 1)]
        assert all(0 <= q < b.shape[0] for q in rows), "read outside the band"
        res[i] = b[rows].max(0)
    t = torch.from_numpy(res)
    if out is not None:
        out.copy_(t)
        return out
    return t


def _box_ref(img, window):
    r = window // 2
    H = img.shape[0]
    return np.stack([img[[min(max(y + d, 0), H - 1) for d in range(-r, r + 1)]].max(0) for y in range(H)])


def _worker_c5(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W = 4320, 6                                   # C5's row count (BASELINE config 4), narrow rows
        rng = np.random.default_rng(5)
        img = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
        res = {}
        for w in (3, 5):
            for nch in (1, 4, 7):
                o0, on, b0, bn = par.stripe_bounds(H, world, rank, w)
                band = torch.from_numpy(np.ascontiguousarray(img[b0:b0 + bn]))
                stripe, full = par.run_stripes(band, H, w, "angular", "minimax", filter_fn=_box_filter_rows,
                                               nchunks=nch)
                res[(w, nch)] = (o0, stripe.numpy(), full.numpy())
        # empty shards: B < world images, H < world rows
        B = 2
        lo, hi = par.shard_range(B, world, rank)
        local = torch.zeros((hi - lo, 3, 3, 3), dtype=torch.uint8) + torch.arange(lo, hi, dtype=torch.uint8).view(-1, 1, 1, 1)
        combos = [("angular", "exact"), ("angular", "minimax")]

        def fake_filter(x, window, c, v):
            return x + (1 if v == "minimax" else 0)

        outs, stats = par.run_batch_sharded(local, B, 3, combos, filter_fn=fake_filter, stats_fn=_numpy_stats_multi)
        h_small = 3
        o0, on, b0, bn = par.stripe_bounds(h_small, world, rank, 3)
        band = torch.from_numpy(np.ascontiguousarray(img[:h_small][b0:b0 + bn]))
        _, full_small = par.run_stripes(band, h_small, 3, "angular", "minimax", filter_fn=_box_filter_rows)
        q.put((rank, res, {k: v.numpy() for k, v in stats.items()}, full_small.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_multiprocess_c5_stripes_and_empty_shards(world):
    """World sizes 4 and 8 with C5's real stripe bounds (H = 4320): every
    chunking of the overlapped gather reassembles the single-process result;
    ranks with empty shards (B = 2 images, H = 3 rows < world) still join the
    collectives (no hang) and the gathered stats are complete."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_c5, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (4320, 6, 3), dtype=np.uint8)
    refs = {w: _box_ref(img, w) for w in (3, 5)}
    small = _box_ref(img[:3], 3)
    for rank, res, stats, full_small in results:
        for (w, nch), (o0, stripe, full) in res.items():
            assert np.array_equal(full, refs[w]), (rank, w, nch)
            assert np.array_equal(stripe, refs[w][o0:o0 + stripe.shape[0]]), (rank, w, nch)
        assert np.array_equal(full_small, small), rank
        mm = stats[("angular", "minimax")]
        assert mm.shape == (2, 8) and np.all(mm[:, 0] == 9) and np.all(mm[:, 1] == 27)
        assert np.all(stats[("angular", "exact")][:, 0] == 0)


# ---------------------------------------------------------------- bench warm-up with a collective per step
def _worker_warmup(rank, world, port, q):
    import sys
    import time
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    calls = []

    def step():                          # unequal step times + one collective per step (as C4's stats all_gather)
        time.sleep(0.004 * (rank + 1))
        t = torch.ones(1)
        dist.all_reduce(t)
        calls.append(float(t.item()))
    if rank == 0:
        time.sleep(0.3)                  # ranks start their warm-up at different times
    n = bench.joint_warmup(step, lambda: None, torch, dist, "cpu", 3, 0.5)
    t = torch.tensor([float(n)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)   # would hang / mismatch if the counts differed
    q.put((rank, n, len(calls), float(t.item()), set(calls)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_joint_warmup_same_step_count(world):
    """bench.py's warm-up: every rank runs the same number of steps although
    their step times and start times differ (a per-rank time test deadlocked
    the N > 1 C4 bench in round 2: the first rank to stop entered the barrier
    while the others were still in the step's all_gather)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_warmup, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    counts = {n for _, n, _, _, _ in res}
    assert len(counts) == 1 and min(counts) >= 3, res
    for _, n, ncalls, tmax, sums in res:
        assert ncalls == n and tmax == n and sums == {float(world)}
