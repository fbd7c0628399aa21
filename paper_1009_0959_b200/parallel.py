"""Multi-GPU partitioner: one process per GPU, torch.distributed
(NCCL over NVLink/NVSwitch on B200 nodes; gloo in the CPU tests).

The filter is embarrassingly parallel: every output pixel depends only on its
(2r+1)^2 input neighbourhood, so there is no exchange on the data path.
* Batch sharding (BASELINE config 3 / C4): rank r filters images
  [r B / k, (r+1) B / k); the per-image statistics of the outputs against
  their references (e.g. each minimax filter against the exact one of its
  criterion, the paper's fidelity measure) come from one fused pass per
  reference (vf_image_stats_multi) and cross ranks in ONE all_gather
  (B x comparisons x 8 doubles).
* Row stripes (config 4 / C5): rank r owns output rows [r H / k, (r+1) H / k)
  and reads them plus w//2 halo rows on each interior side (clamped at the
  global border); the output is gathered in row chunks, the all_gather of
  chunk i (NCCL's stream) overlapping the filtering of chunk i + 1.
Outputs are bit-identical to the single-GPU result for every k (tested).
Ranks with no work (B < k images, H < k rows) still take part in every
collective with empty contributions, so no rank blocks.

The per-rank compute is injectable (`filter_fn`, `stats_fn`) so the
partitioning and collective logic can be tested on CPU with gloo; the
defaults call the CUDA library (no CPU fallback).
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import torch
import torch.distributed as dist


# ----------------------------------------------------------------- partitions
def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous balanced split of n items: [lo, hi) of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def stripe_bounds(H: int, world: int, rank: int, window: int):
    """Rows of rank `rank`'s stripe: (out_row0, out_rows, band_row0, band_rows).
    The band holds the output rows plus w//2 halo rows on each side, clamped to
    the global image [0, H) (the kernel clamps against the GLOBAL rows, so the
    border replicate padding is unchanged by the split)."""
    r = window // 2
    lo, hi = shard_range(H, world, rank)
    blo, bhi = max(0, lo - r), min(H, hi + r)
    return lo, hi - lo, blo, bhi - blo


# ----------------------------------------------------------------- default compute (CUDA)
def _cuda_filter_batch(imgs: torch.Tensor, window: int, criterion, variant) -> torch.Tensor:
    from . import vf
    return vf.vf_filter_batch(imgs, window, criterion, variant)


def _cuda_filter_rows(band, band_row0, H, out_row0, out_rows, window, criterion, variant, out=None):
    from . import vf
    return vf.vf_filter_rows(band, band_row0, H, out_row0, out_rows, window, criterion, variant, out=out)


def _cuda_stats_multi(a: torch.Tensor, bs) -> torch.Tensor:
    """[len(bs), B, 8] float64: one fused pass over the reference (vf_image_stats_multi)."""
    from . import vf
    out = []
    for i in range(0, len(bs), 8):                        # the library compares up to 8 outputs per pass
        out.append(vf.vf_image_stats_multi(a, list(bs[i:i + 8])))
    return torch.cat(out) if len(out) > 1 else out[0]


# ----------------------------------------------------------------- batch sharding
def all_gather_rows(local: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """all_gather of per-rank row blocks with unequal row counts (possibly 0):
    pad to the largest count, all_gather_into_tensor, strip the padding."""
    world = len(counts)
    m = max(max(counts), 1)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[i * m: i * m + counts[i]] for i in range(world)])


def gather_group_stats(outs: dict, B: int, groups, group=None, stats_fn: Callable = _cuda_stats_multi):
    """Per-image statistics of output groups against their references, all
    ranks' images in batch order: groups = [(reference combo, [combo, ...]),
    ...] -> {(reference, combo): [B, 8] float64}.  One fused stats pass per
    group (stats_fn(ref, [outs...]) -> [n, B_local, 8]) and ONE all_gather of
    [B_local, sum n, 8]: the only cross-rank traffic of the batch path."""
    world = dist.get_world_size(group)
    counts = [shard_range(B, world, r)[1] - shard_range(B, world, r)[0] for r in range(world)]
    keys, parts = [], []
    for ref, cs in groups:
        ref = tuple(ref)
        cs = [tuple(c) for c in cs]
        keys += [(ref, c) for c in cs]
        a = outs[ref]
        if a.shape[0] > 0:
            parts.append(stats_fn(a, [outs[c] for c in cs]).to(torch.float64))     # [n, B_local, 8]
        else:
            parts.append(torch.zeros((len(cs), 0, 8), dtype=torch.float64, device=a.device))
    s = torch.cat(parts) if len(parts) > 1 else parts[0]
    g = all_gather_rows(s.permute(1, 0, 2).contiguous(), counts, group)   # [B, N, 8]
    return {k: g[:, i] for i, k in enumerate(keys)}


def gather_batch_stats(outs: dict, B: int, combos, reference: Optional[Tuple] = None, group=None,
                       stats_fn: Callable = _cuda_stats_multi):
    """Per-image statistics of every filter's local outputs against the
    `reference` combo's (default: the first), all_gathered over the ranks in
    batch order: {combo: [B, 8] float64} (one stats pass, one all_gather)."""
    ref = tuple(reference) if reference is not None else tuple(combos[0])
    res = gather_group_stats(outs, B, [(ref, [tuple(c) for c in combos])], group, stats_fn)
    return {c: v for (_, c), v in res.items()}


def run_batch_sharded(imgs_local: torch.Tensor, B: int, window: int, combos, reference: Optional[Tuple] = None,
                      group=None, filter_fn: Callable = _cuda_filter_batch, stats_fn: Callable = _cuda_stats_multi):
    """Filter this rank's shard of a B-image batch with every (criterion,
    variant) in `combos`; gather per-image statistics of each filter against
    the `reference` combo (default: the first) from all ranks.

    imgs_local: [B_local, H, W, 3] = images shard_range(B, world, rank) of the
    batch (B_local = 0 on ranks beyond B: they filter nothing but still join
    the collective).  Returns (local outputs {combo: tensor}, gathered stats
    {combo: [B, 8] float64}) -- the stats are the only data that crosses ranks."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if B < 1:
        raise ValueError("empty batch")
    lo, hi = shard_range(B, world, rank)
    if imgs_local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} expects {hi - lo} images, got {imgs_local.shape[0]}")
    if hi > lo:
        outs = {tuple(c): filter_fn(imgs_local, window, *c) for c in combos}
    else:
        outs = {tuple(c): torch.empty_like(imgs_local) for c in combos}
    return outs, gather_batch_stats(outs, B, combos, reference, group, stats_fn)


# ----------------------------------------------------------------- row stripes
def stripe_chunks(H: int, world: int, window: int, nchunks: int):
    """Chunk size (rows) of the chunked stripe gather: every rank's stripe is
    cut into `nchunks` chunks of the same padded size (the largest stripe /
    nchunks, rounded up), so each chunk is one equal-sized all_gather."""
    m = max(stripe_bounds(H, world, r, window)[1] for r in range(world))
    return max(1, -(-m // max(1, nchunks)))


def run_stripes(band: torch.Tensor, H: int, window: int, criterion, variant, group=None,
                filter_fn: Callable = _cuda_filter_rows, gather: bool = True, nchunks: int = 4):
    """Filter this rank's stripe of an H-row image from its band (rows
    stripe_bounds(...)[2:] of the image) and, if `gather`, assemble the full
    output on every rank.  filter_fn(band, band_row0, H, out_row0, out_rows,
    window, criterion, variant, out=...) writes the rows into `out`.  The
    stripe is filtered in `nchunks` row chunks; the all_gather of chunk i is
    issued asynchronously (on NCCL's stream) right after its filter call, so
    it overlaps the filtering of chunk i + 1.
    Returns (stripe, full_or_None)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out_row0, out_rows, band_row0, band_rows = stripe_bounds(H, world, rank, window)
    if band.shape[0] != band_rows:
        raise ValueError(f"rank {rank}: band must hold rows [{band_row0}, {band_row0 + band_rows})")
    W = band.shape[1]
    if not gather:
        if out_rows == 0:
            return band.new_empty((0, W, 3)), None
        return filter_fn(band, band_row0, H, out_row0, out_rows, window, criterion, variant), None
    cr = stripe_chunks(H, world, window, nchunks)
    nch = -(-max(stripe_bounds(H, world, r, window)[1] for r in range(world)) // cr)
    # padded local stripe: chunk j = rows [j cr, (j + 1) cr) of this rank's stripe
    local = band.new_zeros((nch * cr, W, 3))
    recv = band.new_empty((nch, world * cr, W, 3))
    works = []
    for j in range(nch):
        r0 = j * cr
        rows = min(cr, out_rows - r0)
        if rows > 0:
            chunk = local[r0: r0 + rows]                      # contiguous view
            res = filter_fn(band, band_row0, H, out_row0 + r0, rows, window, criterion, variant, out=chunk)
            if res.data_ptr() != chunk.data_ptr():
                chunk.copy_(res)
        works.append(dist.all_gather_into_tensor(recv[j], local[r0: r0 + cr], group=group, async_op=True))
    for wk in works:
        wk.wait()
    counts = [stripe_bounds(H, world, r, window)[1] for r in range(world)]
    # recv[j][r cr : (r + 1) cr] = chunk j of rank r
    parts = []
    for r in range(world):
        rr = recv[:, r * cr:(r + 1) * cr].reshape(nch * cr, W, 3)
        parts.append(rr[: counts[r]])
    full = torch.cat(parts)
    return local[:out_rows], full


def stats_summary(stats: torch.Tensor, H: int, W: int) -> dict:
    """MAE / MSE / PSNR / NCD / fraction of differing pixels from gathered
    [B, 8] stats (vf_image_stats layout), over the whole batch (max |a-b| is
    the batch maximum)."""
    import math
    s = stats.sum(0).tolist()
    B = stats.shape[0]
    npix = B * H * W
    mse = s[2] / (3 * npix)
    return {"images": B, "diff_frac": s[0] / npix, "mae": s[1] / (3 * npix), "mse": mse,
            "psnr_db": math.inf if mse == 0 else 10 * math.log10(255.0 ** 2 / mse),
            "ncd": s[3] / s[4] if s[4] > 0 else float("nan"), "max_abs": float(stats[:, 5].max()) if B else 0.0}
