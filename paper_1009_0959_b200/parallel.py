"""Multi-GPU partitioner: one process per GPU, torch.distributed
(NCCL over NVLink/NVSwitch on B200 nodes; gloo in the CPU tests).

The filter is embarrassingly parallel: every output pixel depends only on its
(2r+1)^2 input neighbourhood, so there is no exchange on the data path.
* Batch sharding (BASELINE config 3 / C4): rank r filters images
  [r B / k, (r+1) B / k); the only collective is one all_gather of the
  per-image statistics (B x 8 doubles).
* Row stripes (config 4 / C5): rank r owns output rows [r H / k, (r+1) H / k)
  and reads them plus w//2 halo rows on each interior side (clamped at the
  global border); the output stripes are gathered to rank 0 (all_gather of
  equal-sized, padded stripes).
Outputs are bit-identical to the single-GPU result for every k (tested).

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


def _cuda_filter_rows(band, band_row0, H, out_row0, out_rows, window, criterion, variant):
    from . import vf
    return vf.vf_filter_rows(band, band_row0, H, out_row0, out_rows, window, criterion, variant)


def _cuda_stats(a: torch.Tensor, b: torch.Tensor, ref_norm: bool = True) -> torch.Tensor:
    from . import vf
    return vf.vf_image_stats(a, b, ref_norm=ref_norm)


# ----------------------------------------------------------------- batch sharding
def all_gather_rows(local: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """all_gather of per-rank row blocks with unequal row counts: pad to the
    largest count, all_gather_into_tensor, strip the padding."""
    world = len(counts)
    m = max(counts)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    out = torch.empty((world * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, pad, group=group)
    return torch.cat([out[i * m: i * m + counts[i]] for i in range(world)])


def gather_batch_stats(outs: dict, B: int, combos, reference: Optional[Tuple] = None, group=None,
                       stats_fn: Callable = _cuda_stats):
    """Per-image statistics of every filter's local outputs against the
    `reference` combo's (default: the first), all_gathered over the ranks in
    batch order: {combo: [B, 8] float64}.  This is the only cross-rank traffic
    of the batch path (B x 8 doubles per filter)."""
    world = dist.get_world_size(group)
    counts = [shard_range(B, world, r)[1] - shard_range(B, world, r)[0] for r in range(world)]
    ref = tuple(reference) if reference is not None else tuple(combos[0])
    stats = {}
    ref_norm = None   # column 4 (sum |ref_Lab|) depends on the reference only: computed once
    for c in combos:
        if ref_norm is None or stats_fn is not _cuda_stats:
            s = stats_fn(outs[ref], outs[tuple(c)]).to(torch.float64)
            ref_norm = s[:, 4].clone()
        else:
            s = stats_fn(outs[ref], outs[tuple(c)], ref_norm=False).to(torch.float64)
            s[:, 4] = ref_norm
        stats[tuple(c)] = all_gather_rows(s, counts, group)
    return stats


def run_batch_sharded(imgs_local: torch.Tensor, B: int, window: int, combos, reference: Optional[Tuple] = None,
                      group=None, filter_fn: Callable = _cuda_filter_batch, stats_fn: Callable = _cuda_stats):
    """Filter this rank's shard of a B-image batch with every (criterion,
    variant) in `combos`; gather per-image statistics of each filter against
    the `reference` combo (default: the first) from all ranks.

    imgs_local: [B_local, H, W, 3] = images shard_range(B, world, rank) of the
    batch.  Returns (local outputs {combo: tensor}, gathered stats {combo:
    [B, 8] float64}) -- the stats are the only data that crosses ranks."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(B, world, rank)
    if imgs_local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} expects {hi - lo} images, got {imgs_local.shape[0]}")
    outs = {tuple(c): filter_fn(imgs_local, window, *c) for c in combos}
    return outs, gather_batch_stats(outs, B, combos, reference, group, stats_fn)


# ----------------------------------------------------------------- row stripes
def run_stripes(band: torch.Tensor, H: int, window: int, criterion, variant, group=None,
                filter_fn: Callable = _cuda_filter_rows, gather: bool = True):
    """Filter this rank's stripe of an H-row image from its band (rows
    stripe_bounds(...)[2:] of the image) and, if `gather`, assemble the full
    output on every rank (returned on all ranks; rank 0 is the consumer).
    Returns (stripe, full_or_None)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    out_row0, out_rows, band_row0, band_rows = stripe_bounds(H, world, rank, window)
    if band.shape[0] != band_rows:
        raise ValueError(f"rank {rank}: band must hold rows [{band_row0}, {band_row0 + band_rows})")
    stripe = filter_fn(band, band_row0, H, out_row0, out_rows, window, criterion, variant)
    if not gather:
        return stripe, None
    counts = [stripe_bounds(H, world, r, window)[1] for r in range(world)]
    full = all_gather_rows(stripe, counts, group)
    return stripe, full


def stats_summary(stats: torch.Tensor, H: int, W: int) -> dict:
    """MAE / MSE / PSNR / NCD / fraction of differing pixels from gathered
    [B, 8] stats (vf_image_stats layout), over the whole batch."""
    import math
    s = stats.sum(0).tolist()
    B = stats.shape[0]
    npix = B * H * W
    mse = s[2] / (3 * npix)
    return {"images": B, "diff_frac": s[0] / npix, "mae": s[1] / (3 * npix), "mse": mse,
            "psnr_db": math.inf if mse == 0 else 10 * math.log10(255.0 ** 2 / mse),
            "ncd": s[3] / s[4] if s[4] > 0 else float("nan")}
