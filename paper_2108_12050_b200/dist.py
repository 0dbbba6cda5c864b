"""Multi-GPU plumbing for the MHFD hot path.

Images are independent, so a batch is sharded contiguously across ranks (one process per
GPU) and the only collective is the all-gather of every image's (count, score) — 12
bytes per image — over NCCL (gloo in the CPU tests).  No image data crosses GPUs.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [start, end) of image indices owned by `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or global_batch < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def gather_results(counts: torch.Tensor, scores: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather per-image (count, score) from every rank -> (world, n_local, 2) float64.

    Every rank must hold the same number of local images (the bench's weak-scaling
    batches); counts are exact integers below 2^53, so float64 carries them losslessly."""
    local = torch.stack([counts.to(torch.float64), scores.to(torch.float64)], 1).contiguous()
    world = dist.get_world_size()
    if out is None:
        out = torch.empty((world * local.shape[0], 2), dtype=torch.float64, device=local.device)
    dist.all_gather_into_tensor(out, local)   # rank r's block at rows [r*n, (r+1)*n)
    return out.view(world, local.shape[0], 2)


# ------------------------------------------------------------------ single-image sharding
# SURVEY.md §8(f) f2 (the paper's own multi-GPU goal, without its
# gather of whole L planes): one image split into row bands, one per rank.  Every rank
# holds the image (broadcast, 1 B/px), computes the candidates of its band
# (mhfd_detect_band: its blur windows and NMS neighbours are evaluated locally, the
# percentiles are the whole image's), the bands' lists are all-gathered in rank order
# (= raster order of the whole image), and every rank prunes the full list.

def band_rows(height: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row band [y0, y1) of `rank` (heights differ by <= 1)."""
    return shard(height, world, rank)


def gather_candidates(cands: torch.Tensor, n: int | torch.Tensor) -> tuple[torch.Tensor, int]:
    """All-gather every rank's candidate records (rows of `cands`) in rank order ->
    (concatenated records, exact total).  Two collectives: every rank's (count, capacity),
    then the records padded to the largest stored count.  A rank stores at most
    cands.shape[0] records (mhfd_detect_band truncates its list but reports the exact
    count), so every rank clamps each rank's record count the same way from the gathered
    (count, capacity) pairs before the second collective (no rank waits on a shape only
    it knows): the
    concatenation is then the first records of the whole image's raster list, and the
    returned total stays exact (callers compare it with the pruning capacity)."""
    world = dist.get_world_size()
    dev = cands.device
    n_t = (n.reshape(1) if isinstance(n, torch.Tensor) else torch.tensor([int(n)])).to(dev, torch.int64)
    mine = torch.cat([n_t.reshape(1), torch.tensor([cands.shape[0]], dtype=torch.int64, device=dev)])
    meta = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(meta, mine)   # (count, stored capacity) of every rank
    meta_h = [int(c) for c in meta.cpu().tolist()]
    counts_h = meta_h[0::2]
    stored = [min(c, cap) for c, cap in zip(counts_h, meta_h[1::2])]   # identical on every rank
    m = max(max(stored), 1)
    rec = cands.shape[1]
    local = torch.zeros((m, rec), dtype=cands.dtype, device=dev)
    k = stored[dist.get_rank()]
    local[:k] = cands[:k]
    allc = torch.empty((world * m, rec), dtype=cands.dtype, device=dev)
    dist.all_gather_into_tensor(allc, local)
    parts = [allc[r * m: r * m + stored[r]] for r in range(world)]
    return torch.cat(parts, 0), sum(counts_h)


def focus_score_single_image(det, image: torch.Tensor, src: int = 0):
    """Score ONE image on all ranks (each rank a row band; NCCL broadcast + all-gathers).
    `image` is the (H, W) tile on this rank's device (its content matters on `src`
    only).  Returns (blobs, count, score, flags) of mhfd_prune_candidates, identical on
    every rank and bit-identical to det.detect / det.focus_score on the whole image,
    including candidate overflow: when the image has more than det.max_candidates
    candidates, the first max_candidates in raster order are pruned and flags bit 0 is
    set, as mhfd_detect_batch does."""
    dist.broadcast(image, src)
    y0, y1 = band_rows(det.height, dist.get_world_size(), dist.get_rank())
    cands, n = det.detect_band(image, y0, y1)
    allc, total = gather_candidates(cands, n)
    cap = det.max_candidates
    over = total > cap
    blobs, cnt, score, flags = det.prune_candidates(allc[:cap] if over else allc, min(total, cap))
    if over:
        flags |= 1
    return blobs, cnt, score, flags


def halo_rows(det, rounds: int = 5) -> int:
    """Rows a band is extended by for the sharded pruning: a blob decided in synchronous
    round t depends on the candidates within (t + 1) D (mhfd_prune_band), so a halo of
    (rounds + 1) D certifies every band blob decided by round `rounds`.  5 rounds certified
    all 8 bands of sharp and defocused C3 and C5 tiles (3 suffice for C3;
    tools/halo_sweep.py)."""
    return (rounds + 1) * det.interaction_radius()


def focus_score_single_image_sharded(det, image: torch.Tensor, src: int = 0, halo: int | None = None):
    """Score ONE image on all ranks with the pruning sharded too (each
    rank prunes its own band from the candidates of the band plus `halo` rows on each
    side, mhfd_prune_band; one all-reduce of (kept, certificate failures, band
    candidates) replaces the all-gather of the candidate list and the replicated
    pruning).  Falls back to focus_score_single_image's gather + replicated pruning when
    some band's certificate fails or the image has more candidates than max_candidates
    (whose truncation rule needs the whole list).  Returns (count, score, sharded) with
    count and score identical on every rank and equal to det.focus_score on the whole
    image; `sharded` says which path produced them."""
    dist.broadcast(image, src)
    world, rank = dist.get_world_size(), dist.get_rank()
    H, cap = det.height, det.max_candidates
    y0, y1 = band_rows(H, world, rank)
    h = halo_rows(det) if halo is None else int(halo)
    e0, e1 = max(0, y0 - h), min(H, y1 + h)
    cands, n = det.detect_band(image, e0, e1)
    n_ext = int(n.item())
    if n_ext <= cap:
        kept, cert, nband = det.prune_band(cands, n_ext, e0, e1, y0, y1)
        red = torch.stack([kept[0].to(torch.int64), 1 - cert[0].to(torch.int64), nband[0].to(torch.int64)])
    else:   # the extended band alone overflows the pruning capacity: not certifiable
        red = torch.tensor([0, 1, cap + 1], dtype=torch.int64, device=cands.device)
    dist.all_reduce(red)   # SUM: kept blobs, failed certificates, candidates
    kept_all, fails, total = (int(v) for v in red.cpu().tolist())
    if fails == 0 and total <= cap:
        return kept_all, float(kept_all), True
    _, cnt, score, _ = focus_score_single_image(det, image, src)
    return int(cnt.item()), float(score.item()), False
