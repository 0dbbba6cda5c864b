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
