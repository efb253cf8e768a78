"""Host-side multi-process plumbing (torch.distributed): rank layout, IPC blob
exchange, max-over-ranks timing. Kept free of CUDA so it is testable with the
gloo backend on CPU (tests/test_dist_gloo.py).
"""

from __future__ import annotations

from typing import Optional

import torch

__all__ = ["rank_layout", "gpu_of_rank", "exchange_blobs", "max_over_ranks"]


def rank_layout(P: int, n_gpus: int, gpu_index: int) -> range:
    """WAGMA ranks hosted by GPU `gpu_index`: block mapping r -> r // (P / n_gpus)."""
    if n_gpus < 1 or P % n_gpus:
        raise ValueError(f"n_gpus={n_gpus} must divide P={P}")
    if not 0 <= gpu_index < n_gpus:
        raise ValueError(f"gpu_index={gpu_index} out of range")
    R = P // n_gpus
    return range(gpu_index * R, (gpu_index + 1) * R)


def gpu_of_rank(rank: int, P: int, n_gpus: int) -> int:
    return rank // (P // n_gpus)


def exchange_blobs(gpu_index: int, blob: bytes, group=None) -> dict[int, bytes]:
    """All-gather every process's (gpu_index, IPC blob); returns {gpu_index: blob}."""
    import torch.distributed as dist
    out: list = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, (gpu_index, blob), group=group)
    blobs = {int(g): b for g, b in out}
    if len(blobs) != len(out):
        raise RuntimeError("two processes claimed the same gpu_index")
    return blobs


def max_over_ranks(x: float, group=None, device: Optional[torch.device] = None) -> float:
    """Max of a scalar over all ranks (device timings are reported as the max)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
