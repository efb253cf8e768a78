"""Replica diagnostics on the device (drop-in for the replica part of `wagma.optim.compute_diagnostics`).

The reference's `compute_diagnostics` (optim.py:199-210) reports the replica
mean mu_t and the spread potential Gamma_t = sum_r ||W_r - mu_t||^2, and its
recorder asserts that replicas are bit-identical after every global sync
(optim.py:289-293). Here the sums run in fp64 on the device
(`wg_replicas_sum` / `wg_replicas_spread`); across processes the replica sum
vector and the spread are all-reduced with torch.distributed. The problem
terms (loss and gradient norm at mu) belong to the synthetic problems, which
are out of scope.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Mapping, Optional

import torch

from .context import DeviceContext

__all__ = ["ReplicaDiagnostics", "replica_diagnostics", "gamma_bound", "check_after_sync"]


@dataclass
class ReplicaDiagnostics:
    mu: torch.Tensor          # fp64 replica mean over all P ranks
    gamma: float              # sum_r ||W_r - mu||^2 over all P ranks
    identical: bool           # every replica bit-identical (the reference's np.array_equal check)


def replica_diagnostics(ctx: DeviceContext, replicas: Mapping[int, torch.Tensor],
                        process_group=None) -> ReplicaDiagnostics:
    ranks = sorted(replicas)
    if sorted(ranks) != list(ctx.local_ranks):
        raise ValueError("pass the replicas of every rank this process hosts")
    for r in ranks:
        ctx._check_vec(replicas[r], f"W[{r}]")
    ptrs = (ctypes.c_void_p * len(ranks))(*[replicas[r].data_ptr() for r in ranks])
    stream = ctx.stream_handle()
    total = torch.zeros(ctx.n, dtype=torch.float64, device=ctx.torch_device)
    ctx._raise(ctx.lib.wg_replicas_sum(ctx._h, ptrs, len(ranks), total.data_ptr(), stream), "wg_replicas_sum")
    import torch.distributed as dist
    multi = ctx.n_gpus > 1 and dist.is_available() and dist.is_initialized()
    if multi:
        dist.all_reduce(total, group=process_group)
    mu = total / ctx.P
    out = torch.zeros(2, dtype=torch.float64, device=ctx.torch_device)
    ctx._raise(ctx.lib.wg_replicas_spread(ctx._h, ptrs, len(ranks), mu.data_ptr(), out.data_ptr(), stream),
               "wg_replicas_spread")
    # bit identity (optim.py:289-291): out[1] = max |W_r - W_first| over the
    # local replicas (exact); across GPUs the first local replicas must also
    # agree bit for bit -- compared through two integer checksums of their bits
    first = replicas[ranks[0]]
    bits = first.view(torch.int32 if first.dtype == torch.float32 else torch.int64).to(torch.int64)
    ident = torch.stack([out[1], (bits.sum() & 0xFFFFFFFFFFFF).to(torch.float64),
                         (((bits * 0x9E3779B1) % 1000000007).sum() & 0xFFFFFFFFFFFF).to(torch.float64)])
    if multi:
        dist.all_reduce(out[:1], group=process_group)
        lo, hi = ident.clone(), ident.clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=process_group)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=process_group)
        identical = bool(hi[0].item() == 0.0 and torch.equal(lo[1:], hi[1:]))
    else:
        identical = bool(ident[0].item() == 0.0)
    gamma = float(out[0].item())
    return ReplicaDiagnostics(mu=mu, gamma=gamma, identical=identical)


def gamma_bound(P: int, eta: float, M_hat: float, tau: int) -> float:
    """Replica-spread bound 16 P eta^2 M^2 tau^2 the potential is checked against (optim.py:213-215)."""
    return 16.0 * P * eta ** 2 * M_hat ** 2 * tau ** 2


def check_after_sync(diag: ReplicaDiagnostics, t: int) -> None:
    """The recorder's post-sync rule (optim.py:289-293): after a global sync the
    spread must vanish (relative to |mu|^2), else ProtocolFault."""
    from .collective import ProtocolFault

    mu_sq = float(torch.dot(diag.mu, diag.mu).item())
    if diag.gamma > 1e-12 * max(1.0, mu_sq):
        raise ProtocolFault(f"replica spread {diag.gamma} nonzero after sync at t={t}")
