"""Multi-rank drivers of the fused device path.

- `replay`: drives Alg. 2 (optim.py:403-452) for every rank of a context
  with the contribution stamps of a recorded run forced per version -- the
  reference's `contribution_log` -- so a device trajectory can be compared
  with the reference's `run_training` bit for bit.
- `TickSchedule`: deterministic emulation of stragglers for ranks that share
  one GPU. Ranks sharing a GPU must run in one launch (a kernel may not spin
  on a kernel that is not running), so time advances in launch ticks: a
  victim of iteration t (`StragglerPolicy.victims`, netsim.py:75-82) sits
  out `delay_ticks` ticks before it can join t, everyone else proceeds, and
  the global sync waits for all ranks (optim.py:406-411). The device's live
  activation protocol then decides who was timely; the descriptors it locked
  are the device's contribution log.
- `contribution_log`: reads those descriptors back.
"""

from __future__ import annotations

from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _lib
from .optim import GroupAveragingOptimizer, is_sync_iteration

__all__ = ["replay", "TickSchedule", "contribution_log"]

GradFn = Callable[[int, int], torch.Tensor]  # (rank, t) -> gradient on device


def replay(opt: GroupAveragingOptimizer, grad_fn: GradFn, T: int, *,
           stamps: Optional[np.ndarray] = None, etas: Optional[np.ndarray] = None,
           check_every: int = 0, on_step: Optional[Callable[[int], None]] = None) -> None:
    """Run iterations 0..T-1 for all local ranks, one launch per iteration.

    stamps[t, r] (optional) forces the contribution stamps of group version t
    (alpha mode); etas[t, r] overrides the schedule's step size; on_step(t)
    runs after iteration t is enqueued (e.g. `MetricsRecorder.record`).
    """
    ctx = opt.ctx
    ranks = list(ctx.local_ranks)
    for t in range(T):
        grads = {r: grad_fn(r, t) for r in ranks}
        jobs = opt.jobs({r: t for r in ranks}, grads)
        if etas is not None:
            for j in jobs:
                j.eta = float(etas[t, j.rank])
        forced = None
        if stamps is not None and opt.kind(t) == _lib.WG_JOB_STEP and opt.cfg.alpha:
            forced = {t: [int(s) for s in stamps[t]]}
            opt.forced_log.update(forced)
        ctx.launch(jobs, forced=forced)
        if on_step is not None:
            on_step(t)
        if check_every and (t + 1) % check_every == 0:
            torch.cuda.current_stream(ctx.torch_device).synchronize()
            ctx.check()


class TickSchedule:
    """Launch-tick emulation of stragglers on one GPU (see module docstring)."""

    def __init__(self, P: int, T: int, tau: Optional[int], victims: Callable[[int], frozenset],
                 delay_ticks: int = 1):
        self.P, self.T, self.tau = P, T, tau
        self.victims = victims
        self.delay_ticks = delay_ticks

    def ticks(self):
        """Yield {rank: iteration} per launch until every rank finished T iterations."""
        it = [0] * self.P
        waited = [0] * self.P
        while any(t < self.T for t in it):
            ready = {}
            for r in range(self.P):
                t = it[r]
                if t >= self.T:
                    continue
                need = self.delay_ticks if r in self.victims(t) else 0
                if waited[r] < need:
                    waited[r] += 1
                    continue
                ready[r] = t
            at_sync = {r: t for r, t in ready.items() if is_sync_iteration(t, self.tau)}
            if at_sync:
                ts = set(at_sync.values())
                if len(at_sync) < self.P or len(ts) != 1:
                    for r in at_sync:  # wait at the global barrier
                        del ready[r]
            if ready:
                yield dict(ready)
                for r in ready:
                    it[r] += 1
                    waited[r] = 0

    def run(self, opt: GroupAveragingOptimizer, grad_fn: GradFn) -> list[dict[int, int]]:
        history = []
        for versions in self.ticks():
            grads = {r: grad_fn(r, t) for r, t in versions.items()}
            opt.step_mixed(versions, grads)
            history.append(versions)
        return history


def contribution_log(ctx, T: int, tau: Optional[int]) -> np.ndarray:
    """Locked contribution stamps [T, P] of every group version (-2: none)."""
    out = np.full((T, ctx.P), -2, dtype=np.int64)
    for v in range(T):
        if is_sync_iteration(v, tau):
            continue
        stamps, locked = ctx.query_version(v)
        if locked:
            out[v] = stamps
    return out


def synthetic_grad(rank: int, t: int, n: int, dtype=torch.float32, device="cuda", scale: float = 0.01,
                   seed: int = 1234) -> torch.Tensor:
    """g_t ~ N(0, scale^2) per (rank, t), seeded [seed, rank, t]."""
    gen = torch.Generator(device=device)
    gen.manual_seed((seed * 1_000_003 + rank) * 1_000_003 + t)
    return torch.randn(n, generator=gen, device=device, dtype=dtype) * scale
