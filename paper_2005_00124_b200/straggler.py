"""Deterministic straggler schedule (drop-in for `wagma.netsim.StragglerPolicy`/`DelayModel`).

The reference injects load imbalance by picking victims per iteration with
numpy's PCG64 (`StragglerPolicy.victims`, netsim.py:75-82) and adding a
fixed extra delay (`compute_delay`, netsim.py:103-117). The victim choice is
reproduced with the very same numpy call, so the schedule is bit-identical;
the delay itself becomes a device-side spin on the victim's stream
(`DeviceContext.delay`), so no host sleep sits inside a timed region.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = ["StragglerPolicy", "FixedVictims", "DelayModel", "compute_delay", "BucketedLengthDelay", "WMT_BUCKETS"]


@dataclass(frozen=True)
class StragglerPolicy:
    """Per-iteration delay injection: pick victims, add a fixed extra delay."""

    victims_per_iteration: int
    extra_delay_ms: float
    selection_seed: int = 0

    def victims(self, iteration: int, P: int) -> frozenset[int]:
        if self.victims_per_iteration <= 0:
            return frozenset()
        if self.victims_per_iteration > P:
            raise ValueError("victims_per_iteration exceeds process count")
        rng = np.random.default_rng([self.selection_seed, iteration])
        picks = rng.choice(P, size=self.victims_per_iteration, replace=False)
        return frozenset(int(v) for v in picks)


class FixedVictims(StragglerPolicy):
    """One fixed victim rank every iteration (the reference tests' `_FixedVictims`,
    tests/test_optim.py:193-197): C4's injected straggler."""

    def __init__(self, rank: int, extra_delay_ms: float):
        super().__init__(1, extra_delay_ms, 0)
        object.__setattr__(self, "rank", int(rank))

    def victims(self, iteration: int, P: int) -> frozenset[int]:
        if not 0 <= self.rank < P:
            raise ValueError(f"victim rank {self.rank} outside 0..{P - 1}")
        return frozenset({self.rank})


@dataclass(frozen=True)
class DelayModel:
    """Compute timing of one run (netsim.py:85-100); delays in ms, >= 0."""

    base_compute_ms: float = 1.0
    jitter_max_ms: float = 0.0
    link_latency_ms: float = 1.0
    straggler: Optional[StragglerPolicy] = None

    def __post_init__(self) -> None:
        if min(self.base_compute_ms, self.jitter_max_ms, self.link_latency_ms) < 0:
            raise ValueError("delays must be non-negative")


def compute_delay(proc: int, iteration: int, model: DelayModel, rng_seed: int, P: int) -> float:
    """base + uniform jitter + extra if victim (netsim.py:103-117), in ms."""
    if not 0 <= proc < P:
        raise ValueError(f"rank {proc} out of range for P={P}")
    delay = model.base_compute_ms
    if model.jitter_max_ms > 0:
        rng = np.random.default_rng([rng_seed, iteration, proc])
        delay += float(rng.uniform(0.0, model.jitter_max_ms))
    if model.straggler is not None and proc in model.straggler.victims(iteration, P):
        delay += model.straggler.extra_delay_ms
    return delay


# (sequence length, share of batches) -- a WMT-style length-bucketed batching
# profile: most batches are short, a long tail of long ones.
WMT_BUCKETS = ((16, 0.18), (24, 0.20), (32, 0.19), (48, 0.16), (64, 0.12), (96, 0.08), (128, 0.05),
               (192, 0.015), (256, 0.005))


@dataclass(frozen=True)
class BucketedLengthDelay:
    """Per-(rank, iteration) compute time from a bucketed sequence-length draw.

    The imbalance of the Transformer experiment (arXiv 2005.00124 §6.2,
    PAPER.md:795): every rank's batch holds sentences of one length bucket,
    so its step time scales with the bucket's length. The reference only has
    uniform jitter plus victims (netsim.py:85-117); this is the new delay
    model SURVEY.md §8(d) asks for C3. Deterministic in (seed, iteration,
    rank) through numpy's PCG64, like `compute_delay`'s jitter.
    """

    base_ms: float
    buckets: tuple = WMT_BUCKETS
    seed: int = 0

    def mean_length(self) -> float:
        tot = sum(p for _, p in self.buckets)
        return sum(L * p for L, p in self.buckets) / tot

    def delay_ms(self, rank: int, iteration: int) -> float:
        rng = np.random.default_rng([self.seed, iteration, rank])
        lengths = np.array([L for L, _ in self.buckets], dtype=np.float64)
        probs = np.array([p for _, p in self.buckets], dtype=np.float64)
        L = float(rng.choice(lengths, p=probs / probs.sum()))
        return self.base_ms * L / self.mean_length()
