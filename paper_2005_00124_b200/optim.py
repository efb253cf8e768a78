"""Group model averaging SGD on the device (drop-in for the hot path of `wagma.optim`).

Keeps the reference's configuration surface -- `EtaSchedule`,
`OptimizerConfig` (with the same validation and errors), `is_sync_iteration`,
`ConfigError`, `DivergenceError` -- and replaces the per-worker Alg. 2 loop
(`_GroupAveragingWorker`, optim.py:371-452) by `GroupAveragingOptimizer`,
whose `step()` issues ONE fused device launch per iteration for all ranks a
process hosts: local SGD/momentum update, send-buffer install, group (or
global) allreduce and the averaging rule, touching each weight once.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass, field
from typing import Mapping, Optional

import numpy as np
import torch

from . import _lib
from .context import DeviceContext, DivergenceError, Job, JobStatus
from .topology import GroupingParams, InvalidParamsError

__all__ = [
    "EtaSchedule",
    "OptimizerConfig",
    "ConfigError",
    "DivergenceError",
    "is_sync_iteration",
    "GroupAveragingOptimizer",
]


class ConfigError(ValueError):
    """Invalid run configuration (optim.py:77-78)."""


@dataclass(frozen=True)
class EtaSchedule:
    """Learning-rate schedule: constant, step decay, or P/sqrt(T) (optim.py:85-103)."""

    kind: str = "constant"
    value: float = 0.1
    decay_factor: float = 0.5
    decay_every: int = 0

    def rate(self, t: int, P: int, T: int) -> float:
        if self.kind == "constant":
            return self.value
        if self.kind == "step":
            if self.decay_every <= 0:
                raise ConfigError("step schedule needs decay_every >= 1")
            return self.value * self.decay_factor ** (t // self.decay_every)
        if self.kind == "theorem":
            return float(P / np.sqrt(T))
        raise ConfigError(f"unknown eta schedule kind {self.kind!r}")


@dataclass
class OptimizerConfig:
    """The four averaging parameters plus local-update settings (optim.py:106-148).

    ``tau=None`` means no global synchronization. ``alpha`` selects the
    wait-avoiding group allreduce, ``beta`` the blocking one; both off
    degrades to local SGD with period tau.
    """

    T: int
    S: int = 1
    tau: Optional[int] = None
    alpha: bool = True
    beta: bool = False
    eta: EtaSchedule = field(default_factory=EtaSchedule)
    b: int = 1
    update_rule: str = "sgd"
    momentum: float = 0.9

    def validate(self, P: int) -> None:
        if self.alpha and self.beta:
            raise ConfigError("alpha and beta can not both be set")
        if self.T < 1:
            raise ConfigError("T must be >= 1")
        if self.tau is not None and self.tau < 1:
            raise ConfigError("tau must be >= 1 or None")
        if self.b < 1:
            raise ConfigError("batch size must be >= 1")
        if self.update_rule not in ("sgd", "momentum"):
            raise ConfigError(f"unknown update rule {self.update_rule!r}")
        try:
            GroupingParams(P, self.S, 0)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc
        if self.eta.kind == "constant" and self.eta.value <= 0:
            raise ConfigError("eta must be positive")
        if self.eta.kind == "theorem" and self.tau is not None:
            horizon = P ** 4 * self.tau ** 4
            if self.T < horizon:
                warnings.warn(f"theorem schedule expects T >= P^4 tau^4 = {horizon}, got T={self.T}",
                              stacklevel=2)


def is_sync_iteration(t: int, tau: Optional[int]) -> bool:
    """(optim.py:151-152)"""
    return tau is not None and (t + 1) % tau == 0


class GroupAveragingOptimizer:
    """Alg. 2 for the ranks of one `DeviceContext`, one fused launch per step.

    Owns the replicas W_r (initialised to ``w0`` on every rank, optim.py:328)
    and the local momentum buffers m_r (never averaged, optim.py:165/179).
    ``step(t, grads)`` enqueues iteration t for the given ranks on the
    current stream: sync iterations run the blocking global average
    (optim.py:406-411, 449-452), other iterations the wait-avoiding (alpha)
    or blocking (beta) group average (optim.py:412-447), or a plain local
    step when both flags are off (optim.py:427-428).
    """

    def __init__(self, ctx: DeviceContext, cfg: OptimizerConfig, w0: torch.Tensor, *, T: Optional[int] = None):
        cfg.validate(ctx.P)
        if cfg.S != ctx.S:
            raise ConfigError(f"config S={cfg.S} differs from the context's S={ctx.S}")
        self.use_group = cfg.alpha or cfg.beta
        if self.use_group and bool(cfg.alpha) != ctx.activation_enabled:
            raise ConfigError("alpha/beta must match the context's activation_enabled")
        if cfg.tau != ctx.tau:
            raise ConfigError(f"config tau={cfg.tau} differs from the context's tau={ctx.tau}")
        if self.use_group and cfg.tau is not None and (ctx.staleness_bound is None or ctx.staleness_bound > cfg.tau):
            # every endpoint uses staleness_bound=opt.tau (optim.py:386); a
            # tighter bound is allowed (fault-injection tests), a looser one
            # would average over-stale replicas silently
            raise ConfigError(f"context staleness_bound={ctx.staleness_bound} is looser than tau={cfg.tau}")
        self.ctx = ctx
        self.cfg = cfg
        self.T = cfg.T if T is None else T
        # contribution stamps forced on replayed versions (the metrics
        # recorder's staleness source when no descriptor was locked)
        self.forced_log: dict[int, list[int]] = {}
        self.momentum = cfg.update_rule == "momentum"
        w0 = w0.to(device=ctx.torch_device, dtype=ctx.dtype).contiguous()
        self.W: dict[int, torch.Tensor] = {}
        self.m: dict[int, Optional[torch.Tensor]] = {}
        for r in ctx.local_ranks:
            self.W[r] = w0.clone()
            self.m[r] = torch.zeros_like(w0) if self.momentum else None
            ctx.set_initial_model(r, w0)
        # host fast path (step): the replicas are owned here, their pointers fixed
        self._arr = None
        self._slot: list = []
        self._wptr = {r: w.data_ptr() for r, w in self.W.items()}
        self._mptr = {r: (mm.data_ptr() if mm is not None else None) for r, mm in self.m.items()}

    def kind(self, t: int) -> int:
        if is_sync_iteration(t, self.cfg.tau):
            return _lib.WG_JOB_SYNC_STEP
        return _lib.WG_JOB_STEP if self.use_group else _lib.WG_JOB_LOCAL_STEP

    def jobs(self, versions: Mapping[int, int], grads: Mapping[int, torch.Tensor]) -> list[Job]:
        """Jobs for {rank: iteration} with gradients {rank: g}."""
        out = []
        for r, t in versions.items():
            out.append(Job(rank=r, kind=self.kind(t), version=t, W=self.W[r], m=self.m[r], g=grads[r],
                           eta=self.cfg.eta.rate(t, self.ctx.P, self.T), beta=self.cfg.momentum,
                           momentum=self.momentum))
        return out

    def step(self, t: int, grads: Mapping[int, torch.Tensor], *, forced_stamps: Optional[list[int]] = None,
             stream=None) -> None:
        """Iteration t for every rank in ``grads`` (all local ranks normally).

        Raises DivergenceError (optim.py:174-175) if an earlier launch
        produced a non-finite W'; the check reads the host-mapped error word,
        so it costs no synchronisation and lags the device by the launches in
        flight (``ctx.check()`` after a synchronise is exact).
        """
        self.ctx.check_async()
        forced = {t: forced_stamps} if forced_stamps is not None else None
        if forced:
            self.forced_log.update(forced)
        if not self._fast_step(t, grads, forced, stream):
            self.ctx.launch(self.jobs({r: t for r in grads}, grads), forced=forced, stream=stream)

    def _fast_step(self, t: int, grads: Mapping[int, torch.Tensor], forced, stream) -> bool:
        """Host fast path of step(): a persistent job array (the optimizer's own
        W / m, validated once) in which only the gradient pointer, version,
        kind and step size change; each gradient is still checked (device,
        dtype, size, contiguity, 16-byte alignment). Returns False (general
        path) for a gradient that needs realigning."""
        ctx = self.ctx
        arr = self._arr
        if arr is None or len(grads) > len(arr):
            arr = self._arr = (_lib.WgJob * max(len(ctx.local_ranks), len(grads)))()
            self._slot = [None] * len(arr)  # (rank, W ptr, m ptr) whose fixed fields a slot holds
        kind = self.kind(t)
        eta = float(self.cfg.eta.rate(t, ctx.P, self.T))
        rule = _lib.WG_UPDATE_MOMENTUM if self.momentum else _lib.WG_UPDATE_SGD
        dev, dt, n = ctx.torch_device, ctx.dtype, ctx.n
        i = 0
        for r, g in grads.items():
            if r not in self.W:
                raise InvalidParamsError(f"rank {r} is not hosted by this process")
            gp = g.data_ptr()
            if gp % 16:
                return False
            if g.device != dev or g.dtype != dt or g.numel() != n or not g.is_contiguous():
                ctx._check_vec(g, "g")  # raises with the message
            wp = self.W[r].data_ptr()
            if wp != self._wptr.get(r):  # a replica replaced by the caller: validate it once
                ctx._check_vec(self.W[r], "W")
                self._wptr[r] = wp
            mm = self.m[r]
            mp = mm.data_ptr() if mm is not None else None
            if mp != self._mptr.get(r):
                ctx._check_vec(mm, "m")
                self._mptr[r] = mp
            a = arr[i]
            key = (r, wp, mp)
            if self._slot[i] != key:
                a.rank, a.update_rule, a.beta = r, rule, float(self.cfg.momentum)
                a.W, a.m = wp, mp
                a.fresh = a.acc_out = None
                self._slot[i] = key
            a.kind, a.version, a.eta, a.g = kind, t, eta, gp
            i += 1
        ctx.launch_array(arr, i, forced, stream)
        return True

    def step_mixed(self, versions: Mapping[int, int], grads: Mapping[int, torch.Tensor],
                   forced: Optional[dict[int, list[int]]] = None, stream=None) -> None:
        """One launch in which ranks may be at different iterations (stragglers)."""
        self.ctx.check_async()
        if forced:
            self.forced_log.update(forced)
        self.ctx.launch(self.jobs(versions, grads), forced=forced, stream=stream)

    def statuses(self) -> list[JobStatus]:
        return self.ctx.statuses()
