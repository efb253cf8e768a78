"""Wait-avoiding group allreduce and blocking global allreduce (drop-in for `wagma.collective`).

Same class and method names, arguments, results and errors as the
reference (`/root/reference/pkg/src/wagma/collective.py`), with the
simulator slot taken by a `DeviceContext`:

- ``GroupAllreduce(ctx, rank, P, S, on_complete, initial_model, mask_rule,
  activation_enabled, staleness_bound, contribution_log)``
- ``install_fresh(vec, iteration)`` / ``join_or_check(version, fresh)``
- ``SyncAllreduce(ctx, rank, P, on_complete).join(iteration, vec)``

Each join is one device launch of the fused kernel (job kind GROUP_SUM /
SYNC_SUM): it installs ``fresh`` in the rank's send ring, takes part in
(or raises) the version's activation, pulls the group's contributions over
NVLink and returns the accumulator. Ranks hosted by the same process join
together inside ``with ctx.batch():`` -- one launch for all of them, the
device analogue of joins that happen at the same simulated instant.

Semantics kept from the reference: exactly-once contribution per (rank,
version); a member contributes its send buffer as of the activation, so a
member that joins after the activation is late (``ALREADY_DONE`` with the
accumulator that already holds its stale contribution; the caller applies
the S+1 rule, optim.py:443-444); version regression and staleness-bound
faults; bit-identical sums on every member (fixed butterfly order).
Deliberate difference: the device does no work on behalf of a rank that
has not joined, so passive completions are not reported through
``on_complete``; the late join returns the finished accumulator instead.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass
from enum import Enum
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .context import DeviceContext, DeviceProtocolFault, Job
from .topology import MASK_RULE_EXAMPLE, InvalidParamsError

__all__ = [
    "ProtocolFault",
    "VersionRegressionError",
    "SendBuffer",
    "JoinStatus",
    "JoinResult",
    "GroupAllreduce",
    "SyncAllreduce",
    "batch",
]


class ProtocolFault(RuntimeError):
    """A message/state inconsistent with the protocol (collective.py:65-66)."""


class VersionRegressionError(ProtocolFault):
    """A process tried to join a version at or below one it already joined (collective.py:69-70)."""


class JoinStatus(Enum):
    ACTIVE = "active"
    ALREADY_DONE = "already_done"


@dataclass
class JoinResult:
    status: JoinStatus
    accumulator: Optional[torch.Tensor] = None


class SendBuffer:
    """View of the model snapshot peers pull (collective.py:84-101).

    ``payload`` is the device send-ring slot of the current stamp;
    ``stamped_iteration`` never decreases.
    """

    def __init__(self, ctx: DeviceContext, rank: int):
        self._ctx = ctx
        self._rank = rank
        self.stamped_iteration = -1

    @property
    def payload(self) -> torch.Tensor:
        view, _ = self._ctx.slot(self._rank, self.stamped_iteration)
        return view

    def install(self, vec, iteration: int) -> None:
        if iteration < self.stamped_iteration:
            raise ProtocolFault(f"send buffer stamp would regress: {self.stamped_iteration} -> {iteration}")
        self._ctx.install(self._rank, iteration, _as_device(self._ctx, vec))
        self.stamped_iteration = iteration


def _as_device(ctx: DeviceContext, vec) -> torch.Tensor:
    t = torch.as_tensor(np.asarray(vec) if not isinstance(vec, torch.Tensor) else vec)
    return t.to(device=ctx.torch_device, dtype=ctx.dtype).contiguous()


def _fault(exc: DeviceProtocolFault) -> ProtocolFault:
    return ProtocolFault(str(exc))


class _Pending:
    def __init__(self, job: Job, resolve: Callable):
        self.job = job
        self.resolve = resolve


def _submit(ctx: DeviceContext, job: Job, resolve: Callable) -> None:
    pend = getattr(ctx, "_wg_batch", None)
    if pend is not None:
        pend.append(_Pending(job, resolve))
        return
    _run(ctx, [_Pending(job, resolve)])


def _run(ctx: DeviceContext, items: list[_Pending]) -> None:
    if not items:
        return
    try:
        ctx.launch([it.job for it in items])
        torch.cuda.current_stream(ctx.torch_device).synchronize()
        ctx.check()
    except DeviceProtocolFault as exc:
        ctx.clear_error()
        raise _fault(exc) from exc
    statuses = ctx.statuses()
    for it, st in zip(items, statuses):
        it.resolve(st)
    _passive_completions(ctx, items, statuses)


def _passive_completions(ctx: DeviceContext, items: list[_Pending], statuses) -> None:
    """Fire the passive completions of this process's endpoints that did not
    join a version a group member just ran (wait-avoiding mode only): the
    group's sum is the launched member's accumulator (every member of a group
    gets the same bits), the stamp is the one the activation locked."""
    eps = getattr(ctx, "_wg_endpoints", None)
    if not eps or not ctx.activation_enabled:
        return
    from .topology import GroupingParams, compute_groups
    launched: dict[int, dict[int, tuple[Job, object]]] = {}
    for it, st in zip(items, statuses):
        if it.job.kind == _lib.WG_JOB_GROUP_SUM and it.job.acc_out is not None:
            launched.setdefault(it.job.version, {})[it.job.rank] = (it.job, st)
    for v, jobs in launched.items():
        waiting = [q for q, ep in eps.items()
                   if q not in jobs and ep.last_joined < v and v not in ep.completed and v not in ep.execution_count]
        if not waiting:
            continue
        stamps, locked = ctx.query_version(v)
        if not locked:
            continue
        part = compute_groups(GroupingParams(ctx.P, ctx.S, v), ctx.mask_rule)
        for q in waiting:
            src = next((jobs[r] for r in part.group_of(q) if r in jobs), None)
            if src is None or stamps[q] >= v:
                continue
            eps[q]._passive_complete(v, src[0].acc_out.clone(), int(stamps[q]), src[1].root)


@contextmanager
def batch(ctx: DeviceContext):
    """Collect the joins of several local ranks into one device launch."""
    if getattr(ctx, "_wg_batch", None) is not None:
        yield
        return
    ctx._wg_batch = []
    try:
        yield
        items = ctx._wg_batch
    finally:
        ctx._wg_batch = None
    _run(ctx, items)


DeviceContext.batch = batch  # type: ignore[attr-defined]


def activation_acts(rank: int, root: int, P: int) -> int:
    """ACT messages `rank` sends in the binomial activation tree rooted at `root`.

    The root sends on every tree edge j < log2 P (collective.py:263-268); rank
    root ^ q receives at hop msb(q) and forwards on the edges above it
    (:270-274). -1 (no activation) sends none.
    """
    if root < 0:
        return 0
    depth = P.bit_length() - 1
    q = rank ^ root
    return depth if q == 0 else depth - q.bit_length()


class GroupAllreduce:
    """Per-process endpoint of the wait-avoiding group allreduce (collective.py:135-345).

    ``on_complete(version, accumulator, timely, contrib_stamp)`` fires when
    a join completes in time (from inside ``join_or_check``, or at the end of
    the enclosing ``ctx.batch()``); a late join returns ``ALREADY_DONE``.
    With ``activation_enabled=False`` every member waits for the whole group
    (blocking group allreduce, collective.py:142-145).
    """

    def __init__(self, ctx: DeviceContext, rank: int, P: int, S: int,
                 on_complete: Callable[[int, torch.Tensor, bool, int], None], initial_model,
                 mask_rule: str = MASK_RULE_EXAMPLE, activation_enabled: bool = True,
                 staleness_bound: Optional[int] = None, contribution_log: Optional[list] = None):
        if P != ctx.P or S != ctx.S:
            raise InvalidParamsError(f"endpoint (P={P}, S={S}) differs from its context (P={ctx.P}, S={ctx.S})")
        if mask_rule != ctx.mask_rule or bool(activation_enabled) != ctx.activation_enabled:
            raise InvalidParamsError("mask_rule / activation_enabled must match the device context")
        if rank not in ctx.local_ranks:
            raise InvalidParamsError(f"rank {rank} is not hosted by this process")
        if (staleness_bound or None) != ctx.staleness_bound:
            # the device enforces the context's bound at activation (collective.py:290-294)
            raise InvalidParamsError(f"staleness_bound={staleness_bound} differs from the context's "
                                     f"{ctx.staleness_bound}")
        self.ctx = ctx
        self.rank = rank
        self.P = P
        self.S = S
        self.on_complete = on_complete
        self.mask_rule = mask_rule
        self.activation_enabled = activation_enabled
        self.staleness_bound = staleness_bound
        self.contribution_log = contribution_log
        self.send_buffer = SendBuffer(ctx, rank)
        ctx.set_initial_model(rank, _as_device(ctx, initial_model))
        self.last_joined = -1
        self.last_completed = -1
        self.completion_tag = -1
        self.execution_count: dict[int, int] = {}
        self.activations_originated = 0
        # message-count equivalents of the reference's simulated transport
        # (collective.py:182-184): ACTs of the binomial activation tree rooted
        # at the activating rank, one PHASE message per butterfly phase
        self.acts_sent = 0
        self.phases_sent = 0
        self._group_phases = S.bit_length() - 1
        # finished versions this rank took part in passively (stale buffer),
        # handed back by its late join (collective.py:208, :341-343)
        self.completed: dict[int, tuple[torch.Tensor, bool, int]] = {}
        eps = getattr(ctx, "_wg_endpoints", None)
        if eps is None:
            eps = ctx._wg_endpoints = {}
        eps[rank] = self

    def install_fresh(self, vec, iteration: int) -> None:
        self.send_buffer.install(vec, iteration)

    def _acts_for(self, root: int) -> int:
        return activation_acts(self.rank, root, self.P)

    def handle_message(self, src: int, body: bytes) -> None:
        """The reference's transport hook (collective.py:226-233). Device memory
        is the transport here: peers never exchange host messages."""
        raise ProtocolFault(f"rank {self.rank}: no host messages on the device transport (from {src})")

    def _executed(self, version: int, stamp: int, root: int, activator: bool) -> None:
        """Bookkeeping of one execution of `version` (collective.py:283-308, 319)."""
        self.execution_count[version] = self.execution_count.get(version, 0) + 1
        if activator:
            self.activations_originated += 1
        self.acts_sent += self._acts_for(root)
        self.phases_sent += self._group_phases
        if self.contribution_log is not None:
            self.contribution_log.append((self.rank, version, stamp))

    def _passive_complete(self, version: int, acc: torch.Tensor, stamp: int, root: int) -> None:
        """Passive participation (collective.py:138-141, 331-345): a group member
        activated `version` while this rank had not joined; its stale send
        buffer (stamp < version) was summed, and the finished accumulator is
        delivered here, not timely, before this rank's own join."""
        self._executed(version, stamp, root, False)
        self.last_completed = max(self.last_completed, version)
        self.completion_tag = version
        self.completed[version] = (acc, False, stamp)
        self.on_complete(version, acc, False, stamp)

    def join_or_check(self, version: int, fresh) -> JoinResult:
        """Join version ``version`` with the fresh local model (collective.py:192-222)."""
        if version <= self.last_joined:
            raise VersionRegressionError(
                f"rank {self.rank}: join for version {version} after joining {self.last_joined}")
        if version < self.send_buffer.stamped_iteration:
            raise ProtocolFault(f"send buffer stamp would regress: {self.send_buffer.stamped_iteration} -> {version}")
        self.last_joined = version
        fresh_t = _as_device(self.ctx, fresh)
        acc = torch.empty_like(fresh_t)
        result = JoinResult(JoinStatus.ACTIVE)
        job = Job(rank=self.rank, kind=_lib.WG_JOB_GROUP_SUM, version=version, fresh=fresh_t, acc_out=acc)

        def resolve(st):
            self.send_buffer.stamped_iteration = version
            self.last_completed = max(self.last_completed, version)
            self.completion_tag = version
            if version in self.completed:
                # it already took part passively (its stale buffer was locked in
                # when a group member activated): the finished accumulator
                # (collective.py:206-208); the device result is bit-identical
                result.status = JoinStatus.ALREADY_DONE
                result.accumulator = self.completed.pop(version)[0]
                return
            self._executed(version, st.contrib_stamp, st.root, st.activator)
            if st.timely:
                self.on_complete(version, acc, True, st.contrib_stamp)
            else:
                result.status = JoinStatus.ALREADY_DONE
                result.accumulator = acc

        _submit(self.ctx, job, resolve)
        return result


class SyncAllreduce:
    """Blocking full-butterfly allreduce over all P processes (collective.py:348-447).

    ``on_complete(iteration, total)`` fires once the bit-identical sum of
    all P contributions is available.
    """

    def __init__(self, ctx: DeviceContext, rank: int, P: int, on_complete: Callable[[int, torch.Tensor], None]):
        if P != ctx.P:
            raise InvalidParamsError(f"endpoint P={P} differs from its context P={ctx.P}")
        if rank not in ctx.local_ranks:
            raise InvalidParamsError(f"rank {rank} is not hosted by this process")
        self.ctx = ctx
        self.rank = rank
        self.P = P
        self.on_complete = on_complete
        self.masks = tuple(1 << j for j in range(P.bit_length() - 1))
        self.last_completed = -1
        self._joined = -1

    def join(self, iteration: int, vec) -> None:
        if self._joined > self.last_completed:
            raise ProtocolFault(f"rank {self.rank}: overlapping sync joins")
        if iteration <= self.last_completed:
            raise ProtocolFault(f"rank {self.rank}: sync for iteration {iteration} after {self.last_completed}")
        self._joined = iteration
        v = _as_device(self.ctx, vec)
        total = torch.empty_like(v)
        job = Job(rank=self.rank, kind=_lib.WG_JOB_SYNC_SUM, version=iteration, fresh=v, acc_out=total)

        def resolve(st):
            self.last_completed = iteration
            self.on_complete(iteration, total)

        _submit(self.ctx, job, resolve)
