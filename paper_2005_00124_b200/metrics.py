"""Per-iteration metrics rows and run manifest (drop-in for the reference's recorder output).

The reference's `_Recorder` (optim.py:253-307) emits one `MetricsRecord`
(optim.py:218-234) per iteration once every worker finished it: the replica
mean's loss and squared gradient norm, the spread potential Gamma_t, the
largest contribution age of that iteration's group version (its
`note_contribution`, optim.py:271-276), and the simulator's clock and
message/byte counters. `harness/runner.py:44-91` writes the rows as
`metrics.csv` (header `CSV_HEADER`, optim.py:74) plus a `manifest.json`.

Here the same rows come from the device:

- `gamma` and mu from `diagnostics.replica_diagnostics` (fp64 device sums,
  all-reduced across GPUs); `loss_mu` / `grad_norm_sq_mu` from optional
  callbacks on mu (the problem is the caller's -- the synthetic problems are
  out of scope); a non-finite loss raises `DivergenceError` and a nonzero
  spread after a global sync raises `ProtocolFault`, as the reference's
  `_emit` does (optim.py:286-293).
- `max_staleness` from the contribution stamps the activation protocol
  locked on the device for that version (`wg_query_version`), or the forced
  stamps of a replayed run; 0 at global syncs (no group version).
- `sim_time_ms` is device time (CUDA events) since the recorder started;
  `msgs_total` counts the messages the reference's transport would have
  carried for the same schedule (one PHASE message per rank per butterfly
  phase; the activation tree's P - 1 ACTs per live group version), and
  `bytes_total` the bytes this path actually moved between GPUs (NVLink
  ingress of every GPU, from the schedule). These three columns are
  transport-specific by construction; the other five match the reference's
  rows for the same trajectory (tests/test_gpu_metrics.py).
"""

from __future__ import annotations

import hashlib
import json
import math
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Optional

import numpy as np
import torch

from . import __version__
from .context import DivergenceError
from .diagnostics import check_after_sync, replica_diagnostics
from .optim import GroupAveragingOptimizer, is_sync_iteration
from .topology import GroupingParams, compute_groups, tree_leaves

__all__ = ["CSV_HEADER", "MetricsRecord", "MetricsRecorder", "metrics_csv_text", "write_run"]

CSV_HEADER = "iteration,sim_time_ms,loss_mu,grad_norm_sq_mu,gamma,max_staleness,msgs_total,bytes_total"


@dataclass(frozen=True)
class MetricsRecord:
    """One row (optim.py:218-234); same fields, same CSV formatting."""

    iteration: int
    sim_time_ms: float
    loss_mu: float
    grad_norm_sq_mu: float
    gamma: float
    max_staleness: int
    msgs_total: int
    bytes_total: int

    def csv_row(self) -> str:
        return (
            f"{self.iteration},{self.sim_time_ms!r},{self.loss_mu!r},"
            f"{self.grad_norm_sq_mu!r},{self.gamma!r},{self.max_staleness},"
            f"{self.msgs_total},{self.bytes_total}"
        )


def metrics_csv_text(records) -> str:
    """`harness/runner.py:metrics_csv_text` for a list of records."""
    lines = [CSV_HEADER]
    lines.extend(rec.csv_row() for rec in records)
    return "\n".join(lines) + "\n"


def _nvlink_bytes(P: int, S: int, R: int, t: int, tau: Optional[int], elem_bytes: int) -> int:
    """NVLink ingress summed over all GPUs for iteration t (pull of remote leaves)."""
    if R >= P:
        return 0
    if is_sync_iteration(t, tau):
        leaves_of = {0: list(range(P))}
        members = {r: 0 for r in range(P)}
    else:
        part = compute_groups(GroupingParams(P, S, t))
        leaves_of, members = {}, {}
        for gi, grp in enumerate(part.groups):
            leaves_of[gi] = list(tree_leaves(GroupingParams(P, S, t), grp[0]))
            for r in grp:
                members[r] = gi
    total = 0
    for g in range(P // R):
        plans = {members[r] for r in range(g * R, (g + 1) * R)}
        for pl in plans:
            total += sum(1 for q in leaves_of[pl] if q // R != g)
    return total * elem_bytes


class MetricsRecorder:
    """Collects one `MetricsRecord` per iteration from a `GroupAveragingOptimizer`.

    Call `record(t)` after `step(t)` on every process (it synchronises and,
    across GPUs, all-reduces). ``loss_fn(mu) -> float`` and
    ``grad_fn(mu) -> array`` receive the fp64 replica mean as a numpy array.
    """

    def __init__(self, opt: GroupAveragingOptimizer, *, loss_fn: Optional[Callable] = None,
                 grad_fn: Optional[Callable] = None, process_group=None):
        self.opt = opt
        self.ctx = opt.ctx
        self.loss_fn = loss_fn
        self.grad_fn = grad_fn
        self.process_group = process_group
        self.records: list[MetricsRecord] = []
        self.max_gamma = 0.0
        self.max_staleness = 0
        self.sync_replica_checks: list[tuple[int, bool]] = []
        self._msgs = 0
        self._bytes = 0
        self._t0 = torch.cuda.Event(enable_timing=True)
        self._t0.record(torch.cuda.current_stream(self.ctx.torch_device))

    def _stamps(self, t: int) -> Optional[list[int]]:
        forced = self.opt.forced_log.get(t)
        if forced is not None:
            return list(forced)
        stamps, locked = self.ctx.query_version(t)
        return stamps if locked else None

    def record(self, t: int) -> MetricsRecord:
        ctx, opt = self.ctx, self.opt
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(torch.cuda.current_stream(ctx.torch_device))
        ev.synchronize()
        ctx.check()
        diag = replica_diagnostics(ctx, opt.W, process_group=self.process_group)
        sync = is_sync_iteration(t, opt.cfg.tau)
        mu = diag.mu.cpu().numpy()
        loss = float(self.loss_fn(mu)) if self.loss_fn else math.nan
        if self.loss_fn and not math.isfinite(loss):
            raise DivergenceError(f"non-finite loss at iteration {t}")
        if self.grad_fn:
            gr = np.asarray(self.grad_fn(mu), dtype=np.float64)
            gns = float(np.dot(gr, gr))
        else:
            gns = math.nan
        if sync:
            self.sync_replica_checks.append((t, diag.identical))
            check_after_sync(diag, t)
        age = 0
        P, S = ctx.P, ctx.S
        if not sync and opt.use_group:
            stamps = self._stamps(t)
            if stamps is not None:
                age = max(0, max(t - int(s) for s in stamps))
            log_s = S.bit_length() - 1
            self._msgs += P * log_s + ((P - 1) if opt.cfg.alpha and t not in opt.forced_log else 0)
            self._bytes += _nvlink_bytes(P, S, ctx.R, t, opt.cfg.tau, ctx.n * (4 if ctx.dtype == torch.float32 else 8))
        elif sync:
            self._msgs += P * (P.bit_length() - 1)
            self._bytes += _nvlink_bytes(P, S, ctx.R, t, opt.cfg.tau, ctx.n * (4 if ctx.dtype == torch.float32 else 8))
        self.max_gamma = max(self.max_gamma, diag.gamma)
        self.max_staleness = max(self.max_staleness, age)
        rec = MetricsRecord(iteration=t, sim_time_ms=float(self._t0.elapsed_time(ev)), loss_mu=loss,
                            grad_norm_sq_mu=gns, gamma=diag.gamma, max_staleness=age, msgs_total=self._msgs,
                            bytes_total=self._bytes)
        self.records.append(rec)
        return rec

    def csv_text(self) -> str:
        return metrics_csv_text(self.records)


def _atomic_write(path: Path, data: str) -> None:
    tmp = path.with_suffix(path.suffix + ".tmp")
    tmp.write_text(data)
    os.replace(tmp, path)


def write_run(recorder: MetricsRecorder, out_dir, config: dict, seed: int) -> tuple[Path, Path, str]:
    """metrics.csv + manifest.json with the reference runner's schema (harness/runner.py:60-91)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    csv_text = recorder.csv_text()
    digest = hashlib.sha256(csv_text.encode()).hexdigest()
    metrics_path = out / "metrics.csv"
    _atomic_write(metrics_path, csv_text)
    manifest = {
        "schema_version": 1,
        "tool_version": __version__,
        "config": config,
        "seed": seed,
        "sim_time_start_ms": 0.0,
        "sim_time_end_ms": recorder.records[-1].sim_time_ms if recorder.records else 0.0,
        "metrics_sha256": digest,
        "metrics_rows": len(recorder.records),
    }
    manifest_path = out / "manifest.json"
    _atomic_write(manifest_path, json.dumps(manifest, indent=2, sort_keys=True) + "\n")
    return metrics_path, manifest_path, digest
