"""Oracle (TEST INFRASTRUCTURE): numpy restatement of the WAGMA hot-path arithmetic.

Restates, in the reference's own operation order, the arithmetic of
`/root/reference/pkg/src/wagma/optim.py` and `collective.py` for one
group-averaging iteration (see oracle/__init__.py for the usage rule):

  local step      m = beta*m + g ; W' = W - eta*m      (optim.py:176-183)
  send buffer     install W' with stamp t              (collective.py:95-101)
  group sum       recursive doubling, acc = incoming + acc per phase
                                                       (collective.py:310-329)
  averaging       timely acc/S ; late (acc + W')/(S+1) (optim.py:439-447)
  global sync     full butterfly (1,2,..,P/2), total/P (collective.py:368,
                                                        428-436; optim.py:449-452)

`replay_training` drives Alg. 2 (`_GroupAveragingWorker`, optim.py:403-452)
for all P ranks given the per-(version, rank) contribution stamps, which is
exactly what decides the arithmetic of a run; the stamps come from the
reference's own contribution log (golden fixtures) or from the device's
stamp log (live protocol tests). Pinned bit-exact against the reference's
`run_training` final weights in tests/test_oracle.py.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .topology_oracle import EXAMPLE, phase_masks


def is_sync_iteration(t: int, tau: Optional[int]) -> bool:
    """`is_sync_iteration` (optim.py:151-152)."""
    return tau is not None and tau > 0 and (t + 1) % tau == 0


def local_step(W: np.ndarray, m: Optional[np.ndarray], g: np.ndarray, eta: float, beta: float,
               update_rule: str):
    """`local_step` arithmetic (optim.py:176-183); returns (W', m')."""
    dt = W.dtype.type
    if update_rule == "momentum":
        if m is None:
            m = np.zeros_like(W)
        m = dt(beta) * m + g
        return W - dt(eta) * m, m
    return W - dt(eta) * g, m


def recursive_doubling(contribs: Sequence[np.ndarray], masks: Sequence[int]) -> list[np.ndarray]:
    """Every rank's accumulator after the in-group recursive doubling.

    Phase r: rank p receives its partner p ^ masks[r]'s accumulator and sets
    acc = incoming + acc (collective.py:317-325). Computed for all ranks at
    once, phase by phase, in the reference's operand order.
    """
    acc = [np.array(c, copy=True) for c in contribs]
    for m in masks:
        acc = [acc[p ^ m] + acc[p] for p in range(len(acc))]
    return acc


def group_round_sums(contribs: Sequence[np.ndarray], P: int, S: int, version: int,
                     rule: str = EXAMPLE) -> list[np.ndarray]:
    """Group accumulators of version `version` for all P ranks."""
    return recursive_doubling(contribs, phase_masks(P, S, version, rule))


def sync_sums(contribs: Sequence[np.ndarray]) -> list[np.ndarray]:
    """`SyncAllreduce` totals: masks (1, 2, ..., P/2) (collective.py:368)."""
    P = len(contribs)
    return recursive_doubling(contribs, [1 << j for j in range(P.bit_length() - 1)])


def finish_group_round(acc: np.ndarray, w_prime: np.ndarray, S: int, timely: bool) -> np.ndarray:
    """`_finish_group_round` (optim.py:439-447)."""
    if timely:
        return acc / S
    return (acc + w_prime) / (S + 1)


def replay_training(*, P: int, S: int, tau: Optional[int], T: int, w0: np.ndarray,
                    grads: np.ndarray, etas: np.ndarray, stamps: np.ndarray,
                    alpha: bool = True, beta: bool = False, update_rule: str = "sgd",
                    momentum: float = 0.9, mask_rule: str = EXAMPLE,
                    dtype=np.float64, return_history: bool = False):
    """Replay Alg. 2 (optim.py:403-452) for all ranks from a contribution schedule.

    grads[t, r] and etas[t, r] are the per-(iteration, rank) gradient and
    step size; stamps[t, r] is the send-buffer stamp rank r contributed to
    group version t (-1 = the initial model, collective.py:93/169), as the
    reference's `contribution_log` records it (collective.py:295-296).
    Returns the final weights [P, d] (and the per-iteration weights).
    """
    dt = np.dtype(dtype).type
    use_group = alpha or beta
    W = [np.array(w0, dtype=dt) for _ in range(P)]
    m: list[Optional[np.ndarray]] = [None] * P
    # send buffer history per rank: stamp -> W' (stamp -1 = W0)
    sendbuf = [{-1: np.array(w0, dtype=dt)} for _ in range(P)]
    history = [np.stack(W)]
    for t in range(T):
        wp = []
        for r in range(P):
            w_new, m[r] = local_step(W[r], m[r], np.asarray(grads[t, r], dtype=dt), float(etas[t, r]),
                                     momentum, update_rule)
            wp.append(w_new)
        if is_sync_iteration(t, tau):
            for r in range(P):
                if use_group:
                    sendbuf[r][t] = wp[r]        # install_fresh (optim.py:407-410)
            totals = sync_sums(wp)
            W = [totals[r] / P for r in range(P)]
        elif use_group:
            for r in range(P):
                sendbuf[r][t] = wp[r]            # join installs fresh (collective.py:205)
            contribs = [sendbuf[q][int(stamps[t, q])] for q in range(P)]
            accs = group_round_sums(contribs, P, S, t, mask_rule)
            W = [finish_group_round(accs[r], wp[r], S, int(stamps[t, r]) == t) for r in range(P)]
        else:
            W = [w.copy() for w in wp]
        history.append(np.stack(W))
    final = np.stack(W)
    return (final, history) if return_history else final


def rel_err_inf(a: np.ndarray, b: np.ndarray) -> float:
    """Norm-infinity relative error max|a-b| / max|b| (tests/test_acceptance.py:221)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(1e-300, float(np.max(np.abs(b)))))
