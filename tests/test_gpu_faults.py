"""Fault injection on the device path (reference: harness/verify.py:234-250,
collective.py:185 and :315-316 `_corrupt_outgoing`; SendBuffer / slot reuse
checks collective.py:96-99, 283-308).

- Corruption: the reference corrupts one process's outgoing PHASE payload and
  checks that the exact-sum verification notices it (and that an uncorrupted
  control trial is exact). Here the peer-visible payload is a rank's send-ring
  slot; corrupting the slot a stale member contributes must change the group
  sums of the other members, and the control trial must be bit-exact.
- Overwritten / torn slots: a contribution whose send-ring slot was reused
  (the ring wrapped past its stamp, or this very launch overwrites it) must
  latch WG_EPROTO (ProtocolFault), never be summed.
"""

import numpy as np
import pytest
import torch

from paper_2005_00124_b200 import _lib
from paper_2005_00124_b200.collective import GroupAllreduce
from paper_2005_00124_b200.context import DeviceContext, DeviceProtocolFault, Job
from paper_2005_00124_b200.topology import GroupingParams, compute_groups

pytestmark = pytest.mark.gpu


def _trial(corrupt):
    """P=8, S=4, version 0; rank 3 joins late, so its contribution is its
    initial send buffer (stamp -1, collective.py:93) read from its slot."""
    P, S, n = 8, 4, 16
    rng = np.random.default_rng(77)
    init = {r: rng.integers(-50, 50, n).astype(np.float64) for r in range(P)}
    fresh = {r: rng.integers(-50, 50, n).astype(np.float64) for r in range(P)}
    ctx = DeviceContext(P, S, n, dtype=torch.float64, timeout_s=5.0)
    results = {}
    groups = [GroupAllreduce(ctx, r, P, S, on_complete=lambda v, acc, t, s, r=r: results.__setitem__(r, acc.cpu().numpy()),
                             initial_model=init[r]) for r in range(P)]
    if corrupt is not None:
        view, held = ctx.slot(corrupt, -1)
        assert held == -1
        view[0] += 1e-3  # the payload peers read (verify.py:181-182)
    with ctx.batch():
        for r in range(P):
            if r != 3:
                groups[r].join_or_check(0, fresh[r])
    late = groups[3].join_or_check(0, fresh[3])
    results[3] = late.accumulator.cpu().numpy()
    ctx.close()
    part = compute_groups(GroupingParams(P, S, 0))
    contrib = {r: (init[r] if r == 3 else fresh[r]) for r in range(P)}
    mismatches = 0
    for r in range(P):
        expected = np.zeros(n)
        for m in part.group_of(r):
            expected = expected + contrib[m]
        mismatches += not np.array_equal(results[r], expected)
    return mismatches


def test_corruption_detected(cuda):
    assert _trial(corrupt=3) > 0, "sum check failed to notice an injected payload corruption"
    assert _trial(corrupt=None) == 0, "control trial should be exact"


def _steps(ctx, P, n, versions, stamps, ranks):
    """Forced-stamp launches (contribution-log replay mode) of `ranks`."""
    W = {r: torch.zeros(n, device=ctx.torch_device, dtype=torch.float64) for r in range(P)}
    m = {r: torch.zeros_like(W[r]) for r in range(P)}
    g = torch.ones(n, device=ctx.torch_device, dtype=torch.float64)
    for v, st in zip(versions, stamps):
        jobs = [Job(rank=r, kind=_lib.WG_JOB_STEP, version=v, W=W[r], m=m[r], g=g, eta=0.1, beta=0.9, momentum=True)
                for r in ranks]
        ctx.launch(jobs, forced={v: st})
        torch.cuda.synchronize()
        ctx.check()


def test_wrapped_slot_is_a_protocol_fault(cuda):
    """A contribution stamp whose slot the ring has reused (ring depth 4,
    stamp 1 while slot 2 already holds stamp 5) -> WG_EPROTO."""
    P, n = 2, 4096
    ctx = DeviceContext(P, 2, n, dtype=torch.float64, ring_depth=4, timeout_s=5.0)
    _steps(ctx, P, n, range(6), [[v, v] for v in range(6)], ranks=(0, 1))
    with pytest.raises(DeviceProtocolFault) as ei:
        _steps(ctx, P, n, [6], [[6, 1]], ranks=(0,))
    assert ei.value.code == _lib.WG_EPROTO
    ctx.close()


def test_slot_overwritten_in_launch_is_a_protocol_fault(cuda):
    """Rank 1 publishes stamp 6 into slot 3 in the very launch that would read
    its stamp-2 contribution from slot 3 (a torn read) -> WG_EPROTO."""
    P, n = 2, 4096
    ctx = DeviceContext(P, 2, n, dtype=torch.float64, ring_depth=4, timeout_s=5.0)
    _steps(ctx, P, n, range(6), [[v, v] for v in range(6)], ranks=(0, 1))
    with pytest.raises(DeviceProtocolFault) as ei:
        _steps(ctx, P, n, [6], [[6, 2]], ranks=(0, 1))
    assert ei.value.code == _lib.WG_EPROTO
    ctx.close()
