"""The drop-in collective API on the device, against the reference's own results.

tests/golden/collective.npz holds accumulators produced by the reference's
`GroupAllreduce` / `SyncAllreduce` endpoints on its simulator (all-timely
rounds, rounds with stale members, literal mask rule, global sync). Here the
same rounds run through `paper_2005_00124_b200.collective` on one GPU (all P
ranks in one process; ranks that join "at the same instant" join inside one
`ctx.batch()`), in fp64: accumulators must be bit-identical. Also restates
the reference's protocol unit tests (test_collective.py).
"""

import json
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2005_00124_b200.collective import (
    GroupAllreduce,
    JoinStatus,
    ProtocolFault,
    SyncAllreduce,
    VersionRegressionError,
)
from paper_2005_00124_b200.context import DeviceContext
from paper_2005_00124_b200.topology import InvalidParamsError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    z = np.load(os.path.join(GOLDEN, "collective.npz"))
    return z, json.loads(str(z["cases"]))


class Node:
    def __init__(self, ctx, rank, P, S, init, **kw):
        self.results = {}
        self.group = GroupAllreduce(ctx, rank, P, S, on_complete=self._done, initial_model=init, **kw)

    def _done(self, version, acc, timely, stamp):
        self.results[version] = (acc.cpu().numpy(), timely, stamp)


def _cases(golden, kind):
    z, cases = golden
    return [c for c in cases if c["kind"] == kind]


def test_group_rounds_all_timely_bit_exact(cuda, golden):
    z, _ = golden
    n = 0
    for c in _cases(golden, "timely"):
        i, P, S, v = c["id"], c["P"], c["S"], c["version"]
        ctx = DeviceContext(P, S, 37, dtype=torch.float64, mask_rule=c["rule"], timeout_s=5.0)
        nodes = [Node(ctx, r, P, S, z[f"c{i}_stale"][r], mask_rule=c["rule"]) for r in range(P)]
        with ctx.batch():
            res = [nodes[r].group.join_or_check(v, z[f"c{i}_fresh"][r]) for r in range(P)]
        for r in range(P):
            assert res[r].status is JoinStatus.ACTIVE
            acc, timely, stamp = nodes[r].results[v]
            assert np.array_equal(acc, z[f"c{i}_acc"][r]), (c, r)
            assert timely and stamp == v
        ctx.close()
        n += 1
    assert n >= 50


def test_group_rounds_with_stale_members_bit_exact(cuda, golden):
    z, _ = golden
    for c in _cases(golden, "stale"):
        i, P, S = c["id"], c["P"], c["S"]
        late = set(c["late"])
        ctx = DeviceContext(P, S, 37, dtype=torch.float64, timeout_s=5.0)
        nodes = [Node(ctx, r, P, S, z[f"c{i}_stale"][r]) for r in range(P)]
        with ctx.batch():  # the early joiners, at (nearly) the same instant
            for r in range(P):
                if r not in late:
                    nodes[r].group.join_or_check(0, z[f"c{i}_fresh"][r])
        late_res = {}
        with ctx.batch():  # the stragglers, long after the activation
            for r in sorted(late):
                late_res[r] = nodes[r].group.join_or_check(0, z[f"c{i}_fresh"][r])
        for r in range(P):
            if r in late:
                assert late_res[r].status is JoinStatus.ALREADY_DONE
                acc = late_res[r].accumulator.cpu().numpy()
            else:
                acc, timely, stamp = nodes[r].results[0]
                assert timely and stamp == 0
            assert np.array_equal(acc, z[f"c{i}_acc"][r]), (c, r)
        # the late fresh model stays in the send buffer for future pulls
        for r in late:
            assert nodes[r].group.send_buffer.stamped_iteration == 0
            assert np.array_equal(nodes[r].group.send_buffer.payload.cpu().numpy(), z[f"c{i}_fresh"][r])
        ctx.close()


def test_sync_allreduce_bit_exact(cuda, golden):
    z, _ = golden
    for c in _cases(golden, "sync"):
        i, P = c["id"], c["P"]
        ctx = DeviceContext(P, 1, 37, dtype=torch.float64, timeout_s=5.0)
        got = {}
        eps = [SyncAllreduce(ctx, r, P, on_complete=lambda it, tot, r=r: got.__setitem__(r, tot.cpu().numpy()))
               for r in range(P)]
        with ctx.batch():
            for r in range(P):
                eps[r].join(3, z[f"c{i}_fresh"][r])
        for r in range(P):
            assert np.array_equal(got[r], z[f"c{i}_acc"][r])
        assert all(np.array_equal(got[r], got[0]) for r in range(P))
        ctx.close()


def test_version_regression_and_s1(cuda):
    ctx = DeviceContext(2, 1, 4, dtype=torch.float64, timeout_s=5.0)
    nodes = [Node(ctx, r, 2, 1, np.zeros(4)) for r in range(2)]
    vec = np.array([4.0, 5.0, 6.0, 7.0])
    res = nodes[0].group.join_or_check(3, vec)  # S=1: completes inside the call with its own buffer
    assert res.status is JoinStatus.ACTIVE
    acc, timely, stamp = nodes[0].results[3]
    assert np.array_equal(acc, vec) and timely and stamp == 3
    with pytest.raises(VersionRegressionError):
        nodes[0].group.join_or_check(2, vec)
    with pytest.raises(VersionRegressionError):
        nodes[0].group.join_or_check(3, vec)
    ctx.close()


def test_blocking_mode_sums_and_requires_group(cuda):
    P, S = 4, 2
    ctx = DeviceContext(P, S, 3, dtype=torch.float64, activation_enabled=False, timeout_s=5.0)
    vecs = [np.arange(3, dtype=np.float64) + 10.0 * (r + 1) for r in range(P)]
    nodes = [Node(ctx, r, P, S, np.zeros(3), activation_enabled=False) for r in range(P)]
    with ctx.batch():
        for r in range(P):
            nodes[r].group.join_or_check(0, vecs[r])
    for r in range(P):
        acc, timely, _ = nodes[r].results[0]
        assert timely and np.array_equal(acc, vecs[r] + vecs[r ^ 1])
    with pytest.raises(InvalidParamsError):  # a blocking group member cannot join alone
        nodes[0].group.join_or_check(1, vecs[0])
    ctx.close()


def test_staleness_bound_enforced_at_activation(cuda):
    ctx = DeviceContext(2, 2, 1, dtype=torch.float64, staleness_bound=3, timeout_s=5.0)
    nodes = [Node(ctx, r, 2, 2, np.zeros(1), staleness_bound=3) for r in range(2)]
    nodes[0].group.install_fresh(np.ones(1), 1)
    # rank 1 activates version 5 while rank 0's buffer is stamped 1: age 4 >= 3
    with pytest.raises(ProtocolFault):
        nodes[1].group.join_or_check(5, np.ones(1))
    ctx.close()


def test_install_regression_rejected(cuda):
    ctx = DeviceContext(2, 2, 2, dtype=torch.float64, timeout_s=5.0)
    node = Node(ctx, 0, 2, 2, np.zeros(2))
    node.group.install_fresh(np.ones(2), 4)
    assert node.group.send_buffer.stamped_iteration == 4
    assert np.array_equal(node.group.send_buffer.payload.cpu().numpy(), np.ones(2))
    with pytest.raises(ProtocolFault):
        node.group.install_fresh(np.ones(2), 3)
    ctx.close()


def test_activation_tree_message_counts(cuda):
    """Exactly one activator per version; the binomial ACT tree rooted at it
    has P-1 edges and every member sends log2 S phase messages
    (test_collective.py:231-245, collective.py:263-274, :319)."""
    P, S, n_versions = 8, 4, 5
    ctx = DeviceContext(P, S, 64, dtype=torch.float64, timeout_s=5.0)
    nodes = [Node(ctx, r, P, S, np.zeros(64)) for r in range(P)]
    rng = np.random.default_rng(3)
    for v in range(n_versions):
        late = {int(x) for x in rng.choice(P, 2, replace=False)} if v % 2 else set()
        with ctx.batch():
            for r in range(P):
                if r not in late:
                    nodes[r].group.join_or_check(v, rng.standard_normal(64))
        if late:
            with ctx.batch():
                for r in sorted(late):
                    nodes[r].group.join_or_check(v, rng.standard_normal(64))
    groups = [nd.group for nd in nodes]
    assert sum(g.activations_originated for g in groups) == n_versions
    assert sum(g.acts_sent for g in groups) == (P - 1) * n_versions
    assert all(g.phases_sent == 2 * n_versions for g in groups)
    with pytest.raises(ProtocolFault):
        groups[0].handle_message(1, b"")
    ctx.close()


def test_mismatched_sync_points_protocol_fault(cuda):
    """collective.py:381-386: one rank joins iteration t as a global sync while
    another joins t as a group round -> ProtocolFault (mismatched sync points),
    not a hang. Co-located ranks share one launch, so the device rejects the
    mixed launch (WG_ESYNC); across GPUs the kernels compare the sync marks
    (test_gpu_multi.py::test_multigpu_mismatched_sync_points)."""
    P = 2
    ctx = DeviceContext(P, 2, 8, dtype=torch.float64, timeout_s=5.0)
    got = {}
    sync = SyncAllreduce(ctx, 0, P, on_complete=lambda t, tot: got.setdefault(t, tot))
    node = Node(ctx, 1, P, 2, np.zeros(8))
    with pytest.raises(ProtocolFault, match="mismatched sync points"):
        with ctx.batch():
            sync.join(3, np.ones(8))
            node.group.join_or_check(3, np.ones(8))
    assert not got
    ctx.close()


def test_straggler_passive_completion_then_already_done(cuda):
    """Restates test_collective.py:124-155 (reference): group {0,1} at version 0,
    rank 1 slow. Rank 0 sums fresh_0 + stale_1; rank 1's endpoint completes
    passively (on_complete, not timely, stamp -1) before its own join, which
    returns ALREADY_DONE with the finished sum and installs its fresh model."""
    P, S, d = 4, 2, 2
    stale = [np.full(d, -float(r + 1)) for r in range(P)]
    fresh = [np.arange(d, dtype=np.float64) + 10.0 * (r + 1) for r in range(P)]
    ctx = DeviceContext(P, S, d, dtype=torch.float64, timeout_s=5.0)
    nodes = [Node(ctx, r, P, S, stale[r]) for r in range(P)]
    with ctx.batch():
        for r in (0, 2, 3):
            nodes[r].group.join_or_check(0, fresh[r])
    acc0, timely0, _ = nodes[0].results[0]
    assert np.array_equal(acc0, fresh[0] + stale[1]) and timely0
    acc1, timely1, stamp1 = nodes[1].results[0]  # passive completion, before rank 1 joined
    assert np.array_equal(acc1, fresh[0] + stale[1])
    assert not timely1 and stamp1 == -1
    assert nodes[1].group.execution_count[0] == 1
    res = nodes[1].group.join_or_check(0, fresh[1])
    assert res.status is JoinStatus.ALREADY_DONE
    assert np.array_equal(res.accumulator.cpu().numpy(), fresh[0] + stale[1])
    # fresh model stays in the send buffer for future pulls
    assert np.array_equal(nodes[1].group.send_buffer.payload.cpu().numpy(), fresh[1])
    assert nodes[1].group.send_buffer.stamped_iteration == 0
    assert nodes[1].group.execution_count[0] == 1  # executed exactly once (A4)
    ctx.close()
