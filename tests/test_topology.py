"""Schedule generator (C++ via the C ABI) against the reference, bit-exact.

Restates the reference's known-answer tests (`pkg/tests/test_topology.py`,
A1/A2 of `pkg/tests/test_acceptance.py`) against the drop-in module and
checks the full A2 grid (P <= 1024, both rules) against the reference's own
outputs frozen in tests/golden/topology.json. CPU only.
"""

import hashlib
import json
import math
import os

import pytest

from conftest import GOLDEN
from oracle import topology_oracle as oracle_topo
from paper_2005_00124_b200.topology import (
    MASK_RULE_LITERAL,
    GroupingParams,
    InvalidParamsError,
    compute_groups,
    mixing_reachable,
    peer,
    phase_masks,
    tree_leaves,
)


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(GOLDEN, "topology.json")) as fp:
        return json.load(fp)


def groups_as_sets(partition):
    return {frozenset(g) for g in partition.groups}


def test_masks_known_answers():
    assert phase_masks(GroupingParams(8, 4, 0)).masks == (1, 2)
    assert phase_masks(GroupingParams(8, 4, 1)).masks == (4, 1)
    assert phase_masks(GroupingParams(8, 8, 0)).masks == (1, 2, 4)
    assert phase_masks(GroupingParams(16, 1, 7)).masks == ()
    assert phase_masks(GroupingParams(16, 4, 1)).masks == (4, 8)
    assert phase_masks(GroupingParams(8, 4, 1), rule=MASK_RULE_LITERAL).masks == (4, 4)


@pytest.mark.parametrize("P,S", [(3, 2), (8, 3), (4, 8), (0, 1)])
def test_invalid_params(P, S):
    with pytest.raises(InvalidParamsError):
        GroupingParams(P, S, 0)
    with pytest.raises(InvalidParamsError):
        GroupingParams(8, 4, -1)


def test_unknown_rule_rejected():
    with pytest.raises(InvalidParamsError):
        phase_masks(GroupingParams(8, 4, 0), rule="bogus")


def test_worked_examples_and_group_of():
    assert groups_as_sets(compute_groups(GroupingParams(8, 4, 0))) == {frozenset({0, 1, 2, 3}),
                                                                       frozenset({4, 5, 6, 7})}
    part = compute_groups(GroupingParams(8, 4, 1))
    assert groups_as_sets(part) == {frozenset({0, 1, 4, 5}), frozenset({2, 3, 6, 7})}
    assert part.group_of(5) == (0, 1, 4, 5)
    assert part.group_of(6) == (2, 3, 6, 7)


def test_a2_grid_masks_bit_exact(golden):
    for key, masks in golden["masks"].items():
        P, S, t, rule = key.split(",")
        assert list(phase_masks(GroupingParams(int(P), int(S), int(t)), rule).masks) == masks, key


def test_a2_grid_partitions_bit_exact(golden):
    n = 0
    for key, digest in golden["groups_sha"].items():
        P, S, t, rule = key.split(",")
        part = compute_groups(GroupingParams(int(P), int(S), int(t)), rule)
        k = ";".join(",".join(str(r) for r in g) for g in part.groups)
        assert hashlib.sha256(k.encode()).hexdigest() == digest, key
        if key in golden["groups_full"]:
            assert [list(g) for g in part.groups] == golden["groups_full"][key]
        n += 1
    assert n == len(golden["masks"])


def test_mixing_and_peer_known_answers(golden):
    for P, S, start, k, rule, want in golden["mixing"]:
        assert mixing_reachable(GroupingParams(P, S, 0), start, k, rule) == want, (P, S, start, k, rule)
    for rank, mask, P, want in golden["peer"]:
        if want is None:
            with pytest.raises(InvalidParamsError):
                peer(rank, mask, P)
        else:
            assert peer(rank, mask, P) == want
    with pytest.raises(InvalidParamsError):
        mixing_reachable(GroupingParams(8, 4, 0), 0, 0)


def test_partition_periodicity():
    for P, S in [(16, 4), (64, 4), (256, 16), (8, 2)]:
        gp, GP = int(math.log2(S)), int(math.log2(P))
        period = GP // math.gcd(gp, GP)
        for t in range(6):
            assert compute_groups(GroupingParams(P, S, t)).groups == \
                compute_groups(GroupingParams(P, S, t + period)).groups


def test_tree_leaves_follow_recursive_doubling():
    # leaf i = rank ^ XOR{masks[r] : bit r of i}; every member's tree holds
    # exactly its group (with multiplicity for repeated literal masks).
    for P, S, rule in [(8, 4, "example"), (16, 8, "example"), (8, 4, "literal"), (32, 16, "literal")]:
        for t in range(8):
            params = GroupingParams(P, S, t)
            for rank in range(P):
                leaves = tree_leaves(params, rank, rule)
                assert list(leaves) == oracle_topo.leaf_ranks(P, S, t, rank, rule)
                assert set(leaves) == set(compute_groups(params, rule).group_of(rank))
                assert len(leaves) == S
