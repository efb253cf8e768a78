"""Hierarchical (GPU-local subtree) sums are bit-identical to the reference's
recursive doubling (CPU, no GPU needed).

The device sums a plan either over its leaves or -- when the lowest hl tree
levels stay inside one GPU under the block rank mapping (wg_launch, mirrored
by bench.hier_levels) -- first over each GPU's block of 2^hl consecutive
leaves (the subtree partials the producers publish), then over the partials,
optionally reduce-scattered over their keys. Both must reproduce the
reference's `acc = incoming + acc` recursion (collective.py:310-329) bit for
bit at every rank; this restates that claim on random fp32 data for every
(P, S, t, GPU count) of the box sizes.
"""

import importlib.util
import os

import numpy as np
import pytest

from conftest import ROOT
from oracle import topology_oracle as otopo
from oracle import wagma_oracle as wo


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _tree(vals):
    """Butterfly tree in leaf order: level r pairs subtrees i and i ^ (1 << r)."""
    vals = list(vals)
    while len(vals) > 1:
        vals = [vals[2 * i] + vals[2 * i + 1] for i in range(len(vals) // 2)]
    return vals[0]


@pytest.mark.parametrize("P", [4, 8, 16])
def test_subtree_partials_bit_identical(P):
    hier_levels = _bench().hier_levels
    rng = np.random.default_rng(P)
    contribs = [(rng.standard_normal(257) * 10.0 ** rng.integers(-3, 4)).astype(np.float32) for _ in range(P)]
    n_hier = 0
    for S in [s for s in (2, 4, 8, 16) if s <= P]:
        for t in range(6):
            ref = wo.group_round_sums(contribs, P, S, t)  # the reference's operand order
            for G in [g for g in (2, 4, 8) if g <= P]:
                R = P // G
                for p in range(P):
                    leaves = otopo.leaf_ranks(P, S, t, p)
                    full = _tree([contribs[q] for q in leaves])
                    assert np.array_equal(full, ref[p])
                    hl = hier_levels(leaves, R)
                    if not hl:
                        continue
                    n_hier += 1
                    # every block of 2^hl leaves lives on one GPU
                    blocks = [leaves[u:u + (1 << hl)] for u in range(0, len(leaves), 1 << hl)]
                    assert all(len({q // R for q in b}) == 1 for b in blocks)
                    partials = [_tree([contribs[q] for q in b]) for b in blocks]
                    assert np.array_equal(_tree(partials), ref[p]), (P, S, t, G, p)
    assert n_hier > 0
