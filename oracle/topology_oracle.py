"""Oracle (TEST INFRASTRUCTURE): restatement of the reference schedule generator.

Restates `/root/reference/pkg/src/wagma/topology.py` (see oracle/__init__.py
for the usage rule). Pinned against tests/golden/topology.json.
"""

from __future__ import annotations

import numpy as np

EXAMPLE = "example"
LITERAL = "literal"


class OracleInvalidParams(ValueError):
    pass


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def check_params(P: int, S: int, t: int) -> None:
    """`GroupingParams.__post_init__` (topology.py:64-72)."""
    if not _is_pow2(P) or not _is_pow2(S) or S > P or t < 0:
        raise OracleInvalidParams((P, S, t))


def phase_masks(P: int, S: int, t: int, rule: str = EXAMPLE) -> tuple[int, ...]:
    """`phase_masks` (topology.py:118-142)."""
    check_params(P, S, t)
    gp = S.bit_length() - 1          # group_phases  (topology.py:79-80)
    GP = P.bit_length() - 1          # global_phases (topology.py:75-76)
    if rule == EXAMPLE:              # topology.py:127-128
        return tuple(1 << ((t * gp + r) % GP) for r in range(gp)) if GP else ()
    if rule == LITERAL:              # topology.py:129-139
        out = []
        mask = 1
        shift = (t * gp) % GP if GP else 0   # shift0 (topology.py:83-87)
        for _ in range(gp):
            mask = (mask << shift) % P
            if mask == 0:
                mask = 1
            out.append(mask)
            shift = (shift + 1) % GP if GP else 0
        return tuple(out)
    raise OracleInvalidParams(rule)


def xor_span(masks) -> list[int]:
    """`_xor_span` (topology.py:154-159)."""
    span = {0}
    for m in masks:
        span |= {s ^ m for s in span}
    return sorted(span)


def compute_groups(P: int, S: int, t: int, rule: str = EXAMPLE) -> tuple[tuple[int, ...], ...]:
    """`compute_groups` (topology.py:162-181): cosets of the XOR span, sorted."""
    span = xor_span(phase_masks(P, S, t, rule))
    seen: set[int] = set()
    groups = []
    for p in range(P):
        if p in seen:
            continue
        members = tuple(sorted(p ^ s for s in span))
        groups.append(members)
        seen.update(members)
    return tuple(groups)


def peer(rank: int, mask: int, P: int) -> int:
    """`peer` (topology.py:145-151)."""
    if not 0 <= rank < P or not (_is_pow2(mask) and mask < P):
        raise OracleInvalidParams((rank, mask, P))
    return rank ^ mask


def mixing_reachable(P: int, S: int, start_t: int, k: int, rule: str = EXAMPLE) -> bool:
    """`mixing_reachable` (topology.py:184-208)."""
    if k < 1 or start_t < 0:
        raise OracleInvalidParams((start_t, k))
    reach = [1 << p for p in range(P)]
    for t in range(start_t, start_t + k):
        nxt = list(reach)
        for grp in compute_groups(P, S, t, rule):
            merged = 0
            for m in grp:
                merged |= reach[m]
            for m in grp:
                nxt[m] = merged
        reach = nxt
    full = (1 << P) - 1
    return all(r == full for r in reach)


def leaf_ranks(P: int, S: int, t: int, rank: int, rule: str = EXAMPLE) -> list[int]:
    """Leaf order of the butterfly tree the reference's recursive doubling
    builds at `rank` (collective.py:310-329): leaf i is
    rank ^ XOR{masks[r] : bit r of i}; level r of the tree combines leaves
    i and i ^ (1 << r)."""
    masks = phase_masks(P, S, t, rule)
    out = []
    for i in range(1 << len(masks)):
        q = rank
        for r, m in enumerate(masks):
            if (i >> r) & 1:
                q ^= m
        out.append(q)
    return out


def victims(selection_seed: int, iteration: int, P: int, k: int) -> frozenset[int]:
    """`StragglerPolicy.victims` (netsim.py:75-82) -- the same numpy PCG64 call."""
    if k <= 0:
        return frozenset()
    rng = np.random.default_rng([selection_seed, iteration])
    return frozenset(int(v) for v in rng.choice(P, size=k, replace=False))
