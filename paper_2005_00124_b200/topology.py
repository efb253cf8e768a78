"""Butterfly phase schedules and dynamic group partitions (drop-in for `wagma.topology`).

Same names, arguments, return types and errors as the reference module
(`/root/reference/pkg/src/wagma/topology.py`); the computation itself runs
in the C++ schedule generator of libwagma_b200.so (`csrc/topology.cpp`),
which is also what plans the device kernel's summation trees, so the
schedule the kernel executes is the one these functions report.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _lib

__all__ = [
    "GroupingParams",
    "PhasePlan",
    "GroupPartition",
    "InvalidParamsError",
    "phase_masks",
    "compute_groups",
    "peer",
    "mixing_reachable",
    "tree_leaves",
    "MASK_RULE_EXAMPLE",
    "MASK_RULE_LITERAL",
]

MASK_RULE_EXAMPLE = "example"
MASK_RULE_LITERAL = "literal"

_INT32_MAX = 2**31 - 1


class InvalidParamsError(ValueError):
    """Raised for process counts / group sizes / ranks outside the contract
    (topology.py:45-46)."""


def _is_pow2(n: int) -> bool:
    return n >= 1 and (n & (n - 1)) == 0


def _rule_code(rule: str) -> int:
    try:
        return _lib.RULES[rule]
    except (KeyError, TypeError):
        raise InvalidParamsError(f"unknown mask rule {rule!r}") from None


def _check(rc: int, what: str) -> None:
    if rc == _lib.WG_EINVAL:
        raise InvalidParamsError(f"{what}: {_lib.last_error() or 'invalid parameters'}")
    if rc != _lib.WG_OK:
        raise RuntimeError(f"{what}: error {rc}")


@dataclass(frozen=True)
class GroupingParams:
    """Grouping inputs: P ranks, group size S, iteration index t (topology.py:53-87).

    P and S must be powers of two with 1 <= S <= P; t >= 0.
    """

    P: int
    S: int
    t: int = 0

    def __post_init__(self) -> None:
        if not _is_pow2(self.P):
            raise InvalidParamsError(f"P={self.P} is not a power of two")
        if not _is_pow2(self.S):
            raise InvalidParamsError(f"S={self.S} is not a power of two")
        if self.S > self.P:
            raise InvalidParamsError(f"S={self.S} exceeds P={self.P}")
        if self.t < 0:
            raise InvalidParamsError(f"iteration t={self.t} is negative")
        if self.P > 2**30:
            raise InvalidParamsError(f"P={self.P} exceeds the supported 2**30")

    @property
    def global_phases(self) -> int:
        return self.P.bit_length() - 1

    @property
    def group_phases(self) -> int:
        return self.S.bit_length() - 1

    @property
    def shift0(self) -> int:
        """Phase offset of this iteration within the butterfly cycle."""
        if self.global_phases == 0:
            return 0
        return (self.t * self.group_phases) % self.global_phases


@dataclass(frozen=True)
class PhasePlan:
    """Ordered single-bit masks executed by one iteration, phase by phase."""

    P: int
    S: int
    t: int
    masks: tuple[int, ...]

    def __len__(self) -> int:
        return len(self.masks)


@dataclass(frozen=True)
class GroupPartition:
    """Disjoint rank groups active at one iteration (topology.py:103-115).

    ``groups`` is sorted by smallest member; each group is a sorted tuple.
    """

    iteration: int
    groups: tuple[tuple[int, ...], ...]
    rank_to_group: dict[int, int] = field(repr=False, hash=False, compare=False, default_factory=dict)

    def group_of(self, rank: int) -> tuple[int, ...]:
        return self.groups[self.rank_to_group[rank]]


def _t64(t: int) -> int:
    # iteration indices beyond int64 are reduced modulo lcm-free periods:
    # the masks only depend on t mod log2(P), so t mod 2**62 * ... is not
    # needed for any realistic run; reject instead of silently wrapping.
    if t > 2**62:
        raise InvalidParamsError(f"iteration t={t} too large")
    return t


def phase_masks(params: GroupingParams, rule: str = MASK_RULE_EXAMPLE) -> PhasePlan:
    """Compute the log2(S) butterfly masks for iteration t (topology.py:118-142)."""
    code = _rule_code(rule)
    lib = _lib.load()
    buf = (ctypes.c_int * 32)()
    n = ctypes.c_int(0)
    _check(lib.wg_phase_masks(params.P, params.S, _t64(params.t), code, buf, ctypes.byref(n)), "phase_masks")
    return PhasePlan(P=params.P, S=params.S, t=params.t, masks=tuple(buf[i] for i in range(n.value)))


def compute_groups(params: GroupingParams, rule: str = MASK_RULE_EXAMPLE) -> GroupPartition:
    """Partition ranks into the groups induced by iteration t's masks (topology.py:162-181)."""
    code = _rule_code(rule)
    lib = _lib.load()
    P = params.P
    members = (ctypes.c_int * P)()
    offsets = (ctypes.c_int * (P + 1))()
    ng = ctypes.c_int(0)
    _check(lib.wg_compute_groups(P, params.S, _t64(params.t), code, members, offsets, ctypes.byref(ng)),
           "compute_groups")
    flat = list(members)
    groups = []
    rank_to_group: dict[int, int] = {}
    for g in range(ng.value):
        grp = tuple(flat[offsets[g]:offsets[g + 1]])
        groups.append(grp)
        for r in grp:
            rank_to_group[r] = g
    return GroupPartition(iteration=params.t, groups=tuple(groups), rank_to_group=rank_to_group)


def peer(rank: int, mask: int, P: int) -> int:
    """Exchange partner of ``rank`` under single-bit ``mask``: rank XOR mask (topology.py:145-151)."""
    if not (-(2**31) <= rank <= _INT32_MAX and -(2**31) <= mask <= _INT32_MAX and 0 < P <= _INT32_MAX):
        raise InvalidParamsError(f"rank {rank} / mask {mask} / P {P} out of range")
    out = ctypes.c_int(0)
    _check(_lib.load().wg_peer(rank, mask, P, ctypes.byref(out)), f"peer(rank={rank}, mask={mask}, P={P})")
    return out.value


def mixing_reachable(params: GroupingParams, start_t: int, k: int, rule: str = MASK_RULE_EXAMPLE) -> bool:
    """True iff k consecutive iterations' groupings connect every rank pair (topology.py:184-208)."""
    if k < 1:
        raise InvalidParamsError(f"iteration count k={k} must be >= 1")
    if start_t < 0:
        raise InvalidParamsError(f"start_t={start_t} is negative")
    code = _rule_code(rule)
    out = ctypes.c_int(0)
    _check(_lib.load().wg_mixing_reachable(params.P, params.S, _t64(start_t), k, code, ctypes.byref(out)),
           "mixing_reachable")
    return bool(out.value)


def tree_leaves(params: GroupingParams, rank: int, rule: str = MASK_RULE_EXAMPLE) -> tuple[int, ...]:
    """Leaf order of the butterfly summation tree at ``rank`` (the device
    kernel's fixed reduction order; collective.py:310-329)."""
    code = _rule_code(rule)
    buf = (ctypes.c_int * (1 << params.group_phases))()
    n = ctypes.c_int(0)
    _check(_lib.load().wg_tree_leaves(params.P, params.S, _t64(params.t), code, rank, buf, ctypes.byref(n)),
           "tree_leaves")
    return tuple(buf[i] for i in range(n.value))
