"""Subtree partition of the H^2 tree across 2^s ranks.

Rank g owns, at every level l >= s, the nodes [g 2^(l-s), (g+1) 2^(l-s)) of
the complete binary cluster tree (its top-level subtree), the leaves, basis
nodes and coupling/dense block rows below them; levels < s are replicated.
One mat-vec then needs exactly two collectives: an all-gather of x^ at the
levels >= s (each rank's slice of a level is contiguous in the
level-concatenated node-vector pool) and an all-gather of the cluster-order
y slices.  This module is the single source of that index arithmetic; the
C++ side (Matrix::own_begin/own_end in csrc/h2b_internal.hpp) mirrors it and
tests/test_partition*.py check both agree.
"""
from __future__ import annotations


def log2_exact(p: int) -> int:
    if p < 1 or p & (p - 1):
        raise ValueError("partition count must be a power of two")
    return p.bit_length() - 1


def owned_range(level: int, s: int, g: int) -> tuple[int, int]:
    if level < s:
        return 0, 1 << level
    return g << (level - s), (g + 1) << (level - s)


def vec_offsets(ranks) -> list[int]:
    off = [0]
    for l, k in enumerate(ranks):
        off.append(off[-1] + (1 << l) * int(k))
    return off


class PartitionPlan:
    """Index plan of one rank: x^ slices to all-gather, the y slice it produces."""

    def __init__(self, depth: int, ranks, m: int, nparts: int, part: int):
        self.depth, self.ranks, self.m = depth, [int(k) for k in ranks], m
        self.nparts, self.part = nparts, part
        self.s = log2_exact(nparts)
        if self.s > depth:
            raise ValueError("more partitions than leaves")
        if not 0 <= part < nparts:
            raise ValueError("partition index out of range")
        self.off = vec_offsets(self.ranks)

    def level_slice(self, l: int) -> tuple[int, int, int]:
        """(level offset, level length, per-rank chunk) in the x^ pool, l >= s."""
        k = self.ranks[l]
        return self.off[l], (1 << l) * k, (1 << (l - self.s)) * k

    def gather_levels(self):
        return [l for l in range(self.s, self.depth + 1) if self.ranks[l] > 0]

    def leaf_range(self) -> tuple[int, int]:
        return owned_range(self.depth, self.s, self.part)

    def y_slice(self) -> tuple[int, int]:
        a, b = self.leaf_range()
        return a * self.m, b * self.m
