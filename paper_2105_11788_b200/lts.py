"""Boundary types of the refinement path: transition systems in, leader-form
partitions and run statistics out.

Mirrors the reference's domain types (/root/reference/pkg/src/parbisim/lts.py)
name for name and with the same validation and error behaviour, so code that
drives `parbisim` can switch to this package unchanged.  The one addition is
an array-backed constructor, :meth:`Lts.from_arrays`, that keeps the
transition columns as int32 numpy arrays: building millions of Transition
tuples costs seconds in Python, while the CUDA path only needs
the three columns.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, NamedTuple, Sequence

import numpy as np

StateId = int
ActionId = int


class Transition(NamedTuple):
    """One labelled edge ``source --action--> target`` (lts.py:19-22)."""

    source: StateId
    action: ActionId
    target: StateId


class Lts:
    """Immutable labelled transition system (lts.py:25-56).

    ``action_labels[a]`` is the label string of action id ``a``.  States are
    ``0..n-1``.  Either a tuple of :class:`Transition` or, via
    :meth:`from_arrays`, three int32 columns back the transitions; the other
    form is materialised on first use.
    """

    __slots__ = ("n", "action_labels", "initial_state", "_transitions", "_cols")

    def __init__(self, n: int, action_labels: Sequence[str], transitions: Iterable = (),
                 initial_state: StateId = 0):
        labels = tuple(action_labels)
        trans = tuple(Transition(*t) for t in transitions)
        self._init(n, labels, initial_state)
        object.__setattr__(self, "_transitions", trans)
        object.__setattr__(self, "_cols", None)
        k = len(labels)
        for t in trans:
            if not (0 <= t.source < n and 0 <= t.target < n):
                raise ValueError(f"transition {t} mentions a state outside 0..{n - 1}")
            if not 0 <= t.action < k:
                raise ValueError(f"transition {t} uses an undeclared action id")

    def _init(self, n, labels, initial_state):
        if n < 1:
            raise ValueError("state count must be at least 1")
        if len(set(labels)) != len(labels):
            raise ValueError("duplicate action labels")
        if not 0 <= initial_state < n:
            raise ValueError("initial state out of range")
        object.__setattr__(self, "n", int(n))
        object.__setattr__(self, "action_labels", labels)
        object.__setattr__(self, "initial_state", int(initial_state))

    @classmethod
    def from_arrays(cls, n: int, src, act, dst, action_labels: Sequence[str] | int,
                    initial_state: StateId = 0, validate: bool = True) -> "Lts":
        """Array-backed system; ``action_labels`` may be a label count."""
        if isinstance(action_labels, (int, np.integer)):
            action_labels = tuple(f"a{i}" for i in range(int(action_labels)))
        self = cls.__new__(cls)
        self._init(n, tuple(action_labels), initial_state)
        cols = tuple(np.ascontiguousarray(np.asarray(c, dtype=np.int32).reshape(-1))
                     for c in (src, act, dst))
        if not (cols[0].size == cols[1].size == cols[2].size):
            raise ValueError("transition columns differ in length")
        if validate and cols[0].size:
            k = len(self.action_labels)
            for name, c, hi in (("source", cols[0], n), ("target", cols[2], n)):
                if c.min() < 0 or c.max() >= hi:
                    raise ValueError(f"a transition {name} lies outside 0..{n - 1}")
            if cols[1].min() < 0 or cols[1].max() >= k:
                raise ValueError("a transition uses an undeclared action id")
        object.__setattr__(self, "_transitions", None)
        object.__setattr__(self, "_cols", cols)
        return self

    def __setattr__(self, name, value):
        raise AttributeError("Lts is immutable")

    @property
    def transitions(self) -> tuple[Transition, ...]:
        if self._transitions is None:
            s, a, t = self._cols
            object.__setattr__(self, "_transitions",
                               tuple(Transition(int(x), int(y), int(z))
                                     for x, y, z in zip(s.tolist(), a.tolist(), t.tolist())))
        return self._transitions

    def columns(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(src, act, dst) as contiguous int32 arrays."""
        if self._cols is None:
            m = len(self._transitions)
            flat = np.fromiter((v for t in self._transitions for v in t), dtype=np.int32,
                               count=3 * m).reshape(m, 3) if m else np.zeros((0, 3), np.int32)
            object.__setattr__(self, "_cols", tuple(np.ascontiguousarray(flat[:, k])
                                                    for k in range(3)))
        return self._cols

    @property
    def m(self) -> int:
        return int(self._cols[0].size) if self._cols is not None else len(self._transitions)

    def __eq__(self, other) -> bool:
        if not isinstance(other, Lts):
            return NotImplemented
        if (self.n, self.action_labels, self.initial_state) != (other.n, other.action_labels,
                                                                 other.initial_state):
            return False
        return all(np.array_equal(x, y) for x, y in zip(self.columns(), other.columns()))

    def __repr__(self) -> str:
        return f"Lts(n={self.n}, m={self.m}, action_labels={self.action_labels!r})"


def lts_from_labeled_edges(n: int, edges: Iterable[tuple[int, str, int]],
                           initial_state: int = 0, extra_labels: Iterable[str] = ()) -> Lts:
    """Lts from ``(source, label, target)`` triples; action ids follow the
    sorted label order, ``extra_labels`` declares unused labels
    (lts.py:59-73)."""
    edges = list(edges)
    labels = sorted(set(extra_labels).union(lab for _, lab, _ in edges))
    rank = {lab: i for i, lab in enumerate(labels)}
    return Lts(n, tuple(labels), [Transition(s, rank[lab], t) for s, lab, t in edges],
               initial_state)


class Partition:
    """Partition of ``0..n-1`` in leader form: ``block[s]`` is the leader of
    s's block and every leader leads itself (lts.py:76-114)."""

    __slots__ = ("block",)

    def __init__(self, block: Sequence[int], _trusted: bool = False):
        if isinstance(block, np.ndarray):
            arr = np.asarray(block, dtype=np.int64).reshape(-1)
            if arr.size == 0:
                raise ValueError("a partition needs at least one state")
            if not _trusted:
                n = arr.size
                bad = np.nonzero((arr < 0) | (arr >= n))[0]
                if bad.size:
                    s = int(bad[0])
                    raise ValueError(f"block label {int(arr[s])} of state {s} is out of range")
                bad = np.nonzero(arr[arr] != arr)[0]
                if bad.size:
                    s = int(bad[0])
                    raise ValueError(f"state {s} names leader {int(arr[s])}, which is not its own leader")
            blk = tuple(arr.tolist())
        else:
            blk = tuple(int(b) for b in block)
            if not blk:
                raise ValueError("a partition needs at least one state")
            if not _trusted:
                n = len(blk)
                for s, b in enumerate(blk):
                    if b < 0 or b >= n:
                        raise ValueError(f"block label {b} of state {s} is out of range")
                    if blk[b] != b:
                        raise ValueError(f"state {s} names leader {b}, which is not its own leader")
        object.__setattr__(self, "block", blk)

    def __setattr__(self, name, value):
        raise AttributeError("Partition is immutable")

    def __len__(self) -> int:
        return len(self.block)

    def __eq__(self, other) -> bool:
        return isinstance(other, Partition) and self.block == other.block

    def __hash__(self) -> int:
        return hash(self.block)

    def __repr__(self) -> str:
        return f"Partition({list(self.block)!r})"

    def blocks(self) -> dict[int, list[int]]:
        """Leader -> ascending member list."""
        out: dict[int, list[int]] = {}
        for s, b in enumerate(self.block):
            out.setdefault(b, []).append(s)
        return out


def partition_from_assignment(assignment: Sequence[int]) -> Partition:
    """Canonical partition of an arbitrary id assignment: each block is led by
    its smallest state (lts.py:117-128)."""
    if len(assignment) == 0:
        raise ValueError("a partition needs at least one state")
    arr = np.asarray(assignment)
    _, first, inverse = np.unique(arr, return_index=True, return_inverse=True)
    return Partition(first[inverse.reshape(-1)], _trusted=True)


def partitions_equal(p: Partition, q: Partition) -> bool:
    """Same equivalence relation, leader names aside (lts.py:131-141)."""
    if len(p) != len(q):
        raise ValueError("partitions cover different numbers of states")
    a = np.asarray(p.block)
    b = np.asarray(q.block)
    pairs = np.unique(np.stack([a, b], axis=1), axis=0)
    return len(pairs) == len(np.unique(a)) == len(np.unique(b))


def partition_refines(fine: Partition, coarse: Partition) -> bool:
    """Every block of ``fine`` lies inside one block of ``coarse``
    (lts.py:144-149)."""
    if len(fine) != len(coarse):
        raise ValueError("partitions cover different numbers of states")
    f = np.asarray(fine.block)
    c = np.asarray(coarse.block)
    return bool(np.all(c == c[f]))


def block_count(p: Partition) -> int:
    return len(set(p.block))


def trivial_partition(n: int) -> Partition:
    """One block led by state 0."""
    return Partition([0] * n, _trusted=n > 0)


def discrete_partition(n: int) -> Partition:
    return Partition(range(n), _trusted=n > 0)


@dataclass(frozen=True)
class RunStats:
    """Statistics of one refinement run (lts.py:164-184).

    ``supersteps`` counts loop iterations that selected a splitter (the
    terminal pass is not counted); ``splits_per_iteration[k]`` is the number
    of blocks split in iteration k+1.
    """

    supersteps: int
    splits_per_iteration: tuple[int, ...]
    final_block_count: int
    initial_block_count: int

    def __post_init__(self):
        if self.supersteps != len(self.splits_per_iteration):
            raise ValueError("supersteps must equal len(splits_per_iteration)")
        if self.initial_block_count < 1 or self.final_block_count < self.initial_block_count:
            raise ValueError("block counts cannot shrink during refinement")
