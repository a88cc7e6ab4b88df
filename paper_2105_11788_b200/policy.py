"""Write policies and run-time errors of the refinement path.

Mirrors /root/reference/pkg/src/parbisim/pram.py:29-71.  The reference
simulates a CRCW PRAM and resolves concurrent writes per policy; on the GPU
the Priority rule ("lowest processor index wins", pram.py:153-154) is what
the kernels implement with order-independent atomics.  Common with its
pairwise elections (Alg. 6, rcpp.py:101-179) elects exactly the same
winners, so it maps to the same kernels.  Arbitrary(seed) picks other legal
winners; the GPU runs it with the Priority winners, which the Arbitrary
model also allows (any single writer may win): the resulting
partition is the same coarsest bisimulation, while the round count may
differ from the reference's crc32-salted choice.
"""
from __future__ import annotations

from dataclasses import dataclass


class WritePolicy:
    __slots__ = ()


@dataclass(frozen=True)
class Priority(WritePolicy):
    pass


@dataclass(frozen=True)
class Arbitrary(WritePolicy):
    seed: int


@dataclass(frozen=True)
class Common(WritePolicy):
    pass


class PolicyViolationError(RuntimeError):
    """Concurrent Common-policy writes disagreed on a value (pram.py:60-67)."""

    def __init__(self, address, values):
        self.address = address
        self.values = sorted(set(values))
        super().__init__(f"conflicting common writes to cell {address!r}: values {self.values}")


class SuperstepLimitError(RuntimeError):
    """The refinement loop exceeded its superstep guard (pram.py:70-71)."""


def policy_kind(policy) -> str:
    """'priority' | 'common' | 'arbitrary' for this package's policies and,
    by class name, for the reference's own policy objects."""
    name = type(policy).__name__
    if name in ("Priority", "Common", "Arbitrary"):
        return name.lower()
    raise TypeError(f"unknown write policy {policy!r}")
