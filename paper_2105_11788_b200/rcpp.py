"""Single-relation partition refinement (RCPP, Alg. 2) on the B200.

Drop-in for /root/reference/pkg/src/parbisim/rcpp.py: `RelationInput`,
`rcpp_run` and `NONE_LABEL` keep the reference's names, arguments, results
and exceptions; `rcpp_arrays` is the array-level API underneath.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .bcrp import _ObserverBridge, _check_policy, _guard_error, _options, _plain_common, _raise_for
from .policy import PolicyViolationError, SuperstepLimitError
from .lts import Partition, RunStats

# Block labels are state ids, so -1 is "no label" (rcpp.py:32-35).
NONE_LABEL = -1


@dataclass(frozen=True)
class RelationInput:
    """A binary relation over 0..n-1 plus the partition to refine
    (rcpp.py:38-55).  ``edges`` may be a sequence of pairs or an (m, 2)
    int array; pi0 is used verbatim, including non-minimum leaders."""

    n: int
    edges: object
    pi0: Partition

    def __post_init__(self):
        e = self.edges
        if isinstance(e, np.ndarray):
            arr = np.ascontiguousarray(e, dtype=np.int32).reshape(-1, 2)
        else:
            pairs = [(int(s), int(t)) for s, t in e]
            arr = np.asarray(pairs, dtype=np.int32).reshape(-1, 2)
        if self.n < 1:
            raise ValueError("state count must be at least 1")
        if len(self.pi0) != self.n:
            raise ValueError("pi0 covers a different number of states")
        if arr.size:
            bad = np.nonzero((arr < 0).any(axis=1) | (arr >= self.n).any(axis=1))[0]
            if bad.size:
                s, t = arr[bad[0]]
                raise ValueError(f"edge ({int(s)}, {int(t)}) outside 0..{self.n - 1}")
        object.__setattr__(self, "_arr", arr)
        if not isinstance(e, np.ndarray):
            object.__setattr__(self, "edges", tuple((int(s), int(t)) for s, t in arr.tolist()))

    @classmethod
    def from_arrays(cls, n: int, src, dst, pi0) -> "RelationInput":
        arr = np.stack([N.as_i32(src), N.as_i32(dst)], axis=1)
        p = pi0 if isinstance(pi0, Partition) else Partition(np.asarray(pi0))
        return cls(n, arr, p)

    def columns(self) -> tuple[np.ndarray, np.ndarray]:
        a = self._arr
        return np.ascontiguousarray(a[:, 0]), np.ascontiguousarray(a[:, 1])


def _relation_columns(rel):
    if isinstance(rel, RelationInput):
        s, d = rel.columns()
    else:  # the reference's RelationInput (edges: tuple of pairs)
        m = len(rel.edges)
        flat = (np.fromiter((v for e in rel.edges for v in e), dtype=np.int32,
                            count=2 * m).reshape(m, 2) if m else np.zeros((0, 2), np.int32))
        s, d = np.ascontiguousarray(flat[:, 0]), np.ascontiguousarray(flat[:, 1])
    return int(rel.n), s, d, N.as_i32(rel.pi0.block)


def rcpp_arrays(n: int, src, dst, pi0, *, max_supersteps: int | None = None, observer=None,
                device: int = 0, mode: int = N.MODE_AUTO, flags: int = 0):
    """Refine leader-form ``pi0`` over edges (src[i], dst[i]).

    Returns ``(block, RunStats, native_stats)``.
    """
    src, dst, pi0 = N.as_i32(src), N.as_i32(dst), N.as_i32(pi0)
    if pi0.size != n:
        raise ValueError("pi0 covers a different number of states")
    guard = N.DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 16
    block = np.empty(n, np.int32)
    splits = np.zeros(cap, np.int32)
    st = N.Stats()
    bridge = _ObserverBridge(observer) if observer is not None else None
    opt = _options(device, mode, bridge, flags)  # an observer implies stepped rounds
    rc = N.lib().bisim_rcpp_ex(n, src.size, N.ptr(src), N.ptr(dst), N.ptr(pi0), guard,
                               N.ptr(block), N.ptr(splits), cap, ctypes.byref(st),
                               ctypes.byref(opt))
    _raise_for(rc, bridge, st)
    R = int(st.supersteps)
    stats = RunStats(supersteps=R, splits_per_iteration=tuple(splits[:R].tolist()),
                     final_block_count=int(st.final_blocks),
                     initial_block_count=int(st.initial_blocks))
    return block, stats, st.as_dict()


def rcpp_run(rel, policy, *, common_election: bool | None = None, observer=None,
             max_supersteps: int | None = None, device: int = 0):
    """Refine ``rel.pi0`` to the coarsest stable partition of the relation
    (rcpp.py:220-259); ``max_supersteps`` defaults to ``3n + 9``."""
    _check_policy(policy, common_election)
    n, src, dst, pi0 = _relation_columns(rel)
    if _plain_common(policy, common_election):
        _plain_common_rcpp(n, src, dst, pi0, max_supersteps, observer, device)
    block, stats, _ = rcpp_arrays(n, src, dst, pi0, max_supersteps=max_supersteps,
                                  observer=observer, device=device)
    return Partition(block, _trusted=True), stats


class _RoundOne(Exception):
    pass


def _plain_common_rcpp(n, src, dst, pi0, max_supersteps, observer, device):
    """rcpp_run under plain Common, as the reference executes it
    (rcpp.py:75-98, :196-204 with common_election=False).

    Two or more initial blocks: every leader is unstable and writes C at the
    first select.  One block (leader L): round 1 splits off the states whose
    "has an edge" mark differs from L's; two or more of them write
    new_leader[L] in sub-phase A (conflict), exactly one makes round 2's
    select see two unstable labels (conflict after round 1, whose observer
    call happens), none is the Priority run.  The round-1 split set is read
    from the GPU's Priority round 1 (identical to Common's up to sub_a).
    """
    guard = 3 * n + 9 if max_supersteps is None else int(max_supersteps)
    leaders = np.unique(pi0)
    if leaders.size >= 2:
        try:  # input validation only: a guard of 0 trips at the first superstep
            rcpp_arrays(n, src, dst, pi0, max_supersteps=0, device=device)
        except SuperstepLimitError:
            pass
        if guard < 1:
            raise _guard_error(1, guard)
        raise PolicyViolationError("C", leaders.tolist())
    L = int(leaders[0])
    got = {}

    def first(k, part):
        got["block"] = np.asarray(part.block, np.int32)
        raise _RoundOne

    try:
        rcpp_arrays(n, src, dst, pi0, max_supersteps=max_supersteps, observer=first,
                    device=device)
    except _RoundOne:
        pass
    if "block" not in got:
        return None            # no round ran (no conflict possible): Priority run
    S = np.nonzero(got["block"] != L)[0]
    if S.size >= 2:
        raise PolicyViolationError(("new_leader", L), S.tolist())
    if S.size == 1:
        if observer is not None:
            observer(1, Partition(got["block"], _trusted=True))
        if guard < 2:
            raise _guard_error(2, guard)
        raise PolicyViolationError("C", sorted([L, int(S[0])]))
    return None                # nothing split: the Priority run is the Common run


__all__ = ["NONE_LABEL", "RelationInput", "rcpp_arrays", "rcpp_run"]
