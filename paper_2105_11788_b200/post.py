"""The steps either side of the refinement path, on the GPU.

* :func:`quotient` -- the quotient system of a partition
  (/root/reference/pkg/src/parbisim/aut.py:132-152): one state per block,
  blocks numbered densely in leader order, duplicate transitions merged in
  first-occurrence order.
* :func:`is_stable` -- every state sees the same (action, target block) pairs
  as its leader (/root/reference/pkg/src/parbisim/oracle.py:128-141);
  :func:`is_stable_under` -- the same for one target set (oracle.py:144-154).
* :func:`canonical_arrays` -- leader form of an arbitrary id assignment
  (/root/reference/pkg/src/parbisim/lts.py:117-128), for assignments too
  large for host code.

Each has an array-level form (``*_arrays``: int32 columns in and out) and a
reference-typed form taking :class:`Lts` / :class:`Partition` objects.  All
work happens in libbisim.so (``bisim_quotient``, ``bisim_is_stable``,
``bisim_canonical``); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .bcrp import lts_columns
from .lts import Lts, Partition


def _check(rc: int):
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(N.last_error())
    N.check(rc)


def quotient_arrays(n: int, src, act, dst, num_actions: int, block, initial_state: int = 0,
                    device: int = 0):
    """Quotient of the system (src, act, dst) by the leader-form ``block``.

    Returns ``(q_n, q_src, q_act, q_dst, q_initial)``; action ids are
    unchanged.
    """
    src, act, dst, block = (N.as_i32(x) for x in (src, act, dst, block))
    if block.size != n:
        raise ValueError("partition covers a different number of states")
    m = src.size
    cap = max(m, 1)
    qs, qa, qd = (np.empty(cap, np.int32) for _ in range(3))
    qn, qm, qi = ctypes.c_int32(0), ctypes.c_int64(0), ctypes.c_int32(0)
    _check(N.lib().bisim_quotient(n, m, int(num_actions), N.ptr(src), N.ptr(act), N.ptr(dst),
                                  N.ptr(block), int(initial_state), ctypes.byref(qn),
                                  ctypes.byref(qm), N.ptr(qs), N.ptr(qa), N.ptr(qd),
                                  ctypes.byref(qi), device))
    k = int(qm.value)
    return int(qn.value), qs[:k].copy(), qa[:k].copy(), qd[:k].copy(), int(qi.value)


def quotient(lts, p, device: int = 0) -> Lts:
    """Quotient system (aut.py:132-152); raises ValueError on a size mismatch."""
    if len(p) != lts.n:
        raise ValueError("partition covers a different number of states")
    n, src, act, dst, A = lts_columns(lts)
    block = np.asarray(p.block, np.int32)
    qn, qs, qa, qd, qi = quotient_arrays(n, src, act, dst, A, block,
                                         getattr(lts, "initial_state", 0), device)
    return Lts.from_arrays(qn, qs, qa, qd, tuple(lts.action_labels), qi, validate=False)


def is_stable_arrays(n: int, src, act, dst, num_actions: int, block, device: int = 0) -> bool:
    src, act, dst, block = (N.as_i32(x) for x in (src, act, dst, block))
    if block.size != n:
        raise ValueError("partition covers a different number of states")
    out = ctypes.c_int32(0)
    _check(N.lib().bisim_is_stable(n, src.size, int(num_actions), N.ptr(src), N.ptr(act),
                                   N.ptr(dst), N.ptr(block), ctypes.byref(out), device))
    return bool(out.value)


def is_stable(lts, partition, device: int = 0) -> bool:
    """True when every block is stable under every block (oracle.py:128-141)."""
    if len(partition) != lts.n:
        raise ValueError("partition covers a different number of states")
    n, src, act, dst, A = lts_columns(lts)
    return is_stable_arrays(n, src, act, dst, A, np.asarray(partition.block, np.int32), device)


def is_stable_under_arrays(n: int, src, act, dst, num_actions: int, block, states,
                           device: int = 0) -> bool:
    src, act, dst, block = (N.as_i32(x) for x in (src, act, dst, block))
    if block.size != n:
        raise ValueError("partition covers a different number of states")
    st = np.ascontiguousarray(np.fromiter((int(x) for x in states), dtype=np.int64))
    st = st[(st >= 0) & (st < n)].astype(np.int32)  # other ids are never reached
    out = ctypes.c_int32(0)
    _check(N.lib().bisim_is_stable_under(n, src.size, int(num_actions), N.ptr(src), N.ptr(act),
                                         N.ptr(dst), N.ptr(block), N.ptr(st), st.size,
                                         ctypes.byref(out), device))
    return bool(out.value)


def is_stable_under(lts, partition, states, device: int = 0) -> bool:
    """True when every block either wholly reaches ``states`` via each action
    or wholly avoids it (oracle.py:144-154)."""
    if len(partition) != lts.n:
        raise ValueError("partition covers a different number of states")
    n, src, act, dst, A = lts_columns(lts)
    return is_stable_under_arrays(n, src, act, dst, A, np.asarray(partition.block, np.int32),
                                  states, device)


def canonical_arrays(assignment, device: int = 0) -> np.ndarray:
    """Leader form of an id assignment: states sharing an id share a block led
    by its smallest state (lts.py:117-128).  Ids are int64."""
    a = np.ascontiguousarray(np.asarray(assignment, dtype=np.int64).reshape(-1))
    if a.size == 0:
        raise ValueError("a partition needs at least one state")
    out = np.empty(a.size, np.int32)
    _check(N.lib().bisim_canonical(a.size, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                   N.ptr(out), device))
    return out


def canonical_partition(assignment, device: int = 0) -> Partition:
    return Partition(canonical_arrays(assignment, device), _trusted=True)


__all__ = ["quotient", "quotient_arrays", "is_stable", "is_stable_arrays", "is_stable_under",
           "is_stable_under_arrays", "canonical_arrays", "canonical_partition"]
