"""Labelled bisimulation refinement (BCRP, Alg. 3-5) on the B200.

Drop-in for /root/reference/pkg/src/parbisim/bcrp.py: same entry points
(`bcrp_run`, `preprocess`, `partition_by_outgoing_labels`, `BcrpAux`), same
arguments, results and exceptions.  The work happens in libbisim.so; this
module only converts between the reference's types and int32 arrays.

`bcrp_arrays` is the array-level API underneath: numpy columns
in, the int32 block array plus RunStats out, with no per-transition Python
objects anywhere.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .lts import Lts, Partition, RunStats, Transition
from .policy import PolicyViolationError, SuperstepLimitError, policy_kind


@dataclass(frozen=True)
class BcrpAux:
    """Preprocessing tables (bcrp.py:37-46), in sorted-transition order."""

    lts: Lts
    action_switch: tuple[int, ...]
    order: tuple[int, ...]
    nr_marks: tuple[int, ...]
    off: tuple[int, ...]
    mark_length: int


def lts_columns(lts) -> tuple[int, np.ndarray, np.ndarray, np.ndarray, int]:
    """(n, src, act, dst, |Act|) for this package's Lts or any object with the
    reference Lts attributes (n, action_labels, transitions)."""
    if isinstance(lts, Lts):
        s, a, d = lts.columns()
        return lts.n, s, a, d, len(lts.action_labels)
    trans = lts.transitions
    m = len(trans)
    flat = (np.fromiter((v for t in trans for v in (t[0], t[1], t[2])), dtype=np.int32,
                        count=3 * m).reshape(m, 3) if m else np.zeros((0, 3), np.int32))
    cols = [np.ascontiguousarray(flat[:, k]) for k in range(3)]
    return int(lts.n), cols[0], cols[1], cols[2], len(lts.action_labels)


class _ObserverBridge:
    """Adapts observer(iteration, Partition) to the C callback; an exception
    raised by the observer aborts the native run and is re-raised here."""

    def __init__(self, observer):
        self.observer = observer
        self.exc = None

        def cb(k, block_ptr, n, _user):
            try:
                blk = np.ctypeslib.as_array(block_ptr, shape=(n,)).copy()
                self.observer(int(k), Partition(blk, _trusted=True))
                return 0
            except BaseException as e:  # noqa: BLE001 - re-raised below
                self.exc = e
                return 1

        self.cfunc = N.OBSERVER(cb)


def _options(device: int, mode: int, bridge, flags: int = 0) -> N.Options:
    o = N.Options()
    o.device = device
    o.mode = mode
    o.flags = flags
    if bridge is not None:
        o.observer = bridge.cfunc
    return o


def _raise_for(rc: int, bridge, guard_msg_stats: N.Stats):
    if rc == N.BISIM_OK:
        return
    msg = N.last_error()
    if rc == N.BISIM_ABORTED and bridge is not None and bridge.exc is not None:
        raise bridge.exc
    if rc == N.BISIM_GUARD:
        raise SuperstepLimitError(msg)
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(msg)
    raise N.NativeError(rc, msg)


def bcrp_arrays(n: int, src, act, dst, num_actions: int, *, max_supersteps: int | None = None,
                observer=None, device: int = 0, mode: int = N.MODE_AUTO, flags: int = 0):
    """Coarsest bisimulation of the LTS given by int32 columns.

    Returns ``(block, RunStats, native_stats)`` where ``block`` is an int32
    numpy array in canonical leader form.  ``flags`` (``_native.FLAG_*``)
    selects another schedule of the same program; results never change.
    """
    src, act, dst = N.as_i32(src), N.as_i32(act), N.as_i32(dst)
    m = src.size
    guard = N.DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 16
    block = np.empty(n, np.int32)
    splits = np.zeros(cap, np.int32)
    st = N.Stats()
    bridge = _ObserverBridge(observer) if observer is not None else None
    opt = _options(device, mode, bridge, flags)  # an observer implies stepped rounds
    rc = N.lib().bisim_bcrp_ex(n, m, int(num_actions), N.ptr(src), N.ptr(act), N.ptr(dst), guard,
                               N.ptr(block), N.ptr(splits), cap, ctypes.byref(st),
                               ctypes.byref(opt))
    _raise_for(rc, bridge, st)
    R = int(st.supersteps)
    stats = RunStats(supersteps=R, splits_per_iteration=tuple(splits[:R].tolist()),
                     final_block_count=int(st.final_blocks),
                     initial_block_count=int(st.initial_blocks))
    return block, stats, st.as_dict()


def _plain_common(policy, common_election) -> bool:
    """True for Common without the Alg. 6 election: the reference then
    raises PolicyViolationError at the first conflicting concurrent write
    (pram.py:147-152)."""
    kind = policy_kind(policy)
    if common_election is None:
        common_election = kind == "common"
    return kind == "common" and not common_election


def _guard_error(step: int, limit: int):
    return SuperstepLimitError(f"superstep guard exceeded ({step} > {limit})")


def _label_rounds_common(n, src, act, A, device):
    """(conflict round or -1, old leader, new leader, block) of the plain-
    Common label rounds (bisim_label_rounds_common)."""
    r, lead, win = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    block = np.empty(n, np.int32)
    rc = N.lib().bisim_label_rounds_common(n, src.size, A, N.ptr(src), N.ptr(act),
                                           ctypes.byref(r), ctypes.byref(lead), ctypes.byref(win),
                                           N.ptr(block), device)
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(N.last_error())
    N.check(rc)
    return r.value, lead.value, win.value, block


def _plain_common_bcrp(n, src, act, dst, A, max_supersteps, observer, device):
    """bcrp_run under plain Common, as the reference executes it.

    Until the first conflicting write the Common rounds are the Priority
    rounds.  Conflicts can only occur (a) in a label round's elect phase
    (two states of one block disagree with their leader), (b) at the first
    main-loop select, when the label partition has two or more blocks (every
    leader writes C).  With one block every state has the same label set,
    so every slot of every state is marked in round 1 and nothing splits:
    the Priority run is the Common run.
    """
    guard = 3 * n + A + 8 if max_supersteps is None else int(max_supersteps)
    r, lead, win, block = _label_rounds_common(n, src, act, A, device)
    trip = max(guard, 0) + 1                   # the superstep at which the guard fires
    if r >= 0:
        if trip <= r + 1:                      # before the conflicting label round
            raise _guard_error(trip, guard)
        raise PolicyViolationError(("new_leader", lead), np.nonzero(block == win)[0].tolist())
    if trip <= A:
        raise _guard_error(trip, guard)
    leaders = np.unique(block)
    if leaders.size >= 2:
        if guard < A + 1:
            raise _guard_error(A + 1, guard)
        raise PolicyViolationError("C", leaders.tolist())
    return None   # one block: run the Priority program


def _check_policy(policy, common_election):
    return policy_kind(policy)


def bcrp_run(lts, policy, *, common_election: bool | None = None, observer=None,
             max_supersteps: int | None = None, device: int = 0):
    """Coarsest strong bisimulation of a labelled system (bcrp.py:192-315).

    Same contract as the reference: returns ``(Partition, RunStats)``;
    ``observer(iteration, partition)`` is called after every counted
    superstep; ``max_supersteps`` defaults to ``3n + |Act| + 8`` and raises
    :class:`SuperstepLimitError` when exceeded.  Plain ``Common`` (no
    election) raises :class:`PolicyViolationError` exactly where the
    reference does.
    """
    plain = _plain_common(policy, common_election)
    n, src, act, dst, A = lts_columns(lts)
    if plain:
        _plain_common_bcrp(n, N.as_i32(src), N.as_i32(act), N.as_i32(dst), A, max_supersteps,
                           observer, device)
    block, stats, _ = bcrp_arrays(n, src, act, dst, A, max_supersteps=max_supersteps,
                                  observer=observer, device=device)
    return Partition(block, _trusted=True), stats


def partition_by_outgoing_labels(lts, policy, *, common_election: bool | None = None,
                                 device: int = 0) -> Partition:
    """States grouped by outgoing label set, min-index leaders
    (bcrp.py:129-141)."""
    n, src, act, _, A = lts_columns(lts)
    if _plain_common(policy, common_election):
        # the engine's guard is |Act| + 1 (bcrp.py:139): never trips here
        r, lead, win, blk = _label_rounds_common(n, N.as_i32(src), N.as_i32(act), A, device)
        if r >= 0:
            raise PolicyViolationError(("new_leader", lead), np.nonzero(blk == win)[0].tolist())
        return Partition(blk, _trusted=True)
    block = np.empty(n, np.int32)
    rc = N.lib().bisim_label_partition(n, src.size, A, N.ptr(src), N.ptr(act), N.ptr(block),
                                       device)
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(N.last_error())
    N.check(rc)
    return Partition(block, _trusted=True)


def preprocess(lts, device: int = 0) -> BcrpAux:
    """Label-ordering tables (bcrp.py:116-126), computed on the GPU
    (``bisim_preprocess_sorted``): the transitions stably sorted by (source,
    action) with a device radix sort, then action_switch, order, nr_marks,
    off and mark_length of that order.  The refinement path itself never
    sorts; this is the reference's table export.
    """
    n, src, act, dst, A = lts_columns(lts)
    m = src.size
    mm = max(m, 1)
    perm, s_src, s_act, s_dst, sw, order = (np.empty(mm, np.int32) for _ in range(6))
    nr = np.empty(n, np.int32)
    off = np.empty(n, np.int32)
    L = ctypes.c_int64(0)
    rc = N.lib().bisim_preprocess_sorted(n, m, A, N.ptr(src), N.ptr(act), N.ptr(dst), N.ptr(perm),
                                         N.ptr(s_src), N.ptr(s_act), N.ptr(s_dst), N.ptr(sw),
                                         N.ptr(order), N.ptr(nr), N.ptr(off), ctypes.byref(L),
                                         device)
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(N.last_error())
    N.check(rc)
    sorted_lts = Lts.from_arrays(n, s_src[:m], s_act[:m], s_dst[:m], lts.action_labels,
                                 getattr(lts, "initial_state", 0), validate=False)
    return BcrpAux(lts=sorted_lts, action_switch=tuple(sw[:m].tolist()),
                   order=tuple(order[:m].tolist()), nr_marks=tuple(nr.tolist()),
                   off=tuple(off.tolist()), mark_length=int(L.value))


__all__ = ["BcrpAux", "bcrp_arrays", "bcrp_run", "partition_by_outgoing_labels", "preprocess",
           "lts_columns", "Transition"]
