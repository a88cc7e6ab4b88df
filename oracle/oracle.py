"""ctypes front end of the CPU oracle (oracle/bisim_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU-baseline legs of bench.py, never by the product package.  The C file
restates the reference's PRAM programs (bcrp.py:49-315, rcpp.py:58-259) under
the Priority policy; this module only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OR_OK, OR_BAD_INPUT, OR_GUARD, OR_NOMEM = 0, 1, 2, 3
_DEFAULT_GUARD = -(2 ** 63)  # INT64_MIN: "use the reference default"


class _Stats(ctypes.Structure):
    _fields_ = [("supersteps", ctypes.c_int64),
                ("label_rounds", ctypes.c_int64),
                ("guard_count", ctypes.c_int64),
                ("initial_blocks", ctypes.c_int32),
                ("final_blocks", ctypes.c_int32),
                ("mark_length", ctypes.c_int64),
                ("t_pre_s", ctypes.c_double),
                ("t_label_s", ctypes.c_double),
                ("t_loop_s", ctypes.c_double)]


class OracleGuardError(RuntimeError):
    """The oracle's superstep guard tripped (reference SuperstepLimitError)."""


@dataclass
class OracleResult:
    block: np.ndarray          # int32[n], leader form
    supersteps: int
    splits: np.ndarray         # int32[supersteps]
    initial_blocks: int
    final_blocks: int
    mark_length: int
    snapshots: np.ndarray | None  # int32[k, n] block after rounds 1..k
    t_pre_s: float = 0.0
    t_label_s: float = 0.0
    t_loop_s: float = 0.0


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.POINTER
        i32p = P(ctypes.c_int32)
        L.oracle_preprocess.restype = ctypes.c_int64
        L.oracle_preprocess.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                        i32p, i32p, i32p, i32p, i32p, i32p, i32p]
        L.oracle_label_partition.restype = ctypes.c_int
        L.oracle_label_partition.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                             i32p, i32p, i32p, ctypes.c_int]
        L.oracle_bcrp.restype = ctypes.c_int
        L.oracle_bcrp.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, i32p, i32p,
                                  i32p, ctypes.c_int64, i32p, i32p, ctypes.c_int64, i32p,
                                  ctypes.c_int64, ctypes.c_int64, P(_Stats), ctypes.c_int]
        L.oracle_rcpp.restype = ctypes.c_int
        L.oracle_rcpp.argtypes = [ctypes.c_int32, ctypes.c_int64, i32p, i32p, i32p,
                                  ctypes.c_int64, i32p, i32p, ctypes.c_int64, i32p,
                                  ctypes.c_int64, ctypes.c_int64, P(_Stats), ctypes.c_int]
        L.oracle_bcrp_fast.restype = ctypes.c_int
        L.oracle_bcrp_fast.argtypes = [ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, i32p, i32p,
                                       i32p, ctypes.c_int64, i32p, i32p, ctypes.c_int64,
                                       P(_Stats), ctypes.c_int]
        L.oracle_rcpp_fast.restype = ctypes.c_int
        L.oracle_rcpp_fast.argtypes = [ctypes.c_int32, ctypes.c_int64, i32p, i32p, i32p,
                                       ctypes.c_int64, i32p, i32p, ctypes.c_int64, P(_Stats)]
        vp = ctypes.c_void_p
        u8p = P(ctypes.c_uint8)
        i64p = P(ctypes.c_int64)
        L.oracle_open.restype = vp
        L.oracle_open.argtypes = [ctypes.c_int, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                  i32p, i32p, i32p, i32p, ctypes.c_int, P(_Stats)]
        L.oracle_set_state.restype = None
        L.oracle_set_state.argtypes = [vp, i32p, u8p]
        L.oracle_rounds.restype = ctypes.c_int64
        L.oracle_rounds.argtypes = [vp, ctypes.c_int64, ctypes.c_int, P(ctypes.c_double)]
        L.oracle_block.restype = i32p
        L.oracle_block.argtypes = [vp]
        L.oracle_close.restype = None
        L.oracle_close.argtypes = [vp]
        L.oracle_fast_states.restype = ctypes.c_int
        L.oracle_fast_states.argtypes = [ctypes.c_int, ctypes.c_int32, ctypes.c_int64,
                                         ctypes.c_int32, i32p, i32p, i32p, i32p, ctypes.c_int64,
                                         i64p, i32p, u8p, ctypes.c_int]
        _lib = L
    return _lib


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def preprocess(n, src, act, num_actions):
    """Returns (perm, action_switch, order, nr_marks, off, mark_length) in the
    reference's sorted-transition order (bcrp.py:116-126)."""
    src, act = _i32(src), _i32(act)
    m = src.size
    perm = np.empty(max(m, 1), np.int32)
    sw = np.empty(max(m, 1), np.int32)
    order = np.empty(max(m, 1), np.int32)
    nr = np.empty(n, np.int32)
    off = np.empty(n, np.int32)
    L = lib().oracle_preprocess(n, m, num_actions, _ptr(src), _ptr(act), _ptr(perm), _ptr(sw),
                                _ptr(order), _ptr(nr), _ptr(off))
    if L < 0:
        raise MemoryError("oracle preprocess failed")
    return perm[:m], sw[:m], order[:m], nr, off, int(L)


def label_partition(n, src, act, num_actions, threads=1) -> np.ndarray:
    src, act = _i32(src), _i32(act)
    block = np.empty(n, np.int32)
    rc = lib().oracle_label_partition(n, src.size, num_actions, _ptr(src), _ptr(act),
                                      _ptr(block), threads)
    if rc != OR_OK:
        raise RuntimeError(f"oracle label partition failed ({rc})")
    return block


def bcrp_fast(n, src, act, dst, num_actions, max_supersteps=None, threads=1) -> OracleResult:
    """Event-driven sequential restatement (oracle/bisim_fast.c): same
    results as bcrp(), round cost O(|C| + in(C) + touched blocks)."""
    src, act, dst = _i32(src), _i32(act), _i32(dst)
    guard = _DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + num_actions + 9 if max_supersteps is None else max(int(max_supersteps), 0) + 1
    block = np.empty(n, np.int32)
    splits = np.zeros(cap + 1, np.int32)
    st = _Stats()
    rc = lib().oracle_bcrp_fast(n, src.size, num_actions, _ptr(src), _ptr(act), _ptr(dst), guard,
                                _ptr(block), _ptr(splits), cap, ctypes.byref(st), threads)
    return _finish(rc, st, block, splits, None, 0)


def rcpp_fast(n, src, dst, pi0, max_supersteps=None) -> OracleResult:
    """Event-driven sequential restatement of rcpp() (oracle/bisim_fast.c)."""
    src, dst, pi0 = _i32(src), _i32(dst), _i32(pi0)
    guard = _DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 10 if max_supersteps is None else max(int(max_supersteps), 0) + 1
    block = np.empty(n, np.int32)
    splits = np.zeros(cap + 1, np.int32)
    st = _Stats()
    rc = lib().oracle_rcpp_fast(n, src.size, _ptr(src), _ptr(dst), _ptr(pi0), guard, _ptr(block),
                                _ptr(splits), cap, ctypes.byref(st))
    return _finish(rc, st, block, splits, None, 0)


def _finish(rc, st, block, splits, snap, snap_rounds):
    if rc == OR_GUARD:
        raise OracleGuardError(f"superstep guard exceeded at superstep {st.guard_count}")
    if rc != OR_OK:
        raise RuntimeError(f"oracle failed ({rc})")
    R = int(st.supersteps)
    snaps = None
    if snap is not None:
        snaps = snap[:min(R, snap_rounds)]
    return OracleResult(block=block, supersteps=R, splits=splits[:R].copy(),
                        initial_blocks=int(st.initial_blocks),
                        final_blocks=int(st.final_blocks), mark_length=int(st.mark_length),
                        snapshots=snaps, t_pre_s=st.t_pre_s, t_label_s=st.t_label_s,
                        t_loop_s=st.t_loop_s)


def bcrp(n, src, act, dst, num_actions, max_supersteps=None, snap_rounds=0,
         threads=1, stop_after=-1) -> OracleResult:
    src, act, dst = _i32(src), _i32(act), _i32(dst)
    guard = _DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + num_actions + 9 if max_supersteps is None else max(int(max_supersteps), 0) + 1
    block = np.empty(n, np.int32)
    splits = np.zeros(cap + 1, np.int32)
    snap = np.empty((snap_rounds, n), np.int32) if snap_rounds else None
    st = _Stats()
    rc = lib().oracle_bcrp(n, src.size, num_actions, _ptr(src), _ptr(act), _ptr(dst), guard,
                           _ptr(block), _ptr(splits), cap,
                           _ptr(snap) if snap is not None else None, snap_rounds,
                           stop_after, ctypes.byref(st), threads)
    return _finish(rc, st, block, splits, snap, snap_rounds)


def rcpp(n, src, dst, pi0, max_supersteps=None, snap_rounds=0, threads=1,
         stop_after=-1) -> OracleResult:
    src, dst, pi0 = _i32(src), _i32(dst), _i32(pi0)
    guard = _DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 10 if max_supersteps is None else max(int(max_supersteps), 0) + 1
    block = np.empty(n, np.int32)
    splits = np.zeros(cap + 1, np.int32)
    snap = np.empty((snap_rounds, n), np.int32) if snap_rounds else None
    st = _Stats()
    rc = lib().oracle_rcpp(n, src.size, _ptr(src), _ptr(dst), _ptr(pi0), guard, _ptr(block),
                           _ptr(splits), cap, _ptr(snap) if snap is not None else None,
                           snap_rounds, stop_after, ctypes.byref(st), threads)
    return _finish(rc, st, block, splits, snap, snap_rounds)


class OracleRun:
    """Literal oracle with setup done once (timed once) and the main loop
    resumable from any reachable state: bench.py times windows of rounds from
    the start, middle and end of a run this way (see fast_states)."""

    def __init__(self, inst, threads: int):
        self.threads = threads
        self.bcrp = inst.kind == "bcrp"
        self.n = inst.n
        self._keep = [_i32(inst.src), _i32(inst.dst)]
        if self.bcrp:
            self._keep += [_i32(inst.act), None]
        else:
            self._keep += [None, _i32(inst.pi0)]
        src, dst, act, pi0 = self._keep
        st = _Stats()
        self.h = lib().oracle_open(int(self.bcrp), inst.n, src.size,
                                   inst.num_actions if self.bcrp else 0, _ptr(src),
                                   _ptr(act) if act is not None else None, _ptr(dst),
                                   _ptr(pi0) if pi0 is not None else None, threads,
                                   ctypes.byref(st))
        if not self.h:
            raise MemoryError("oracle_open failed")
        self.t_pre_s, self.t_label_s = st.t_pre_s, st.t_label_s
        self.initial_blocks = int(st.initial_blocks)

    def set_state(self, block: np.ndarray, unstable: np.ndarray):
        b = _i32(block)
        u = np.ascontiguousarray(unstable, dtype=np.uint8)
        lib().oracle_set_state(self.h, _ptr(b), u.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)))

    def rounds(self, k: int) -> tuple[int, float]:
        sec = ctypes.c_double(0.0)
        done = lib().oracle_rounds(self.h, int(k), self.threads, ctypes.byref(sec))
        return int(done), sec.value

    def block(self) -> np.ndarray:
        return np.ctypeslib.as_array(lib().oracle_block(self.h), shape=(self.n,)).copy()

    def close(self):
        if self.h:
            lib().oracle_close(self.h)
            self.h = None

    def __del__(self):
        self.close()


def fast_states(inst, stops, threads: int = 1):
    """(blocks[k, n], unstable[k, n]) of the reference program after each
    round in `stops` (ascending), from the event-driven oracle."""
    stops = np.ascontiguousarray(sorted(int(x) for x in stops), dtype=np.int64)
    k, n = stops.size, inst.n
    blocks = np.empty((k, n), np.int32)
    unstable = np.empty((k, n), np.uint8)
    bcrp = inst.kind == "bcrp"
    src, dst = _i32(inst.src), _i32(inst.dst)
    act = _i32(inst.act) if bcrp else None
    pi0 = None if bcrp else _i32(inst.pi0)
    rc = lib().oracle_fast_states(int(bcrp), n, src.size, inst.num_actions if bcrp else 0,
                                  _ptr(src), _ptr(act) if act is not None else None, _ptr(dst),
                                  _ptr(pi0) if pi0 is not None else None, k,
                                  stops.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  _ptr(blocks),
                                  unstable.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)),
                                  threads)
    if rc != OR_OK:
        raise RuntimeError(f"oracle_fast_states failed ({rc})")
    return blocks, unstable
