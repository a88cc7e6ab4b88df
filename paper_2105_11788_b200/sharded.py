"""Transition-sharded refinement of ONE system over several GPUs.

``bcrp_sharded_arrays`` / ``rcpp_sharded_arrays`` take the same columns as
:func:`bcrp_arrays` / :func:`rcpp_arrays` plus a device list; every device
runs a replica of the persistent refinement kernel over the in-edges whose
source falls in its range, and the replicas OR their per-round marks into
each other's memory over NVLink (csrc/kernels_shard.cuh).  Results and
RunStats are identical to the single-GPU call.  A device may be listed more
than once: several replicas then share that GPU (how the mode is tested on a
one-GPU machine).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .lts import RunStats


def _raise(rc: int):
    if rc == N.BISIM_OK:
        return
    msg = N.last_error()
    if rc == N.BISIM_GUARD:
        from .policy import SuperstepLimitError
        raise SuperstepLimitError(msg)
    if rc == N.BISIM_BAD_INPUT:
        raise ValueError(msg)
    raise N.NativeError(rc, msg)


def _finish(n, block, splits, st):
    R = int(st.supersteps)
    stats = RunStats(supersteps=R, splits_per_iteration=tuple(splits[:R].tolist()),
                     final_block_count=int(st.final_blocks),
                     initial_block_count=int(st.initial_blocks))
    return block, stats, st.as_dict()


def bcrp_sharded_arrays(n: int, src, act, dst, num_actions: int, devices, *,
                        max_supersteps: int | None = None, verify: bool = False):
    src, act, dst = N.as_i32(src), N.as_i32(act), N.as_i32(dst)
    dev = N.as_i32(devices)
    guard = N.DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 16
    block = np.empty(n, np.int32)
    splits = np.zeros(cap, np.int32)
    st = N.Stats()
    _raise(N.lib().bisim_bcrp_sharded(n, src.size, int(num_actions), N.ptr(src), N.ptr(act),
                                      N.ptr(dst), guard, N.ptr(block), N.ptr(splits), cap,
                                      ctypes.byref(st), N.ptr(dev), dev.size,
                                      N.SHARD_VERIFY if verify else 0))
    return _finish(n, block, splits, st)


def rcpp_sharded_arrays(n: int, src, dst, pi0, devices, *, max_supersteps: int | None = None,
                        verify: bool = False):
    src, dst, pi0 = N.as_i32(src), N.as_i32(dst), N.as_i32(pi0)
    dev = N.as_i32(devices)
    guard = N.DEFAULT_GUARD if max_supersteps is None else int(max_supersteps)
    cap = 3 * n + 16
    block = np.empty(n, np.int32)
    splits = np.zeros(cap, np.int32)
    st = N.Stats()
    _raise(N.lib().bisim_rcpp_sharded(n, src.size, N.ptr(src), N.ptr(dst), N.ptr(pi0), guard,
                                      N.ptr(block), N.ptr(splits), cap, ctypes.byref(st),
                                      N.ptr(dev), dev.size, N.SHARD_VERIFY if verify else 0))
    return _finish(n, block, splits, st)


__all__ = ["bcrp_sharded_arrays", "rcpp_sharded_arrays"]
