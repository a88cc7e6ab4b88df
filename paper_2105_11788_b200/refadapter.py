"""Drop-in adapter: run an installed reference package's refinement path on
the B200.

    import parbisim
    from paper_2105_11788_b200 import refadapter
    refadapter.install(parbisim)      # parbisim's CLI and API now use libbisim.so
    ...
    refadapter.uninstall(parbisim)

The reference exposes the path as module attributes that its CLI calls and
its tests swap (cli.py:97-119, 148-218; tests/test_cli.py:210).  install()
replaces `bcrp_run`, `rcpp_run`, `partition_by_outgoing_labels` and
`preprocess` in `parbisim`, `parbisim.bcrp`, `parbisim.rcpp` and
`parbisim.cli` with wrappers that take and return the reference's OWN types
(`Lts`, `RelationInput`, `Partition`, `RunStats`, `BcrpAux`) and raise its
OWN exception classes, so callers cannot tell the difference except by
speed.  Nothing here computes anything: the work is the CUDA path behind
this package's `bcrp_run` / `rcpp_run` / ... .
"""
from __future__ import annotations

import functools

from . import bcrp as _bcrp
from . import rcpp as _rcpp
from .policy import PolicyViolationError, SuperstepLimitError

_NAMES = ("bcrp_run", "rcpp_run", "partition_by_outgoing_labels", "preprocess")
_SAVED_ATTR = "_b200_saved"


def _ref_error(ref, e):
    """This package's exception -> the reference's class (same message)."""
    if isinstance(e, SuperstepLimitError):
        return ref.SuperstepLimitError(str(e))
    if isinstance(e, PolicyViolationError):
        return ref.PolicyViolationError(e.address, e.values)
    return e


def _wrap_observer(ref, observer):
    if observer is None:
        return None
    return lambda k, part: observer(k, ref.Partition(tuple(int(b) for b in part.block)))


def _ref_result(ref, part, stats):
    return (ref.Partition(tuple(int(b) for b in part.block)),
            ref.RunStats(supersteps=stats.supersteps,
                         splits_per_iteration=tuple(stats.splits_per_iteration),
                         final_block_count=stats.final_block_count,
                         initial_block_count=stats.initial_block_count))


def make(ref):
    """The four drop-in functions for reference package module `ref`."""

    def bcrp_run(lts, policy, *, common_election=None, observer=None, max_supersteps=None):
        try:
            out = _bcrp.bcrp_run(lts, policy, common_election=common_election,
                                 observer=_wrap_observer(ref, observer),
                                 max_supersteps=max_supersteps)
        except (SuperstepLimitError, PolicyViolationError) as e:
            raise _ref_error(ref, e) from None
        return _ref_result(ref, *out)

    def rcpp_run(rel, policy, *, common_election=None, observer=None, max_supersteps=None):
        try:
            out = _rcpp.rcpp_run(rel, policy, common_election=common_election,
                                 observer=_wrap_observer(ref, observer),
                                 max_supersteps=max_supersteps)
        except (SuperstepLimitError, PolicyViolationError) as e:
            raise _ref_error(ref, e) from None
        return _ref_result(ref, *out)

    def partition_by_outgoing_labels(lts, policy, *, common_election=None):
        try:
            part = _bcrp.partition_by_outgoing_labels(lts, policy, common_election=common_election)
        except PolicyViolationError as e:
            raise _ref_error(ref, e) from None
        return ref.Partition(tuple(int(b) for b in part.block))

    def preprocess(lts):
        aux = _bcrp.preprocess(lts)
        s, a, d = aux.lts.columns()
        sorted_lts = ref.Lts(n=lts.n, action_labels=tuple(lts.action_labels),
                             transitions=tuple(ref.Transition(int(x), int(y), int(z))
                                               for x, y, z in zip(s.tolist(), a.tolist(),
                                                                  d.tolist())),
                             initial_state=getattr(lts, "initial_state", 0))
        return ref.BcrpAux(lts=sorted_lts, action_switch=aux.action_switch, order=aux.order,
                           nr_marks=aux.nr_marks, off=aux.off, mark_length=aux.mark_length)

    funcs = {"bcrp_run": bcrp_run, "rcpp_run": rcpp_run,
             "partition_by_outgoing_labels": partition_by_outgoing_labels,
             "preprocess": preprocess}
    for name, f in funcs.items():
        functools.update_wrapper(f, getattr(ref, name))
    return funcs


def _modules(ref):
    import importlib
    mods = [ref]
    for sub in ("bcrp", "rcpp", "cli"):
        try:
            mods.append(importlib.import_module(f"{ref.__name__}.{sub}"))
        except ImportError:
            pass
    return mods


def install(ref) -> None:
    """Route the reference package's refinement path through libbisim.so."""
    if getattr(ref, _SAVED_ATTR, None) is not None:
        return
    funcs = make(ref)
    saved = []
    for mod in _modules(ref):
        for name in _NAMES:
            if hasattr(mod, name):
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, funcs[name])
    setattr(ref, _SAVED_ATTR, saved)


def uninstall(ref) -> None:
    """Restore the reference package's own functions."""
    saved = getattr(ref, _SAVED_ATTR, None)
    if saved is None:
        return
    for mod, name, f in saved:
        setattr(mod, name, f)
    setattr(ref, _SAVED_ATTR, None)


__all__ = ["install", "make", "uninstall"]
