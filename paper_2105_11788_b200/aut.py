""".aut ingestion and the quotient system.

Drop-in for the reading side of /root/reference/pkg/src/parbisim/aut.py:
:func:`parse_aut` accepts the same texts, returns the same :class:`Lts`
(action ids = ranks of the sorted label strings, lts.py:69-70) and raises
the same :class:`ParseError` messages and line numbers (aut.py:20-28,
:37-92).  The parsing runs in libbisim.so (``bisim_aut_parse``,
multi-threaded C++, csrc/aut.cpp); :func:`read_aut` maps a file directly and
returns an array-backed :class:`Lts`, so VLTS-size inputs never become
Python objects.  :func:`quotient` (aut.py:132-152) runs on the GPU
(paper_2105_11788_b200.post).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _native as N
from .lts import Lts
from .post import quotient  # noqa: F401  (aut.py:132-152 lives beside parse_aut upstream)


class ParseError(ValueError):
    """Malformed .aut text; carries the 1-based line number (aut.py:20-28)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


def _result(rc: int, handle, info) -> Lts:
    L = N.lib()
    if rc == N.BISIM_BAD_INPUT:
        line = int(info.error_line)
        raise ParseError(N.last_error(), line if line > 0 else None)
    N.check(rc)
    try:
        m = int(info.m)
        cols = [np.empty(m, np.int32) for _ in range(3)]
        N.check(L.bisim_aut_columns(handle, *(N.ptr(c) for c in cols)))
        labels = []
        ln = ctypes.c_int64(0)
        for a in range(int(info.num_actions)):
            p = L.bisim_aut_label(handle, a, ctypes.byref(ln))
            labels.append(ctypes.string_at(p, ln.value).decode("utf-8", "surrogatepass"))
    finally:
        L.bisim_aut_free(handle)
    return Lts.from_arrays(int(info.n), cols[0], cols[1], cols[2], tuple(labels),
                           int(info.initial_state), validate=False)


def parse_aut(text: str, threads: int = 0) -> Lts:
    """Parse Aldebaran text (aut.py:79-92)."""
    data = text.encode("utf-8", "surrogatepass")
    handle = ctypes.c_void_p()
    info = N.AutInfo()
    rc = N.lib().bisim_aut_parse(data, len(data), int(threads), ctypes.byref(handle),
                                 ctypes.byref(info))
    return _result(rc, handle, info)


def read_aut(path: str | os.PathLike, threads: int = 0) -> Lts:
    """Parse a .aut file (memory-mapped, UTF-8) into an array-backed Lts."""
    handle = ctypes.c_void_p()
    info = N.AutInfo()
    rc = N.lib().bisim_aut_read_file(os.fsencode(path), int(threads), ctypes.byref(handle),
                                     ctypes.byref(info))
    return _result(rc, handle, info)


__all__ = ["ParseError", "parse_aut", "read_aut", "quotient"]
