"""Loaders for the committed golden fixtures (made by oracle/gen_golden.py
from the unmodified reference)."""
from __future__ import annotations

import functools
import gzip
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def cases() -> dict:
    with gzip.open(os.path.join(GOLDEN, "cases.json.gz"), "rt") as fh:
        return json.load(fh)


@functools.lru_cache(maxsize=None)
def sweep() -> list:
    with gzip.open(os.path.join(GOLDEN, "sweep.json.gz"), "rt") as fh:
        return json.load(fh)


def c1():
    path = os.path.join(GOLDEN, "c1_reference.npz")
    if not os.path.exists(path):
        return None
    with open(os.path.join(GOLDEN, "c1_reference.json")) as fh:
        meta = json.load(fh)
    z = np.load(path)
    return meta, {k: z[k] for k in z.files}


def arrays(rec):
    src = np.asarray(rec["src"], np.int32)
    dst = np.asarray(rec["dst"], np.int32)
    act = np.asarray(rec.get("act", [0] * len(rec["src"])), np.int32)
    return rec["n"], src, act, dst, rec.get("num_actions", 1)
