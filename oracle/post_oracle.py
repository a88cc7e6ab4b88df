"""CPU restatement of the reference's quotient / stability / canonicaliser.

TEST INFRASTRUCTURE ONLY: the checker for paper_2105_11788_b200.post (the
GPU path); imported by tests/ only.  Pinned against fixtures made by the
unmodified reference (oracle/gen_golden.py post -> tests/golden/post.json.gz,
tests/test_oracle_golden.py).

    quotient            /root/reference/pkg/src/parbisim/aut.py:132-152
    is_stable           /root/reference/pkg/src/parbisim/oracle.py:128-141
    is_stable_under     /root/reference/pkg/src/parbisim/oracle.py:144-154
    canonical           /root/reference/pkg/src/parbisim/lts.py:117-128

numpy restatements of the same set algebra (first occurrences via
np.unique(return_index) instead of a Python set), so they finish at the
medium sizes the GPU parity tests use.
"""
from __future__ import annotations

import numpy as np


def _keys(*cols):
    """Row-wise structured keys for np.unique over several int columns."""
    arr = np.empty(len(cols[0]), dtype=[(f"f{k}", np.int64) for k in range(len(cols))])
    for k, c in enumerate(cols):
        arr[f"f{k}"] = c
    return arr


def quotient(n, src, act, dst, block, initial_state=0):
    """aut.py:132-152: leaders = sorted(set(block)) (:141), index = rank
    (:142); keep the first transition of every (index[block[s]], a,
    index[block[t]]) key in transition order (:143-149)."""
    block = np.asarray(block, np.int64)
    if block.size != n:
        raise ValueError("partition covers a different number of states")
    leaders = np.unique(block)
    index = np.full(n, -1, np.int64)
    index[leaders] = np.arange(leaders.size)
    src, act, dst = (np.asarray(x, np.int64) for x in (src, act, dst))
    qs, qd = index[block[src]], index[block[dst]]
    if src.size:
        _, first = np.unique(_keys(qs, act, qd), return_index=True)
        first.sort()
    else:
        first = np.zeros(0, np.int64)
    return (int(leaders.size), qs[first].astype(np.int32), act[first].astype(np.int32),
            qd[first].astype(np.int32), int(index[block[initial_state]]))


def is_stable(n, src, act, dst, block):
    """oracle.py:138-141: sigs[s] = {(a, block[t])}; stable iff sigs[s] ==
    sigs[block[s]] for every s."""
    block = np.asarray(block, np.int64)
    src, act, dst = (np.asarray(x, np.int64) for x in (src, act, dst))
    sig = np.unique(_keys(src, act, block[dst])) if src.size else _keys([], [], [])
    s, a, b = (sig[f"f{k}"] for k in range(3))
    cnt = np.bincount(s, minlength=n)
    if np.any(cnt != cnt[block]):
        return False
    # sig(s) within sig(block[s]); equal sizes then give equality
    lead = _keys(block[s], a, b)
    return bool(np.all(np.isin(lead, sig)))


def is_stable_under(n, src, act, dst, block, states):
    """oracle.py:144-154: reach[s] = {a : s -a-> t, t in states}; stable iff
    reach[s] == reach[block[s]] for every s."""
    block = np.asarray(block, np.int64)
    src, act, dst = (np.asarray(x, np.int64) for x in (src, act, dst))
    target = np.zeros(n, bool)
    st = np.asarray(list(states), np.int64)
    target[st[(st >= 0) & (st < n)]] = True
    sel = target[dst] if dst.size else np.zeros(0, bool)
    pairs = np.unique(_keys(src[sel], act[sel])) if sel.any() else _keys([], [])
    s_, a_ = pairs["f0"], pairs["f1"]
    cnt = np.bincount(s_, minlength=n)
    if np.any(cnt != cnt[block]):
        return False
    return bool(np.all(np.isin(_keys(block[s_], a_), pairs)))


def canonical(assignment):
    """lts.py:124-128: first_seen[v] = smallest index with value v."""
    arr = np.asarray(assignment, np.int64)
    _, first, inv = np.unique(arr, return_index=True, return_inverse=True)
    return first[inv.reshape(-1)].astype(np.int32)
