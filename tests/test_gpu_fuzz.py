"""Randomised parity of the CUDA path with the CPU oracle.

Shapes the fixed fixtures do not cover on their own: label counts around the
32 / 64-bit word boundaries of the label masks and slot vectors (|Act| 31..65,
200, 300: multi-word masks, slot runs longer than 32 bits), hubs with large
in-degree, duplicate transitions and self-loops, states without outgoing
transitions, RCPP with non-canonical pi0 leaders.  Every instance runs with
the default schedule and with a random combination of the schedule flags
(bisim.h BISIM_FLAG_*: forced wide / two-pass phase-B layouts, the batch
phase-A walk, no solo stretches, no bulk retirement, CTA-major placement) --
none may change a result.  The oracle (oracle/bisim_oracle.c) restates
bcrp.py:49-315 / rcpp.py:58-259 and is pinned to the reference in
test_oracle_golden.py.
"""
import numpy as np
import pytest

from oracle import oracle
from paper_2105_11788_b200 import _native as N
from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays

pytestmark = pytest.mark.gpu

FLAGS = [N.FLAG_NO_SKIP, N.FLAG_NO_SOLO, N.FLAG_CTA_MAJOR, N.FLAG_WIDE_LAYOUT, N.FLAG_TWO_PASS,
         N.FLAG_BATCH_WALK]


def _flags(g):
    f = 0
    for x in FLAGS:
        if g.random() < 0.4:
            f |= x
    return f


def _same(block, st, res, what):
    assert np.array_equal(block, res.block), what
    assert st.supersteps == res.supersteps, what
    assert np.array_equal(np.asarray(st.splits_per_iteration, np.int32), res.splits), what
    assert st.initial_block_count == res.initial_blocks, what
    assert st.final_block_count == res.final_blocks, what


def _bcrp_instance(g, k):
    A = [1, 2, 3, 5, 31, 32, 33, 63, 64, 65, 200, 300][k % 12]
    n = int(g.integers(1, 3000))
    m = int(g.integers(0, 6 * n + 1))
    src = g.integers(0, n, m, dtype=np.int32)
    dst = g.integers(0, n, m, dtype=np.int32)
    act = g.integers(0, A, m, dtype=np.int32)
    if m and k % 3 == 0:  # a hub: many in-edges on few states
        hot = g.integers(0, n, max(1, n // 100))
        sel = g.random(m) < 0.3
        dst[sel] = hot[g.integers(0, hot.size, int(sel.sum()))]
    if m and k % 4 == 1:  # duplicates and self-loops
        d = int(g.integers(1, m + 1))
        src = np.concatenate([src, src[:d]])
        dst = np.concatenate([dst, dst[:d]])
        act = np.concatenate([act, act[:d]])
        sl = g.random(src.size) < 0.05
        dst[sl] = src[sl]
    if m and k % 5 == 2:  # a third of the states without outgoing transitions
        keep = src % 3 != 0
        src, dst, act = src[keep], dst[keep], act[keep]
    return n, src, act, dst, A


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_bcrp_vs_oracle(seed):
    g = np.random.default_rng(1000 + seed)
    for k in range(24):
        n, src, act, dst, A = _bcrp_instance(g, k)
        res = oracle.bcrp(n, src, act, dst, A, threads=4)
        what = f"seed={seed} k={k} n={n} m={src.size} A={A}"
        block, st, _ = bcrp_arrays(n, src, act, dst, A)
        _same(block, st, res, what)
        f = _flags(g)
        block, st, _ = bcrp_arrays(n, src, act, dst, A, flags=f)
        _same(block, st, res, f"{what} flags={f}")
        if k % 6 == 0:
            block, st, _ = bcrp_arrays(n, src, act, dst, A, mode=N.MODE_DENSE)
            _same(block, st, res, what + " dense")


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_rcpp_vs_oracle(seed):
    g = np.random.default_rng(2000 + seed)
    for k in range(24):
        n = int(g.integers(1, 4000))
        m = int(g.integers(0, 5 * n + 1))
        src = g.integers(0, n, m, dtype=np.int32)
        dst = g.integers(0, n, m, dtype=np.int32)
        # pi0: a few initial blocks, leaders drawn anywhere in the block
        # (non-canonical: rcpp.py takes pi0 verbatim)
        nb = int(g.integers(1, 6))
        colour = g.integers(0, nb, n)
        pi0 = np.empty(n, np.int32)
        for c in range(nb):
            mem = np.nonzero(colour == c)[0]
            if mem.size:
                pi0[mem] = mem[g.integers(0, mem.size)]
        res = oracle.rcpp(n, src, dst, pi0, threads=4)
        what = f"seed={seed} k={k} n={n} m={m} blocks={nb}"
        block, st, _ = rcpp_arrays(n, src, dst, pi0)
        _same(block, st, res, what)
        f = _flags(g)
        block, st, _ = rcpp_arrays(n, src, dst, pi0, flags=f)
        _same(block, st, res, f"{what} flags={f}")


@pytest.mark.parametrize("flags", [N.FLAG_TWO_PASS | N.FLAG_NO_SOLO | N.FLAG_BATCH_WALK,
                                   N.FLAG_WIDE_LAYOUT | N.FLAG_NO_SOLO])
def test_forced_layouts_on_large_blocks(flags):
    """Blocks of thousands of members (a lifted quotient: every block of the
    coarsest partition has 400 copies) through the forced wide / two-pass
    phase-B layouts, against the oracle."""
    from paper_2105_11788_b200 import workloads as W
    inst = W.lifted_quotient(120000, 300, 16, 4, 3, 2, seed=5)
    res = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=8)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, flags=flags)
    _same(block, st, res, f"lifted flags={flags}")
    assert np.array_equal(block, inst.truth)
