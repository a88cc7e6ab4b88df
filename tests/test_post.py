"""Quotient, stability check and canonicaliser.

CPU: the numpy restatement (oracle/post_oracle.py) against fixtures made by
the unmodified reference (quotient aut.py:132-152, is_stable
oracle.py:128-141, partition_from_assignment lts.py:117-128), plus the
reference's own known-answer tests for quotient (tests/test_aut.py:120-161).

GPU: libbisim.so's bisim_quotient / bisim_is_stable / bisim_canonical against
the same fixtures bit for bit, and against the oracle at sizes the fixtures
do not reach.
"""
import functools
import gzip
import json
import os

import numpy as np
import pytest

from oracle import post_oracle as PO

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def post_cases():
    with gzip.open(os.path.join(GOLDEN, "post.json.gz"), "rt") as fh:
        return json.load(fh)


def _arrays(rec):
    return (rec["n"], np.asarray(rec["src"], np.int32), np.asarray(rec["act"], np.int32),
            np.asarray(rec["dst"], np.int32), rec["num_actions"])


# ---------------------------------------------------------------- oracle (CPU)

def test_fixture_coverage():
    recs = post_cases()
    stable = [p["stable"] for r in recs for p in r["partitions"].values()]
    assert len(recs) >= 400
    assert any(stable) and not all(stable)  # both verdicts are pinned


def test_oracle_quotient_matches_reference_fixtures():
    for rec in post_cases():
        n, src, act, dst, _ = _arrays(rec)
        for name, p in rec["partitions"].items():
            qn, qs, qa, qd, qi = PO.quotient(n, src, act, dst, p["block"], rec["initial_state"])
            assert (qn, qi) == (p["q_n"], p["q_initial"]), name
            assert qs.tolist() == p["q_src"] and qa.tolist() == p["q_act"], name
            assert qd.tolist() == p["q_dst"], name


def test_oracle_is_stable_matches_reference_fixtures():
    for rec in post_cases():
        n, src, act, dst, _ = _arrays(rec)
        for name, p in rec["partitions"].items():
            assert PO.is_stable(n, src, act, dst, p["block"]) == p["stable"], name


def test_oracle_is_stable_under_matches_reference_fixtures():
    verdicts = []
    for rec in post_cases():
        n, src, act, dst, _ = _arrays(rec)
        for name, p in rec["partitions"].items():
            for sub, exp in p["under"]:
                assert PO.is_stable_under(n, src, act, dst, p["block"], sub) == exp, name
                verdicts.append(exp)
    assert any(verdicts) and not all(verdicts)


def test_oracle_canonical_matches_reference_fixtures():
    for rec in post_cases():
        assert PO.canonical(rec["assignment"]).tolist() == rec["canonical"]


def test_oracle_reference_known_answers():
    # tests/test_aut.py:120-147 of the reference
    # five-state relation, FIVE_STATE_FINAL = (0, 1, 2, 3, 3): 4 states, 4 transitions
    src, dst = [0, 1, 1, 2], [3, 4, 2, 1]
    qn, qs, qa, qd, qi = PO.quotient(5, src, [0] * 4, dst, [0, 1, 2, 3, 3])
    assert (qn, qs.size) == (4, 4)
    # discrete partition only removes duplicate transitions
    qn, qs, qa, qd, qi = PO.quotient(2, [0, 0, 1], [0, 0, 0], [1, 1, 0], [0, 1])
    assert (qn, qs.size) == (2, 2)
    # trivial partition collapses to self-loops, one per label
    qn, qs, qa, qd, qi = PO.quotient(3, [0, 1, 2], [0, 1, 0], [1, 2, 0], [0, 0, 0])
    assert qn == 1 and sorted(qa.tolist()) == [0, 1] and set(qs) == {0} and set(qd) == {0}
    # initial state follows its block
    assert PO.quotient(3, [1], [0], [2], [0, 1, 0], initial_state=2)[4] == 0


# ---------------------------------------------------------------- GPU parity

@pytest.mark.gpu
def test_gpu_quotient_matches_reference_fixtures():
    from paper_2105_11788_b200.post import quotient_arrays
    for rec in post_cases():
        n, src, act, dst, A = _arrays(rec)
        for name, p in rec["partitions"].items():
            qn, qs, qa, qd, qi = quotient_arrays(n, src, act, dst, A, p["block"],
                                                 rec["initial_state"])
            assert (qn, qi) == (p["q_n"], p["q_initial"]), name
            assert qs.tolist() == p["q_src"] and qa.tolist() == p["q_act"], name
            assert qd.tolist() == p["q_dst"], name


@pytest.mark.gpu
def test_gpu_is_stable_matches_reference_fixtures():
    from paper_2105_11788_b200.post import is_stable_arrays
    for rec in post_cases():
        n, src, act, dst, A = _arrays(rec)
        for name, p in rec["partitions"].items():
            assert is_stable_arrays(n, src, act, dst, A, p["block"]) == p["stable"], name


@pytest.mark.gpu
def test_gpu_is_stable_under_matches_reference_fixtures():
    from paper_2105_11788_b200.post import is_stable_under_arrays
    for rec in post_cases():
        n, src, act, dst, A = _arrays(rec)
        for name, p in rec["partitions"].items():
            for sub, exp in p["under"]:
                assert is_stable_under_arrays(n, src, act, dst, A, p["block"], sub) == exp, name


@pytest.mark.gpu
def test_gpu_canonical_matches_reference_fixtures():
    from paper_2105_11788_b200.post import canonical_arrays
    for rec in post_cases():
        assert canonical_arrays(rec["assignment"]).tolist() == rec["canonical"]


@pytest.mark.gpu
def test_gpu_reference_typed_wrappers():
    from paper_2105_11788_b200 import (Partition, lts_from_labeled_edges,
                                       partition_from_assignment, trivial_partition)
    from paper_2105_11788_b200.post import is_stable, quotient
    lts = lts_from_labeled_edges(3, [(0, "a", 1), (1, "b", 2), (2, "a", 0)])
    q = quotient(lts, trivial_partition(3))
    assert q.n == 1 and sorted(q.action_labels[t.action] for t in q.transitions) == ["a", "b"]
    lts2 = lts_from_labeled_edges(3, [(1, "a", 2)], initial_state=2)
    assert quotient(lts2, partition_from_assignment([0, 1, 0])).initial_state == 0
    with pytest.raises(ValueError):
        quotient(lts, Partition([0, 0]))
    assert is_stable(lts, Partition([0, 1, 2]))
    assert not is_stable(lts, Partition([0, 0, 2]))


@pytest.mark.gpu
def test_gpu_bad_partitions_rejected():
    from paper_2105_11788_b200.post import is_stable_arrays, quotient_arrays
    z = np.zeros(1, np.int32)
    with pytest.raises(ValueError):
        quotient_arrays(3, z, z, z, 1, [1, 1, 0])   # state 2 names 0, which is not self-led
    with pytest.raises(ValueError):
        is_stable_arrays(3, z, z, z, 1, [0, 5, 0])  # label out of range
    with pytest.raises(ValueError):
        quotient_arrays(2, np.array([0], np.int32), np.array([3], np.int32),
                        np.array([1], np.int32), 2, [0, 1])  # undeclared action


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_gpu_post_vs_oracle_medium(seed):
    """200k transitions, duplicate-heavy keys, against the numpy oracle."""
    from paper_2105_11788_b200.post import canonical_arrays, is_stable_arrays, quotient_arrays
    g = np.random.default_rng(seed)
    n, m, A = 20000, 200000, 5
    src = g.integers(0, n, m).astype(np.int32)
    act = g.integers(0, A, m).astype(np.int32)
    dst = g.integers(0, n, m).astype(np.int32)
    assign = g.integers(-50, 50, n) * 3
    block = PO.canonical(assign)
    assert np.array_equal(canonical_arrays(assign), block)
    got = quotient_arrays(n, src, act, dst, A, block, 7)
    exp = PO.quotient(n, src, act, dst, block, 7)
    assert got[0] == exp[0] and got[4] == exp[4]
    for x, y in zip(got[1:4], exp[1:4]):
        assert np.array_equal(x, y)
    assert is_stable_arrays(n, src, act, dst, A, block) == PO.is_stable(n, src, act, dst, block)
    assert is_stable_arrays(n, src, act, dst, A, np.arange(n)) is True
    from paper_2105_11788_b200.post import is_stable_under_arrays
    for sub in (np.nonzero(block == block[5])[0], g.choice(n, 5000, replace=False), [n + 3, -1]):
        assert (is_stable_under_arrays(n, src, act, dst, A, block, sub)
                == PO.is_stable_under(n, src, act, dst, block, sub))
    # a 70-label system: two mask words per state
    act70 = g.integers(0, 70, m).astype(np.int32)
    sub = g.choice(n, 3000, replace=False)
    for blk in (block, np.arange(n)):
        assert (is_stable_under_arrays(n, src, act70, dst, 70, blk, sub)
                == PO.is_stable_under(n, src, act70, dst, blk, sub))


@pytest.mark.gpu
@pytest.mark.parametrize("size", ["small", "full_c5"])
def test_gpu_coarsest_partition_is_stable(size):
    """The refinement result is stable, its quotient has exactly one state per
    block, and merging two blocks breaks stability (size-independent
    properties) -- on a small lifted system and on config c5 at full size
    (n=10M, m=100M)."""
    from paper_2105_11788_b200 import bcrp_arrays
    from paper_2105_11788_b200 import workloads as W
    from paper_2105_11788_b200.post import is_stable_arrays, quotient_arrays
    inst = (W.lifted_quotient(3000, 200, 64, 4, 2, 2, seed=5) if size == "small"
            else W.c5_vlts(seed=0))
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    assert np.array_equal(block, inst.truth)
    assert is_stable_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, block)
    qn, qs, qa, qd, _ = quotient_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                        block)
    assert qn == st.final_block_count
    # merging one more pair of blocks breaks stability
    leaders = np.unique(block)
    coarser = np.where(block == leaders[1], leaders[0], block).astype(np.int32)
    assert not is_stable_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, coarser)
