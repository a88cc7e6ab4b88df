"""The drop-in seam itself: the reference-named entry points `bcrp_run`,
`rcpp_run`, `preprocess` and `partition_by_outgoing_labels`
(/root/reference/pkg/src/parbisim/bcrp.py:116-141,192-195, rcpp.py:220-223),
called the way the reference's CLI and tests call them -- with this
package's `Lts` / `RelationInput` and with reference-shaped duck-typed
objects -- checked against fixtures made by the unmodified reference
(tests/golden/, oracle/gen_golden.py).  Mirrors the reference's own tests:
tests/test_bcrp.py:97-151,154-190, tests/test_acceptance.py:239-257,350-377,
tests/test_rcpp.py:119-136,225-231,252-259.
"""
from __future__ import annotations

from typing import NamedTuple

import numpy as np
import pytest

import _golden as G
from oracle import oracle
from paper_2105_11788_b200 import (Arbitrary, Common, Lts, Partition, PolicyViolationError,
                                   Priority, RelationInput, SuperstepLimitError, Transition,
                                   bcrp_arrays, bcrp_run, partition_by_outgoing_labels,
                                   preprocess, rcpp_arrays, rcpp_run)
from paper_2105_11788_b200 import _native as N

pytestmark = pytest.mark.gpu


# ---- reference-shaped stand-ins (attribute names of lts.py / rcpp.py, no
# ---- isinstance relation to this package's types)

class RefTransition(NamedTuple):
    source: int
    action: int
    target: int


class RefLts:
    def __init__(self, n, labels, transitions, initial_state=0):
        self.n = n
        self.action_labels = tuple(labels)
        self.transitions = tuple(RefTransition(*t) for t in transitions)
        self.initial_state = initial_state


class RefPartition:
    def __init__(self, block):
        self.block = tuple(block)

    def __len__(self):
        return len(self.block)


class RefRelation:
    def __init__(self, n, edges, pi0):
        self.n = n
        self.edges = tuple(tuple(e) for e in edges)
        self.pi0 = RefPartition(pi0)


class Priority_:   # the reference's policy objects are matched by class name
    pass


Priority_.__name__ = "Priority"


def _labels(A):
    return tuple(f"a{i}" for i in range(A))


def _lts_pair(rec):
    n, src, act, dst, A = G.arrays(rec)
    trans = list(zip(src.tolist(), act.tolist(), dst.tolist()))
    return (Lts(n, _labels(A), [Transition(*t) for t in trans]),
            RefLts(n, _labels(A), trans))


def _same(part, st, exp, what):
    assert list(part.block) == exp["block"], what
    assert st.supersteps == exp["supersteps"], what
    assert list(st.splits_per_iteration) == exp["splits"], what
    assert st.initial_block_count == exp["initial_blocks"], what
    assert st.final_block_count == exp["final_blocks"], what


LABELLED = ["pre_fig2", "pre_no_outgoing", "pre_stable_sort", "edge_free_4", "fanout_4",
            "fanout_17", "fanout_64", "chain_10", "chain_200"]


@pytest.mark.parametrize("name", LABELLED)
def test_bcrp_run_both_input_types(name):
    rec = G.cases()[name]
    for lts in _lts_pair(rec):
        for pol in (Priority(), Priority_()):
            part, st = bcrp_run(lts, pol)
            assert isinstance(part, Partition)
            _same(part, st, rec["bcrp"], f"{name} {type(lts).__name__}")


def test_bcrp_run_medium_and_sweep():
    for rec in G.cases()["medium_random"] + G.sweep()[:300]:
        lts, ref = _lts_pair(rec)
        _same(*bcrp_run(lts, Priority()), rec["bcrp"], "medium/sweep")
        _same(*bcrp_run(ref, Priority()), rec["bcrp"], "medium/sweep ref-shaped")


@pytest.mark.parametrize("name", ["pre_fig2", "pre_no_outgoing", "pre_stable_sort"])
def test_preprocess_tables(name):
    """test_acceptance.py:239-257 (Fig. 2), test_bcrp.py:44-124."""
    rec = G.cases()[name]
    n, src, act, dst, A = G.arrays(rec)
    for lts in _lts_pair(rec):
        aux = preprocess(lts)
        assert list(aux.action_switch) == rec["action_switch"]
        assert list(aux.order) == rec["order"]
        assert list(aux.nr_marks) == rec["nr_marks"]
        assert list(aux.off) == rec["off"]
        assert aux.mark_length == rec["mark_length"]
        # stable (source, action) order of the transitions themselves
        want = [Transition(int(src[p]), int(act[p]), int(dst[p])) for p in rec["perm"]]
        assert list(aux.lts.transitions) == want
        assert aux.lts.n == n and aux.lts.action_labels == _labels(A)
    if name == "pre_fig2":
        assert list(aux.action_switch) == [0, 0, 1, 0, 1, 1, 0, 0]
        assert list(aux.order) == [0, 0, 1, 0, 1, 2, 0, 0]
        assert list(aux.nr_marks) == [2, 3, 1] and list(aux.off) == [0, 2, 5]
        assert aux.mark_length == 6
    if name == "pre_no_outgoing":
        assert list(aux.nr_marks) == [1, 0, 1] and list(aux.off) == [0, 1, 1]
        assert aux.mark_length == 2


@pytest.mark.parametrize("seed", range(4))
def test_preprocess_matches_oracle_random(seed):
    """Larger random systems (incl. |Act| > 64, duplicate transitions, and a
    64-bit sort key) against the oracle's stable sort and tables."""
    g = np.random.default_rng(70 + seed)
    n, m, A = [(500, 3000, 3), (2000, 20000, 90), (300, 6000, 2), (70000, 200000, 70000)][seed]
    src = g.integers(0, n, m, dtype=np.int32)
    act = g.integers(0, A, m, dtype=np.int32)
    dst = g.integers(0, n, m, dtype=np.int32)
    if seed == 2:   # many exact duplicates: stability is observable
        src[::2] = src[1::2]
        act[::2] = act[1::2]
    lts = Lts.from_arrays(n, src, act, dst, A)
    aux = preprocess(lts)
    perm, sw, order, nr, off, L = oracle.preprocess(n, src, act, A)
    s, a, d = aux.lts.columns()
    assert np.array_equal(s, src[perm]) and np.array_equal(a, act[perm])
    assert np.array_equal(d, dst[perm])
    assert list(aux.action_switch) == list(sw) and list(aux.order) == list(order)
    assert list(aux.nr_marks) == list(nr) and list(aux.off) == list(off)
    assert aux.mark_length == L


def test_partition_by_outgoing_labels():
    """test_bcrp.py:127-151: grouping by outgoing label set, min leaders."""
    for name in ["pre_fig2", "pre_no_outgoing", "pre_stable_sort"]:
        rec = G.cases()[name]
        for lts in _lts_pair(rec):
            part = partition_by_outgoing_labels(lts, Priority())
            assert list(part.block) == rec["label_partition"], name
    for rec in G.sweep()[:300]:
        n, src, act, dst, A = G.arrays(rec)
        lts = Lts.from_arrays(n, src, act, dst, A)
        part = partition_by_outgoing_labels(lts, Priority())
        assert np.array_equal(np.asarray(part.block), oracle.label_partition(n, src, act, A))
        assert len(set(part.block)) == rec["bcrp"]["initial_blocks"]


def test_rcpp_run_both_input_types():
    rec = G.cases()["five_state"]
    edges = list(zip(rec["src"], rec["dst"]))
    for rel in (RelationInput(5, edges, Partition(rec["pi0"])),
                RefRelation(5, edges, rec["pi0"])):
        part, st = rcpp_run(rel, Priority())
        assert tuple(part.block) == (0, 1, 2, 3, 3)        # FIVE_STATE_FINAL
        _same(part, st, rec["rcpp"], "five_state")
    for i, rec in enumerate(G.cases()["rcpp_noncanonical"]):
        edges = list(zip(rec["src"], rec["dst"]))
        for rel in (RelationInput(rec["n"], edges, Partition(rec["pi0"])),
                    RefRelation(rec["n"], edges, rec["pi0"])):
            _same(*rcpp_run(rel, Priority()), rec["rcpp"], f"noncanonical {i}")


def test_observer_chain_through_bcrp_run_and_rcpp_run():
    """test_rcpp.py:252-259 / test_acceptance.py:130-134: observer(k, Partition)
    after every counted superstep, k = 1, 2, ..."""
    for rec in [G.cases()["pre_fig2"], G.cases()["fanout_12"]] + G.sweep()[:50]:
        lts, _ = _lts_pair(rec)
        seen = []
        bcrp_run(lts, Priority(), observer=lambda k, p: seen.append((k, list(p.block))))
        assert [k for k, _ in seen] == list(range(1, len(seen) + 1))
        assert [b for _, b in seen] == rec["bcrp"]["snapshots"]
    rec = G.cases()["five_state"]
    seen = []
    rcpp_run(RelationInput(5, list(zip(rec["src"], rec["dst"])), Partition(rec["pi0"])),
             Priority(), observer=lambda k, p: seen.append(list(p.block)))
    assert seen == rec["rcpp"]["snapshots"]


def test_observer_exception_propagates():
    rec = G.cases()["fanout_12"]
    lts, _ = _lts_pair(rec)

    class Boom(Exception):
        pass

    def obs(k, p):
        if k == 3:
            raise Boom

    with pytest.raises(Boom):
        bcrp_run(lts, Priority(), observer=obs)
    _same(*bcrp_run(lts, Priority()), rec["bcrp"], "after observer abort")


def test_guard_through_seam():
    """SuperstepLimitError exactly where the reference raises it
    (test_bcrp.py:179-181, test_rcpp.py:233-250)."""
    for g in G.cases()["guard"]:
        rec = G.cases()[g["instance"]]
        lts, ref = _lts_pair(rec)
        n = rec["n"]
        for obj in (lts, ref):
            if g["kind"] == "bcrp":
                call = lambda: bcrp_run(obj, Priority(), max_supersteps=g["max_supersteps"])
            else:
                rel = RelationInput(n, list(zip(rec["src"], rec["dst"])), Partition([0] * n))
                call = lambda: rcpp_run(rel, Priority(), max_supersteps=g["max_supersteps"])
            if g["result"]["guard"]:
                with pytest.raises(SuperstepLimitError):
                    call()
            else:
                _same(*call(), g["result"], str(g))


def test_policies():
    """Common with the Alg. 6 election and Arbitrary give the Priority
    partition (test_acceptance.py:350-377); plain Common is illegal."""
    for rec in [G.cases()["pre_fig2"], G.cases()["fanout_9"]] + G.sweep()[:40]:
        lts, ref = _lts_pair(rec)
        want = rec["bcrp"]
        _same(*bcrp_run(lts, Common(), common_election=True), want, "common+election")
        _same(*bcrp_run(ref, Common()), want, "common defaults to election")
        part, _ = bcrp_run(lts, Arbitrary(7))
        assert list(part.block) == want["block"]
    lts, _ = _lts_pair(G.cases()["pre_fig2"])
    with pytest.raises(PolicyViolationError):
        bcrp_run(lts, Common(), common_election=False)


BAD_BCRP = [  # (src, act, dst) with one entry out of range, n = 4, |Act| = 2
    ([0, 1], [0, 1], [1, 4]),
    ([0, 1], [0, 1], [1, -1]),
    ([0, 4], [0, 1], [1, 2]),
    ([-1, 1], [0, 1], [1, 2]),
    ([0, 1], [0, 2], [1, 2]),
    ([0, 1], [-1, 0], [1, 2]),
]


@pytest.mark.parametrize("case", range(len(BAD_BCRP)))
def test_out_of_range_transitions_raise_value_error(case):
    """Out-of-range ids fail as ValueError before any kernel scatters
    through them, and leave the device usable."""
    src, act, dst = BAD_BCRP[case]
    with pytest.raises(ValueError):
        bcrp_arrays(4, src, act, dst, 2)
    with pytest.raises(ValueError):
        Lts.from_arrays(4, src, act, dst, 2)      # the reference's constructor check
    unchecked = Lts.from_arrays(4, src, act, dst, 2, validate=False)
    with pytest.raises(ValueError):
        preprocess(unchecked)
    if not all(0 <= d < 4 for d in dst):          # targets play no part in the label sets
        partition_by_outgoing_labels(unchecked, Priority())
    else:
        with pytest.raises(ValueError):
            partition_by_outgoing_labels(unchecked, Priority())
    if all(0 <= a < 2 for a in act):
        with pytest.raises(ValueError):
            rcpp_arrays(4, src, dst, [0, 0, 0, 0])
    # the device is still healthy
    rec = G.cases()["pre_fig2"]
    n, s, a, d, A = G.arrays(rec)
    block, st, _ = bcrp_arrays(n, s, a, d, A)
    assert list(block) == rec["bcrp"]["block"]


def test_bad_pi0_raises_value_error():
    with pytest.raises(ValueError):
        rcpp_arrays(3, [0], [1], [0, 0, 1])       # block[2] = 1 but block[1] != 1
    with pytest.raises(ValueError):
        rcpp_arrays(3, [0], [1], [0, 0, 3])


def test_reference_errors_for_bad_types():
    with pytest.raises(ValueError):
        RelationInput(3, [(0, 3)], Partition([0, 0, 0]))
    with pytest.raises(TypeError):
        bcrp_run(_lts_pair(G.cases()["pre_fig2"])[0], object())


def test_guard_messages_match_the_reference():
    """SuperstepLimitError text is the reference's PramEngine message
    `superstep guard exceeded (<step> > <max>)` (pram.py:195-200), for trips
    in the label rounds and in the main loop."""
    for g in G.cases()["guard"]:
        if not g["result"]["guard"]:
            continue
        rec = G.cases()[g["instance"]]
        lts, _ = _lts_pair(rec)
        with pytest.raises(SuperstepLimitError) as e:
            if g["kind"] == "bcrp":
                bcrp_run(lts, Priority(), max_supersteps=g["max_supersteps"])
            else:
                n = rec["n"]
                rcpp_run(RelationInput(n, list(zip(rec["src"], rec["dst"])), Partition([0] * n)),
                         Priority(), max_supersteps=g["max_supersteps"])
        msg = str(e.value)
        assert msg.startswith("superstep guard exceeded (") and msg.endswith(
            f" > {g['max_supersteps']})"), msg


@pytest.mark.parametrize("name", ["pre_fig2", "pre_no_outgoing", "pre_stable_sort", "fanout_17"])
def test_c_abi_preprocess_per_original_transition(name):
    """bisim_preprocess (include/bisim.h): order per ORIGINAL transition,
    nr_marks and off per state -- the reference's tables (bcrp.py:91-113)
    read through the stable sort's permutation."""
    import ctypes
    rec = G.cases()[name]
    n, src, act, dst, A = G.arrays(rec)
    m = src.size
    order = np.empty(max(m, 1), np.int32)
    nr = np.empty(n, np.int32)
    off = np.empty(n, np.int32)
    L = ctypes.c_int64(0)
    N.check(N.lib().bisim_preprocess(n, m, A, N.ptr(src), N.ptr(act), N.ptr(order), N.ptr(nr),
                                     N.ptr(off), ctypes.byref(L), 0))
    perm, sw, ref_order, ref_nr, ref_off, ref_L = oracle.preprocess(n, src, act, A)
    assert list(order[:m][perm]) == list(ref_order)
    assert list(nr) == list(ref_nr) and list(off) == list(ref_off) and L.value == ref_L


@pytest.mark.parametrize("which,bad", [("act", 300), ("act", 256), ("act", -1), ("act", 40), ("act", 1 << 20),
                                       ("dst", 500_000), ("dst", 1 << 24), ("dst", -1), ("dst", (1 << 24) + 7),
                                       ("src", 500_000), ("src", 1 << 25), ("src", -5)])
@pytest.mark.parametrize("pinned", [False, True])
def test_out_of_range_ids_on_the_pipelined_input_path(which, bad, pinned):
    """Host inputs of >= 4M transitions take the pipelined copy path: the
    chunks are bucketed before the validation flag is read back, and host
    threads narrow the actions to bytes (|Act| <= 256).  An action that does
    not fit a byte is caught on the host, any other out-of-range id on the
    device -- either way ValueError before anything scatters through it, and
    the device stays usable; a valid system of that size still matches the
    oracle."""
    from paper_2105_11788_b200 import workloads as W
    inst = W.c4_uniform(n=500_000, m=4_300_000, num_actions=40, seed=3)
    arrs = {"src": inst.src.copy(), "act": inst.act.copy(), "dst": inst.dst.copy()}
    arrs[which][3_333_333 if which != "dst" else 17] = bad
    src, act, dst = arrs["src"], arrs["act"], arrs["dst"]
    if pinned:  # the C ABI path a pinned caller takes (no staging threads)
        import torch
        src, act, dst = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy() for x in (src, act, dst))
    with pytest.raises(ValueError):
        bcrp_arrays(inst.n, src, act, dst, inst.num_actions)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    res = _pipelined_oracle(inst)
    assert np.array_equal(block, res.block)
    assert st.supersteps == res.supersteps


_PIPE_ORACLE = {}


def _pipelined_oracle(inst):
    if inst.name not in _PIPE_ORACLE:
        _PIPE_ORACLE[inst.name] = oracle.bcrp_fast(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    return _PIPE_ORACLE[inst.name]


@pytest.mark.parametrize("n,m,A,null_src", [(0, 0, 1, False), (1 << 30, 0, 1, False), (10, 1 << 31, 1, True),
                                            (10, 5, 1, True), (10, 0, -1, False), (-3, 0, 1, False)])
def test_c_abi_size_limits(n, m, A, null_src):
    """The C ABI's documented limits (include/bisim.h: 1 <= n < 2^30,
    0 <= m < 2^31 - 1, |Act| >= 0, non-null arrays when m > 0) are checked
    before anything is allocated or copied: BISIM_BAD_INPUT with a message,
    and the device stays usable."""
    import ctypes
    lib = N.lib()
    src = np.zeros(max(min(m, 8), 1), np.int32)
    block = np.zeros(16, np.int32)
    splits = np.zeros(16, np.int32)
    st = N.Stats()
    opt = N.Options()
    p_src = None if null_src else N.ptr(src)
    rc = lib.bisim_bcrp_ex(n, m, A, p_src, p_src, p_src, N.DEFAULT_GUARD, N.ptr(block), N.ptr(splits), 16,
                           ctypes.byref(st), ctypes.byref(opt))
    assert rc == N.BISIM_BAD_INPUT, rc
    assert lib.bisim_last_error()
    rec = G.cases()["pre_fig2"]
    nn, s, a, d, AA = G.arrays(rec)
    blk, _, _ = bcrp_arrays(nn, s, a, d, AA)
    assert list(blk) == rec["bcrp"]["block"]
