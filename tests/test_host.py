"""CPU-only tests: boundary types mirror the reference's behaviour, the C-ABI
library loads and exports every symbol include/bisim.h declares, and the
product path fails loudly (no CPU fallback) without a CUDA device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2105_11788_b200 import (
    Lts,
    Partition,
    RelationInput,
    RunStats,
    Transition,
    block_count,
    discrete_partition,
    lts_from_labeled_edges,
    partition_from_assignment,
    partition_refines,
    partitions_equal,
    trivial_partition,
)
from paper_2105_11788_b200 import _native as N
from paper_2105_11788_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# ---------------------------------------------------------------- C ABI

def _declared_functions():
    text = open(os.path.join(ROOT, "include", "bisim.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bisim_\w+)\s*\(", text)) - {"bisim_observer_fn"})


def test_library_exports_every_declared_symbol():
    L = N.lib()
    declared = _declared_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), name
    assert set(N.EXPORTS) == set(declared)


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {N.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_stats_struct_layout_matches_header():
    # bisim_stats: 3 x i64, 2 x i32, i64, 5 x f64, i64, 2 x i32, i64 = 104 bytes
    assert ctypes.sizeof(N.Stats) == 104


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device error path")
def test_no_cpu_fallback_without_device():
    from paper_2105_11788_b200 import bcrp_arrays
    with pytest.raises(N.NativeError) as e:
        bcrp_arrays(3, [0], [0], [1], 1)
    assert e.value.code == N.BISIM_CUDA
    assert "no CUDA device" in str(e.value)


# ---------------------------------------------------------------- types

def test_lts_validation_matches_reference():
    with pytest.raises(ValueError):
        Lts(0, ("a",), [])
    with pytest.raises(ValueError):
        Lts(2, ("a", "a"), [])
    with pytest.raises(ValueError):
        Lts(2, ("a",), [(0, 0, 2)])
    with pytest.raises(ValueError):
        Lts(2, ("a",), [(0, 1, 1)])
    with pytest.raises(ValueError):
        Lts(2, ("a",), [], initial_state=2)
    with pytest.raises(ValueError):
        Lts.from_arrays(2, [0], [1], [1], 1)


def test_lts_from_labeled_edges_sorted_ids():
    lts = lts_from_labeled_edges(3, [(0, "b", 1), (1, "a", 2)], extra_labels=("c",))
    assert lts.action_labels == ("a", "b", "c")
    assert lts.transitions == (Transition(0, 1, 1), Transition(1, 0, 2))
    s, a, d = lts.columns()
    assert list(s) == [0, 1] and list(a) == [1, 0] and list(d) == [1, 2]
    arr = Lts.from_arrays(3, s, a, d, lts.action_labels)
    assert arr.transitions == lts.transitions and arr == lts and arr.m == 2


def test_partition_validation():
    with pytest.raises(ValueError):
        Partition([])
    with pytest.raises(ValueError):
        Partition([1, 2, 2])          # leader 1 is not its own leader
    with pytest.raises(ValueError):
        Partition([0, 5])
    with pytest.raises(ValueError):
        Partition(np.array([1, 0]))
    p = Partition([1, 1, 2])          # non-minimum leaders are allowed
    assert p.blocks() == {1: [0, 1], 2: [2]}
    assert Partition(np.array([0, 0, 2])) == Partition([0, 0, 2])


def test_partition_helpers():
    assert partition_from_assignment([9, 9, 4]).block == (0, 0, 2)
    assert partition_from_assignment([5, 3, 5, 3, 1]).block == (0, 1, 0, 1, 4)
    assert partitions_equal(Partition([1, 1, 2]), Partition([0, 0, 2]))
    assert not partitions_equal(Partition([0, 0, 2]), Partition([0, 1, 1]))
    assert partition_refines(discrete_partition(3), trivial_partition(3))
    assert not partition_refines(trivial_partition(3), discrete_partition(3))
    assert block_count(Partition([0, 0, 2])) == 2


def test_runstats_validation():
    with pytest.raises(ValueError):
        RunStats(2, (1,), 3, 1)
    with pytest.raises(ValueError):
        RunStats(1, (1,), 1, 2)
    RunStats(1, (0,), 1, 1)


def test_relation_input_validation():
    with pytest.raises(ValueError):
        RelationInput(2, ((0, 5),), trivial_partition(2))
    with pytest.raises(ValueError):
        RelationInput(2, (), trivial_partition(3))
    r = RelationInput(3, [(0, 1), [1, 2]], trivial_partition(3))
    assert r.edges == ((0, 1), (1, 2))
    s, d = r.columns()
    assert list(s) == [0, 1] and list(d) == [1, 2]


# ---------------------------------------------------------------- workloads

def test_lifted_quotient_truth_matches_oracle():
    from oracle import oracle
    inst = W.lifted_quotient(4000, 200, 24, templates=5, labels_per_template=4,
                             edges_per_label=2, seed=3)
    res = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=4)
    assert np.array_equal(res.block, inst.truth)
    assert W.is_stable(inst.n, inst.src, inst.act, inst.dst, inst.truth)


def test_signature_bisim_vs_oracle_random():
    from oracle import oracle
    g = np.random.default_rng(9)
    n, m = 800, 2400
    src, act, dst = (g.integers(0, n, m), g.integers(0, 3, m), g.integers(0, n, m))
    assert np.array_equal(W.signature_bisim(n, src, act, dst),
                          oracle.bcrp(n, src, act, dst, 3).block)


def test_fanout_matches_reference_generator():
    import _golden as G
    for n in (3, 10, 64):
        rec = G.cases()[f"fanout_{n}"]
        inst = W.fanout(n)
        # same multiset of transitions as cli.gen_fanout (order irrelevant)
        got = sorted(zip(inst.src.tolist(), inst.act.tolist(), inst.dst.tolist()))
        exp = sorted(zip(rec["src"], rec["act"], rec["dst"]))
        assert got == exp


def test_c1_generator_matches_reference_fixture():
    import _golden as G
    got = G.c1()
    if got is None:
        pytest.skip("c1 fixture not generated")
    _, z = got
    inst = W.c1_random()
    assert np.array_equal(inst.src, z["src"]) and np.array_equal(inst.act, z["act"])
    assert np.array_equal(inst.dst, z["dst"])
