"""Transition-sharded mode (csrc/kernels_shard.cuh).

One system, several replicas of the persistent kernel, in-edges split by
source range, marks OR-ed into every replica over peer memory each round.
On a one-GPU machine the replicas share device 0 (the device list repeats
it); the code path -- peer pointers, system-scope release/acquire barrier,
double-buffered round state -- is the multi-GPU one.  Results must be
bit-identical to the reference fixtures and to the single-replica run,
including RunStats, and every replica must end with the same partition.
"""
import numpy as np
import pytest

import _golden as G
from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays
from paper_2105_11788_b200 import workloads as W
from paper_2105_11788_b200.policy import SuperstepLimitError
from paper_2105_11788_b200.sharded import bcrp_sharded_arrays, rcpp_sharded_arrays

pytestmark = pytest.mark.gpu

SHARDS = [[0], [0, 0], [0, 0, 0], [0, 0, 0, 0]]


def _same(block, st, exp, what):
    assert list(block) == exp["block"], what
    assert st.supersteps == exp["supersteps"], what
    assert list(st.splits_per_iteration) == exp["splits"], what
    assert st.initial_block_count == exp["initial_blocks"], what
    assert st.final_block_count == exp["final_blocks"], what


@pytest.mark.parametrize("devices", SHARDS, ids=lambda d: f"x{len(d)}")
def test_sharded_medium_and_fanout_golden(devices):
    cases = G.cases()
    recs = [(f"medium_{i}", r) for i, r in enumerate(cases["medium_random"])]
    recs += [(k, cases[k]) for k in ("fanout_10", "fanout_64", "fanout_200", "chain_200",
                                     "edge_free_4", "pre_fig2")]
    for name, rec in recs:
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_sharded_arrays(n, src, act, dst, A, devices, verify=True)
        _same(block, st, rec["bcrp"], name)


@pytest.mark.parametrize("devices", SHARDS[:2], ids=lambda d: f"x{len(d)}")
def test_sharded_sweep_golden(devices):
    for idx, rec in enumerate(G.sweep()[:150]):
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_sharded_arrays(n, src, act, dst, A, devices, verify=True)
        _same(block, st, rec["bcrp"], f"sweep {idx}")
        if "rcpp_trivial" in rec:
            b2, st2, _ = rcpp_sharded_arrays(n, src, dst, np.zeros(n, np.int32), devices,
                                             verify=True)
            _same(b2, st2, rec["rcpp_trivial"], f"sweep rcpp {idx}")


def test_sharded_rcpp_noncanonical_golden():
    for idx, rec in enumerate(G.cases()["rcpp_noncanonical"]):
        n = rec["n"]
        block, st, _ = rcpp_sharded_arrays(n, rec["src"], rec["dst"], rec["pi0"], [0, 0],
                                           verify=True)
        _same(block, st, rec["rcpp"], f"noncanonical {idx}")


@pytest.mark.parametrize("devices", SHARDS, ids=lambda d: f"x{len(d)}")
def test_sharded_lifted_matches_single(devices):
    inst = W.lifted_quotient(200_000, 2000, 32, 6, 3, 2, seed=11)
    ref_block, ref_st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    block, st, ns = bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                        devices, verify=True)
    assert np.array_equal(block, inst.truth)
    assert np.array_equal(block, ref_block)
    assert st == ref_st
    assert ns["kernel_launches"] == len(devices)


def test_sharded_rcpp_kripke_matches_single():
    g = np.random.default_rng(3)
    n = 50_000
    src = np.repeat(np.arange(n, dtype=np.int32), 3)
    dst = g.integers(0, n, src.size).astype(np.int32)
    pi0 = W.canonical(g.integers(0, 4, n))
    ref = rcpp_arrays(n, src, dst, pi0)
    got = rcpp_sharded_arrays(n, src, dst, pi0, [0, 0, 0], verify=True)
    assert np.array_equal(got[0], ref[0]) and got[1] == ref[1]


def test_sharded_chain_round_count():
    inst = W.chain(3000)
    block, st, _ = bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                       [0, 0], verify=True)
    assert st.supersteps == 2 * 3000 - 2
    assert np.array_equal(block, np.arange(3000))


def test_sharded_guard():
    rec = G.cases()["fanout_12"]
    n, src, act, dst, A = G.arrays(rec)
    R = rec["bcrp"]["supersteps"]
    block, st, _ = bcrp_sharded_arrays(n, src, act, dst, A, [0, 0], max_supersteps=A + R + 1)
    assert st.supersteps == R
    with pytest.raises(SuperstepLimitError):
        bcrp_sharded_arrays(n, src, act, dst, A, [0, 0], max_supersteps=A + R)


def test_sharded_rejects_bad_shard_counts():
    z = np.zeros(1, np.int32)
    with pytest.raises(ValueError):
        bcrp_sharded_arrays(2, z, z, z, 1, [0] * 9)
    with pytest.raises(ValueError):
        bcrp_sharded_arrays(2, z, z, z, 1, [])


def _device_count():
    from paper_2105_11788_b200 import _native as N
    return int(N.lib().bisim_device_count())


@pytest.mark.parametrize("g", [2, 4, 8])
def test_sharded_distinct_devices(g):
    """The cross-device branch: peer access between distinct GPUs, the
    cooperative launch per device and the system-scope barrier over NVLink
    (capi.cu run_sharded).  Runs only on a machine with >= g GPUs."""
    if _device_count() < g:
        pytest.skip(f"needs {g} GPUs (this machine has {_device_count()})")
    devices = list(range(g))
    cases = G.cases()
    for name in ("fanout_64", "chain_200", "pre_fig2"):
        rec = cases[name]
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_sharded_arrays(n, src, act, dst, A, devices, verify=True)
        _same(block, st, rec["bcrp"], f"{name} x{g} devices")
    inst = W.lifted_quotient(400_000, 2000, 32, 6, 3, 2, seed=12)
    ref_block, ref_st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    block, st, _ = bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                       devices, verify=True)
    assert np.array_equal(block, inst.truth) and np.array_equal(block, ref_block)
    assert st == ref_st


def test_sharded_rejects_out_of_range_sources():
    with pytest.raises(ValueError):
        bcrp_sharded_arrays(3, [0, 5], [0, 0], [1, 2], 1, [0, 0])
    block, st, _ = bcrp_sharded_arrays(3, [0, 1], [0, 0], [1, 2], 1, [0, 0])
    assert list(block) == [0, 1, 2]
