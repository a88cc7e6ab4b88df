"""Parity of the CUDA path (libbisim.so through the C ABI) with the reference.

Bit-exact comparisons: block arrays (leader form), supersteps,
splits_per_iteration, initial/final block counts, per-round observer
snapshots, guard behaviour.  Small cases compare against fixtures made by
the unmodified reference (tests/golden/); larger ones against the CPU oracle
(oracle/bisim_oracle.c, itself pinned to the reference in
test_oracle_golden.py); full-size configs through exact properties
(lifted-quotient ground truth, chain round counts, stability).
"""
import numpy as np
import pytest

import _golden as G
from oracle import oracle
import functools

from paper_2105_11788_b200 import _native as N
from paper_2105_11788_b200 import bcrp_arrays as _bcrp_arrays
from paper_2105_11788_b200 import rcpp_arrays as _rcpp_arrays
from paper_2105_11788_b200 import workloads as W
from paper_2105_11788_b200.policy import SuperstepLimitError

pytestmark = pytest.mark.gpu

MODES = {"sparse": N.MODE_AUTO, "dense": N.MODE_DENSE}
bcrp_arrays = rcpp_arrays = None  # bound per test by the `mode` fixture


@pytest.fixture(params=list(MODES), autouse=True)
def mode(request):
    """Every parity test runs against both refinement loops."""
    global bcrp_arrays, rcpp_arrays
    m = MODES[request.param]
    bcrp_arrays = functools.partial(_bcrp_arrays, mode=m)
    rcpp_arrays = functools.partial(_rcpp_arrays, mode=m)
    yield request.param


def _same(block, stats, exp, what):
    assert list(block) == exp["block"], what
    assert stats.supersteps == exp["supersteps"], what
    assert list(stats.splits_per_iteration) == exp["splits"], what
    assert stats.initial_block_count == exp["initial_blocks"], what
    assert stats.final_block_count == exp["final_blocks"], what


def _same_oracle(block, stats, res, what):
    assert np.array_equal(block, res.block), what
    assert stats.supersteps == res.supersteps, what
    assert np.array_equal(np.asarray(stats.splits_per_iteration, np.int32), res.splits), what
    assert stats.initial_block_count == res.initial_blocks, what
    assert stats.final_block_count == res.final_blocks, what


class Recorder:
    def __init__(self):
        self.chain = []

    def __call__(self, k, part):
        assert k == len(self.chain) + 1
        self.chain.append(list(part.block))


# ---------------------------------------------------------------- golden

@pytest.mark.parametrize("name", ["pre_fig2", "pre_no_outgoing", "pre_stable_sort"])
def test_small_labelled_golden(name):
    rec = G.cases()[name]
    n, src, act, dst, A = G.arrays(rec)
    block, st, _ = bcrp_arrays(n, src, act, dst, A)
    _same(block, st, rec["bcrp"], name)
    rec_obs = Recorder()
    block2, st2, _ = bcrp_arrays(n, src, act, dst, A, observer=rec_obs)
    _same(block2, st2, rec["bcrp"], name + " stepped")
    assert rec_obs.chain == rec["bcrp"]["snapshots"]


def test_five_state_golden():
    rec = G.cases()["five_state"]
    obs = Recorder()
    block, st, _ = rcpp_arrays(5, rec["src"], rec["dst"], rec["pi0"], observer=obs)
    assert tuple(block) == (0, 1, 2, 3, 3)          # FIVE_STATE_FINAL
    _same(block, st, rec["rcpp"], "five_state")
    assert obs.chain == rec["rcpp"]["snapshots"]
    block, st, _ = rcpp_arrays(5, rec["src"], rec["dst"], rec["pi0"])
    _same(block, st, rec["rcpp"], "five_state persistent")


def test_edge_free():
    rec = G.cases()["edge_free_4"]
    n, src, act, dst, A = G.arrays(rec)
    block, st, _ = rcpp_arrays(n, src, dst, [0] * n)
    assert st.supersteps == 1 and st.splits_per_iteration == (0,)
    _same(block, st, rec["rcpp_trivial"], "edge-free rcpp")
    block, st, _ = bcrp_arrays(n, src, act, dst, A)
    _same(block, st, rec["bcrp"], "edge-free bcrp")


@pytest.mark.parametrize("n", list(range(3, 65)) + [100, 200])
def test_fanout_family(n):
    rec = G.cases()[f"fanout_{n}"]
    nn, src, act, dst, A = G.arrays(rec)
    block, st, _ = bcrp_arrays(nn, src, act, dst, A)
    _same(block, st, rec["bcrp"], f"fanout {n}")
    block, st, _ = rcpp_arrays(nn, src, dst, [0] * nn)
    _same(block, st, rec["rcpp_trivial"], f"fanout {n} rcpp")
    if rec["bcrp"].get("snapshots") is not None:
        obs = Recorder()
        bcrp_arrays(nn, src, act, dst, A, observer=obs)
        assert obs.chain == rec["bcrp"]["snapshots"]


@pytest.mark.parametrize("n", [2, 3, 10, 100, 200])
def test_chain_golden(n):
    rec = G.cases()[f"chain_{n}"]
    nn, src, act, dst, A = G.arrays(rec)
    block, st, _ = bcrp_arrays(nn, src, act, dst, A)
    _same(block, st, rec["bcrp"], f"chain {n}")
    block, st, _ = rcpp_arrays(nn, src, dst, [0] * nn)
    _same(block, st, rec["rcpp_trivial"], f"chain {n} rcpp")


def test_guard_boundaries():
    for g in G.cases()["guard"]:
        rec = G.cases()[g["instance"]]
        n, src, act, dst, A = G.arrays(rec)
        exp = g["result"]
        try:
            if g["kind"] == "bcrp":
                block, st, _ = bcrp_arrays(n, src, act, dst, A, max_supersteps=g["max_supersteps"])
            else:
                block, st, _ = rcpp_arrays(n, src, dst, [0] * n, max_supersteps=g["max_supersteps"])
        except SuperstepLimitError:
            assert exp["guard"], g
            continue
        assert not exp["guard"], g
        _same(block, st, exp, str(g))


def test_rcpp_noncanonical_pi0():
    for i, rec in enumerate(G.cases()["rcpp_noncanonical"]):
        obs = Recorder()
        block, st, _ = rcpp_arrays(rec["n"], rec["src"], rec["dst"], rec["pi0"], observer=obs)
        _same(block, st, rec["rcpp"], f"noncanonical {i}")
        assert obs.chain == rec["rcpp"]["snapshots"]
        block, st, _ = rcpp_arrays(rec["n"], rec["src"], rec["dst"], rec["pi0"])
        _same(block, st, rec["rcpp"], f"noncanonical {i} persistent")


def test_medium_random_golden():
    for i, rec in enumerate(G.cases()["medium_random"]):
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_arrays(n, src, act, dst, A)
        _same(block, st, rec["bcrp"], f"medium {i}")


def test_acceptance_sweep():
    """The reference acceptance sweep's 1000 instances (test_acceptance.py:114-195)."""
    for rec in G.sweep():
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_arrays(n, src, act, dst, A)
        _same(block, st, rec["bcrp"], f"seed {rec['seed']}")
        if "rcpp_trivial" in rec:
            block, st, _ = rcpp_arrays(n, src, dst, [0] * n)
            _same(block, st, rec["rcpp_trivial"], f"seed {rec['seed']} rcpp")


def test_acceptance_sweep_observer_chains():
    for rec in G.sweep()[:200]:
        n, src, act, dst, A = G.arrays(rec)
        obs = Recorder()
        bcrp_arrays(n, src, act, dst, A, observer=obs)
        assert obs.chain == rec["bcrp"]["snapshots"], rec["seed"]


def test_c1_full_reference_run():
    """Config c1 (n=10k, m=50k, |Act|=4): the reference's own 2009 s run."""
    got = G.c1()
    if got is None:
        pytest.skip("c1 fixture not generated")
    meta, z = got
    block, st, _ = bcrp_arrays(meta["n"], z["src"], z["act"], z["dst"], meta["num_actions"])
    assert np.array_equal(block, z["block"])
    assert np.array_equal(np.asarray(st.splits_per_iteration, np.int32), z["splits"])
    assert st.supersteps == meta["supersteps"] == 13962
    assert st.final_block_count == meta["final_blocks"] == 9938


# ---------------------------------------------------------------- oracle

@pytest.mark.parametrize("n,m,A,seed", [(2000, 10000, 4, 11), (5000, 20000, 3, 12),
                                        (3000, 30000, 40, 13), (4000, 8000, 1, 14),
                                        (1000, 50000, 100, 15)])
def test_random_bcrp_vs_oracle(n, m, A, seed):
    g = np.random.default_rng(seed)
    src = g.integers(0, n, m, dtype=np.int32)
    act = g.integers(0, A, m, dtype=np.int32)
    dst = g.integers(0, n, m, dtype=np.int32)
    res = oracle.bcrp(n, src, act, dst, A, threads=4)
    block, st, _ = bcrp_arrays(n, src, act, dst, A)
    _same_oracle(block, st, res, f"random {seed}")


@pytest.mark.parametrize("n,deg,seed", [(3000, 5, 21), (10000, 3, 22), (2000, 1, 23)])
def test_random_rcpp_vs_oracle(n, deg, seed):
    inst = W.c2_kripke(n=n, out_degree=deg, seed=seed)
    res = oracle.rcpp(n, inst.src, inst.dst, inst.pi0, threads=4)
    block, st, _ = rcpp_arrays(n, inst.src, inst.dst, inst.pi0)
    _same_oracle(block, st, res, f"kripke {seed}")


def test_hub_heavy_vs_oracle():
    """Fan-out hubs scaled up: two states with out-degree n, one big block."""
    inst = W.fanout(3000)
    res = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=4)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    _same_oracle(block, st, res, "fanout 3000")


def test_many_labels_vs_oracle():
    """|Act| > 64 exercises multi-word label masks and multi-word slot compares."""
    inst = W.lifted_quotient(6000, 300, 300, templates=5, labels_per_template=70,
                             edges_per_label=1, seed=5)
    res = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=4)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    _same_oracle(block, st, res, "many labels")
    assert np.array_equal(block, inst.truth)


# ---------------------------------------------------------------- full-size configs

def test_c3_chain_full():
    inst = W.chain(200_000)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, 1)
    assert st.supersteps == 2 * inst.n - 2
    assert np.array_equal(block, inst.truth)


def _prefix_parity(run_gpu, run_oracle, K):
    """First K rounds: GPU stepped-mode observer snapshots and per-round
    split counts equal the oracle's truncated trace."""
    snaps = []

    class Stop(Exception):
        pass

    def grab(k, part):
        snaps.append(np.asarray(part.block, np.int32))
        if k == K:
            raise Stop

    with pytest.raises(Stop):
        run_gpu(grab)
    res = run_oracle(K)
    assert res.supersteps == K
    assert len(snaps) == K
    for k in range(K):
        assert np.array_equal(snaps[k], res.snapshots[k]), f"round {k + 1}"
    return res


def test_c2_kripke_prefix_and_final():
    """c2 at full size (n=1M, m=5M): first 30 rounds bit-exact vs the oracle,
    final partition equal to the signature-refinement truth."""
    inst = W.c2_kripke()
    _prefix_parity(lambda obs: rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0, observer=obs),
                   lambda K: oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, snap_rounds=K,
                                         stop_after=K, threads=8), 30)
    block, st, _ = rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0)
    truth = W.signature_bisim(inst.n, inst.src, np.zeros(inst.m, np.int32), inst.dst,
                              init=inst.pi0)
    assert np.array_equal(block, truth)
    assert st.final_block_count == len(np.unique(truth))
    assert st.supersteps <= 2 * inst.n - st.initial_block_count


def test_c4_lifted_prefix():
    inst = W.c4_lifted(n=1_000_000, k=10_000)
    _prefix_parity(lambda obs: bcrp_arrays(inst.n, inst.src, inst.act, inst.dst,
                                           inst.num_actions, observer=obs),
                   lambda K: oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                         snap_rounds=K, stop_after=K, threads=8), 10)
    block, st, _ = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    assert np.array_equal(block, inst.truth)


def test_c5_vlts_lifted_truth():
    inst = W.c5_vlts(n=2_000_000, k=1_000, seed=3)
    block, st, ns = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    assert np.array_equal(block, inst.truth)
    assert st.final_block_count == len(np.unique(inst.truth))


def test_label_grouping_equals_literal_rounds():
    """The hash-grouped label pre-partition equals the literal |Act| rounds
    of bcrp.py:144-184 (FLAG_LITERAL_LABEL_ROUNDS forces the latter)."""
    for seed, (n, m, A) in enumerate([(3000, 9000, 5), (2000, 20000, 70), (5000, 5000, 200)]):
        g = np.random.default_rng(100 + seed)
        src = g.integers(0, n, m, dtype=np.int32)
        act = g.integers(0, A, m, dtype=np.int32)
        dst = g.integers(0, n, m, dtype=np.int32)
        b1, s1, _ = bcrp_arrays(n, src, act, dst, A)
        b2, s2, _ = bcrp_arrays(n, src, act, dst, A, flags=N.FLAG_LITERAL_LABEL_ROUNDS)
        assert np.array_equal(b1, b2) and s1 == s2
        assert np.array_equal(b1, oracle.bcrp(n, src, act, dst, A, threads=4).block)


def test_noop_round_retirement_is_exact(mode):
    """Retiring runs of no-op rounds (splitters whose in-edge sources all sit
    in singleton blocks) gives the oracle's RunStats, as does running every
    round; the c4(i)-shaped case retires most of its rounds in bulk."""
    cases = [W.chain(3000), W.c2_kripke(n=20000, out_degree=3, seed=5),
             W.c4_uniform(n=20000, m=60000, num_actions=40, seed=6),
             W.c4_uniform(n=200_000, m=2_000_000, num_actions=256, seed=7)]
    for inst in cases:
        if inst.kind == "bcrp":
            run = lambda f=0: bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                          flags=f)
            res = oracle.bcrp_fast(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                   threads=4)
        else:
            run = lambda f=0: rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0, flags=f)
            res = oracle.rcpp_fast(inst.n, inst.src, inst.dst, inst.pi0)
        b1, s1, n1 = run()
        _same_oracle(b1, s1, res, inst.name)
        b2, s2, _ = run(N.FLAG_NO_SKIP)
        _same_oracle(b2, s2, res, inst.name + " no-skip")
        if inst.n == 200_000 and mode == "sparse":
            assert n1["rounds_retired"] > inst.n // 2, n1["rounds_retired"]


@pytest.mark.parametrize("flag", ["FLAG_NO_SOLO", "FLAG_NO_SKIP", "FLAG_CTA_MAJOR",
                                  "FLAG_NO_SOLO|FLAG_NO_SKIP", "FLAG_WIDE_LAYOUT|FLAG_NO_SOLO",
                                  "FLAG_TWO_PASS|FLAG_NO_SOLO", "FLAG_BATCH_WALK|FLAG_NO_SOLO",
                                  "FLAG_TWO_PASS|FLAG_BATCH_WALK|FLAG_NO_SOLO|FLAG_NO_SKIP"])
def test_loop_variants_identical(flag):
    """Solo stretches, no-op retirement and work placement never change a
    result: every variant reproduces the oracle on mixed workloads."""
    insts = [W.c2_kripke(n=30000, out_degree=4, seed=8), W.fanout(2000),
             W.lifted_quotient(60000, 600, 12, 4, 3, 2, seed=9)]
    g = np.random.default_rng(31)
    n, m, A = 20000, 80000, 3
    insts.append(W.Instance("rand", "bcrp", n, g.integers(0, n, m, dtype=np.int32),
                            g.integers(0, n, m, dtype=np.int32), g.integers(0, A, m, dtype=np.int32), A))
    for inst in insts:
        if inst.kind == "bcrp":
            res = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=8)
            run = lambda f=0: bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                          flags=f)
        else:
            res = oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, threads=8)
            run = lambda f=0: rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0, flags=f)
        b1, s1, _ = run()
        _same_oracle(b1, s1, res, inst.name)
        f = 0
        for part in flag.split("|"):
            f |= getattr(N, part)
        b2, s2, _ = run(f)
        _same_oracle(b2, s2, res, inst.name + " " + flag)
