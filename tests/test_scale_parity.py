"""Full-size parity on every benchmark configuration (BASELINE.json configs,
SURVEY.md §8d): the GPU's RunStats and result digests against CPU-oracle
runs to completion (tests/golden/scale/, made by oracle/gen_scale.py).

Two oracles produced those fixtures: the literal restatement of the
reference's phases (oracle/bisim_oracle.c, O(n+m) per round, pinned to the
reference) where it finishes in hours on the development host, and the
event-driven restatement (oracle/bisim_fast.c, pinned to the reference
fixtures and to the literal oracle) for every config.  Where both exist the
CPU test below requires them to agree; the GPU tests then compare with the
fast oracle's record, so a config is never checked against the GPU's own
numbers.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np
import pytest

SCALE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "scale")


def _fixture(config: str, which: str = "fast"):
    path = os.path.join(SCALE, f"{config}.{which}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)


def _sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()


KEYS = ("supersteps", "initial_blocks", "final_blocks", "mark_length", "splits_sha256",
        "block_sha256", "n", "m")


def test_literal_and_fast_oracles_agree_at_full_size():
    """CPU: the two independent oracle runs give identical records."""
    pairs = 0
    for path in sorted(glob.glob(os.path.join(SCALE, "*.literal.json"))):
        config = os.path.basename(path).split(".")[0]
        lit, fast = _fixture(config, "literal"), _fixture(config, "fast")
        assert fast is not None, config
        for k in KEYS:
            assert lit[k] == fast[k], (config, k)
        pairs += 1
    assert pairs >= 1


def test_fixtures_cover_every_config():
    for c in ("c1", "c2", "c3", "c4u", "c4l", "c5", "c5s"):
        assert _fixture(c) is not None, c


def test_c1_fixture_is_the_reference_run():
    import _golden as G
    got = G.c1()
    meta, z = got
    rec = _fixture("c1")
    assert rec["supersteps"] == meta["supersteps"]
    assert rec["block_sha256"] == _sha(z["block"])
    assert rec["splits_sha256"] == _sha(z["splits"])


def _run_gpu(inst, flags=0):
    from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays
    if inst.kind == "bcrp":
        return bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, flags=flags)
    return rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0, flags=flags)


def _check(rec, block, st, ns, what):
    assert st.supersteps == rec["supersteps"], what
    assert st.initial_block_count == rec["initial_blocks"], what
    assert st.final_block_count == rec["final_blocks"], what
    assert ns["mark_length"] == rec["mark_length"], what
    splits = np.asarray(st.splits_per_iteration, np.int32)
    if _sha(splits) != rec["splits_sha256"]:
        ref = np.load(os.path.join(SCALE, f"{rec['config']}.fast.npz"))["splits"]
        k = int(np.nonzero(splits[:ref.size] != ref[:splits.size])[0][0]) if \
            splits.size == ref.size else min(splits.size, ref.size)
        pytest.fail(f"{what}: splits_per_iteration first differs at round {k + 1}")
    assert _sha(block) == rec["block_sha256"], what


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c1", "c2", "c3", "c4u", "c4l", "c5", "c5s"])
def test_gpu_full_size_runstats(config):
    import bench
    rec = _fixture(config)
    inst, _ = bench.make_instance(config, 0)
    block, st, ns = _run_gpu(inst)
    _check(rec, block, st, ns, config)
    if inst.truth is not None:
        assert np.array_equal(block, inst.truth), config
    if config == "c4u":
        # c4(i): every round also run one by one (no bulk retirement), and the
        # result is stable (GPU is_stable, oracle.py:128-141); the fixture
        # recorded equality with the signature-refinement fixed point.
        from paper_2105_11788_b200 import _native as N
        from paper_2105_11788_b200.post import is_stable_arrays
        b2, s2, n2 = _run_gpu(inst, flags=N.FLAG_NO_SKIP)
        _check(rec, b2, s2, n2, "c4u no-skip")
        assert is_stable_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, block)
        assert rec.get("signature_equal") is True


@pytest.mark.gpu
def test_gpu_c5s_virtual_sharded_replicas():
    """c5s (one n=40M, m=400M LTS) through the transition-sharded mode with
    two replicas sharing this GPU: identical RunStats and partition."""
    import bench
    from paper_2105_11788_b200.sharded import bcrp_sharded_arrays
    rec = _fixture("c5s")
    inst, _ = bench.make_instance("c5s", 0)
    block, st, ns = bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                        [0, 0], verify=True)
    _check(rec, block, st, ns, "c5s x2 sharded")
    assert np.array_equal(block, inst.truth)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [1, 7])
def test_gpu_c5_other_ranks_lifted_truth(seed):
    """The instances ranks 1..7 refine in `bench.py --gpus N` (c5 seeds 1..7)
    equal their lifted ground truth at full size."""
    from paper_2105_11788_b200 import workloads as W
    inst = W.c5_vlts(seed=seed)
    block, st, _ = _run_gpu(inst)
    assert np.array_equal(block, inst.truth)
    assert st.final_block_count == len(np.unique(inst.truth))


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c5", "c4l", "c2"])
@pytest.mark.parametrize("flags", ["FLAG_TWO_PASS|FLAG_NO_SOLO|FLAG_BATCH_WALK",
                                   "FLAG_WIDE_LAYOUT|FLAG_NO_SKIP|FLAG_CTA_MAJOR"])
def test_gpu_full_size_forced_layouts(config, flags):
    """Every round of a full-size configuration through the heavy-round code
    paths (two-pass split, batch registration wave, 128-member chunks, no
    solo stretches / no bulk retirement): RunStats and block digest still
    equal the oracle's run to completion."""
    import bench
    from paper_2105_11788_b200 import _native as N
    f = 0
    for part in flags.split("|"):
        f |= getattr(N, part)
    rec = _fixture(config)
    inst, _ = bench.make_instance(config, 0)
    block, st, ns = _run_gpu(inst, flags=f)
    _check(rec, block, st, ns, f"{config} {flags}")
