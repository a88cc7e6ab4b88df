"""Plain Common policy (common_election=False) through the seam: the
PolicyViolationError (address, values, message), the SuperstepLimitError or
the result -- and the observer calls made before either -- must equal what
the unmodified reference does (tests/golden/common.json.gz, made by
`oracle/gen_golden.py common`; pram.py:147-152, bcrp.py:144-184,
rcpp.py:75-98,196-204)."""
import functools
import gzip
import json
import os

import pytest

from paper_2105_11788_b200 import (Common, Lts, Partition, PolicyViolationError, RelationInput,
                                   SuperstepLimitError, bcrp_run, partition_by_outgoing_labels,
                                   rcpp_run)

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def fixtures():
    with gzip.open(os.path.join(GOLDEN, "common.json.gz"), "rt") as fh:
        return json.load(fh)


def _guard(g):
    return None if g == "None" else int(g)


def _outcome(run):
    calls = []
    try:
        part, st = run(lambda k, p: calls.append([k, list(p.block)]))
    except PolicyViolationError as e:
        addr = list(e.address) if isinstance(e.address, tuple) else e.address
        return {"raised": "policy", "address": addr, "values": list(e.values), "message": str(e),
                "observed": calls}
    except SuperstepLimitError as e:
        return {"raised": "guard", "message": str(e), "observed": calls}
    return {"raised": None, "block": list(part.block), "supersteps": st.supersteps,
            "splits": list(st.splits_per_iteration), "initial_blocks": st.initial_block_count,
            "final_blocks": st.final_block_count, "observed": calls}


def _lts(rec):
    return Lts.from_arrays(rec["n"], rec["src"], rec["act"], rec["dst"], rec["num_actions"])


def test_bcrp_plain_common_matches_reference():
    for i, rec in enumerate(fixtures()["bcrp"]):
        lts = _lts(rec)
        for g, exp in rec["common"].items():
            got = _outcome(lambda obs: bcrp_run(lts, Common(), common_election=False, observer=obs,
                                                max_supersteps=_guard(g)))
            assert got == exp, (i, g)


def test_label_partition_plain_common_matches_reference():
    for i, rec in enumerate(fixtures()["bcrp"]):
        exp = rec["label_common"]
        try:
            p = partition_by_outgoing_labels(_lts(rec), Common(), common_election=False)
            got = {"raised": None, "block": list(p.block)}
        except PolicyViolationError as e:
            got = {"raised": "policy", "address": list(e.address), "values": list(e.values)}
        assert got == exp, i


def test_rcpp_plain_common_matches_reference():
    for i, rec in enumerate(fixtures()["rcpp"]):
        rel = RelationInput(rec["n"], list(zip(rec["src"], rec["dst"])), Partition(rec["pi0"]))
        for g, exp in rec["common"].items():
            got = _outcome(lambda obs: rcpp_run(rel, Common(), common_election=False, observer=obs,
                                                max_supersteps=_guard(g)))
            assert got == exp, (i, g)


def test_fixture_covers_every_branch():
    kinds = {}
    for rec in fixtures()["bcrp"] + fixtures()["rcpp"]:
        for o in rec["common"].values():
            key = (o["raised"], o["address"][0] if o.get("address") and
                   isinstance(o["address"], list) else o.get("address"))
            kinds[key] = kinds.get(key, 0) + 1
    assert kinds.get(("policy", "new_leader"), 0) > 0 and kinds.get(("policy", "C"), 0) > 0
    assert kinds.get(("guard", None), 0) > 0 and kinds.get((None, None), 0) > 0
