"""Small instances for compute-sanitizer (memcheck / synccheck / racecheck).

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

Runs the five-state relation (Fig. 1), the Fig. 2 system, Fan_out 64 and a
small random system through every execution mode of libbisim.so --
persistent (work-efficient, all schedule variants), dense, stepped
(observer), two sharded replicas on one device -- plus preprocess(), the
label partition, quotient, is_stable, and out-of-range inputs, and checks
each result against the committed reference fixtures.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import _golden as G  # noqa: E402
from paper_2105_11788_b200 import (Lts, Priority, bcrp_arrays, partition_by_outgoing_labels,  # noqa: E402
                                   preprocess, rcpp_arrays)
from paper_2105_11788_b200 import _native as N  # noqa: E402
from paper_2105_11788_b200.post import is_stable_arrays, quotient_arrays  # noqa: E402
from paper_2105_11788_b200.sharded import bcrp_sharded_arrays  # noqa: E402

FLAGS = [0, N.FLAG_NO_SKIP, N.FLAG_NO_SOLO, N.FLAG_NO_SOLO | N.FLAG_NO_SKIP, N.FLAG_CTA_MAJOR,
         N.FLAG_LITERAL_LABEL_ROUNDS, N.FLAG_TWO_PASS | N.FLAG_NO_SOLO | N.FLAG_BATCH_WALK,
         N.FLAG_WIDE_LAYOUT | N.FLAG_NO_SOLO]


def check_bcrp(name):
    rec = G.cases()[name]
    n, src, act, dst, A = G.arrays(rec)
    exp = rec["bcrp"]
    runs = [bcrp_arrays(n, src, act, dst, A, flags=f) for f in FLAGS]
    runs.append(bcrp_arrays(n, src, act, dst, A, mode=N.MODE_DENSE))
    runs.append(bcrp_arrays(n, src, act, dst, A, observer=lambda k, p: None))
    runs.append(bcrp_sharded_arrays(n, src, act, dst, A, [0, 0], verify=True))
    for block, st, _ in runs:
        assert list(block) == exp["block"], name
        assert st.supersteps == exp["supersteps"], name
    lts = Lts.from_arrays(n, src, act, dst, A)
    aux = preprocess(lts)
    if "order" in rec:
        assert list(aux.order) == rec["order"]
    part = partition_by_outgoing_labels(lts, Priority())
    if "label_partition" in rec:
        assert list(part.block) == rec["label_partition"]
    assert is_stable_arrays(n, src, act, dst, A, runs[0][0])
    assert quotient_arrays(n, src, act, dst, A, runs[0][0])[0] == exp["final_blocks"]
    print("ok", name, flush=True)


def main():
    rec = G.cases()["five_state"]
    for f in FLAGS[:4]:
        block, st, _ = rcpp_arrays(5, rec["src"], rec["dst"], rec["pi0"], flags=f)
        assert tuple(block) == (0, 1, 2, 3, 3)
    block, st, _ = rcpp_arrays(5, rec["src"], rec["dst"], rec["pi0"], mode=N.MODE_DENSE)
    assert tuple(block) == (0, 1, 2, 3, 3)
    print("ok five_state", flush=True)
    for name in ("pre_fig2", "pre_no_outgoing", "fanout_64", "chain_200", "edge_free_4"):
        check_bcrp(name)
    for rec in G.cases()["medium_random"][:2]:
        n, src, act, dst, A = G.arrays(rec)
        block, st, _ = bcrp_arrays(n, src, act, dst, A)
        assert list(block) == rec["bcrp"]["block"]
    print("ok medium", flush=True)
    for bad in (([0, 1], [0, 1], [1, 4]), ([0, 4], [0, 1], [1, 2]), ([0, 1], [0, 2], [1, 2])):
        try:
            bcrp_arrays(4, bad[0], bad[1], bad[2], 2)
        except ValueError:
            pass
        else:
            raise AssertionError("out-of-range input accepted")
    print("ok bad inputs", flush=True)
    print("SANITIZE_CASES_OK", flush=True)


if __name__ == "__main__":
    main()
