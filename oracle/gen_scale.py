"""Full-size parity fixtures: run a CPU oracle to completion on a benchmark
configuration and record its RunStats and result digests.

TEST INFRASTRUCTURE ONLY.  Run on the development host (no GPU needed); the
outputs under tests/golden/scale/ are committed and compared with the GPU
path by tests/test_scale_parity.py (-m gpu).

    python oracle/gen_scale.py --oracle literal c5 c4l c2 c3
    python oracle/gen_scale.py --oracle fast c2 c3 c4u c4l c5 c5s

Oracles:
  literal  oracle/bisim_oracle.c: the reference's PRAM phases restated
           phase by phase (bcrp.py:192-315, rcpp.py:220-259), every round
           O(n + m); pinned to the reference in tests/test_oracle_golden.py.
  fast     oracle/bisim_fast.c: a sequential, event-driven restatement of
           the same Priority program whose round costs O(|C| + in(C) +
           touched blocks); pinned to the reference fixtures and to the
           literal oracle in tests/test_oracle_golden.py.

For every (config, oracle) the fixture holds: supersteps, initial/final
block counts, mark length, the sha256 of splits_per_iteration (int32 LE)
and of the final block array (int32 LE), plus the splits array itself
(compressed .npz) so a mismatch can be located to the round.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "tests", "golden", "scale")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()


def run(config: str, which: str, threads: int, signature: bool = False) -> dict:
    import bench
    from oracle import oracle
    inst, desc = bench.make_instance(config, 0)
    t0 = time.time()
    if which == "literal":
        if inst.kind == "bcrp":
            r = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, threads=threads)
        else:
            r = oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, threads=threads)
    else:
        if inst.kind == "bcrp":
            r = oracle.bcrp_fast(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                 threads=threads)
        else:
            r = oracle.rcpp_fast(inst.n, inst.src, inst.dst, inst.pi0)
    wall = time.time() - t0
    rec = {"config": config, "workload": desc, "oracle": which, "kind": inst.kind,
           "n": inst.n, "m": inst.m, "num_actions": inst.num_actions,
           "supersteps": r.supersteps, "initial_blocks": r.initial_blocks,
           "final_blocks": r.final_blocks, "mark_length": r.mark_length,
           "splits_sha256": sha(r.splits), "splits_sum": int(np.asarray(r.splits, np.int64).sum()),
           "block_sha256": sha(r.block), "threads": threads, "wall_s": round(wall, 1),
           "truth_equal": None if inst.truth is None else bool(np.array_equal(r.block, inst.truth))}
    if signature and inst.truth is None:
        # an independent fixed point (iterated signature refinement,
        # workloads.signature_bisim) for configs without an analytic truth
        from paper_2105_11788_b200 import workloads as W
        act = inst.act if inst.kind == "bcrp" else np.zeros(inst.m, np.int32)
        truth = W.signature_bisim(inst.n, inst.src, act, inst.dst,
                                  init=None if inst.kind == "bcrp" else inst.pi0)
        rec["signature_equal"] = bool(np.array_equal(r.block, truth))
    os.makedirs(OUT, exist_ok=True)
    base = os.path.join(OUT, f"{config}.{which}")
    np.savez_compressed(base + ".npz", splits=np.asarray(r.splits, np.int32))
    with open(base + ".json", "w") as fh:
        json.dump(rec, fh, indent=1)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", choices=["literal", "fast"], default="fast")
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--signature", action="store_true",
                    help="also record equality with the signature-refinement fixed point")
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--signature-only", action="store_true",
                    help="add signature_equal to existing fixtures (compares digests)")
    a = ap.parse_args()
    if a.signature_only:
        import bench
        from paper_2105_11788_b200 import workloads as W
        for c in a.configs:
            path = os.path.join(OUT, f"{c}.{a.oracle}.json")
            with open(path) as fh:
                rec = json.load(fh)
            inst, _ = bench.make_instance(c, 0)
            act = inst.act if inst.kind == "bcrp" else np.zeros(inst.m, np.int32)
            truth = W.signature_bisim(inst.n, inst.src, act, inst.dst,
                                      init=None if inst.kind == "bcrp" else inst.pi0)
            rec["signature_equal"] = sha(truth) == rec["block_sha256"]
            with open(path, "w") as fh:
                json.dump(rec, fh, indent=1)
            print(c, rec["signature_equal"], flush=True)
        return
    for c in a.configs:
        rec = run(c, a.oracle, a.threads, a.signature)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
