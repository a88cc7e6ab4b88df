"""Generate golden fixtures by running the UNMODIFIED reference package.

TEST INFRASTRUCTURE ONLY.  Run in the development container, where the
reference lives at /root/reference (read-only); the outputs under
tests/golden/ are committed so the GPU box (which has no /root/reference)
can check against them.

    python oracle/gen_golden.py cases      # small known-answer instances
    python oracle/gen_golden.py sweep      # acceptance-sweep instances
    python oracle/gen_golden.py c1         # config c1 full run (~35 min, 1 core)
    python oracle/gen_golden.py post       # quotient / is_stable / canonical fixtures
    python oracle/gen_golden.py aut        # parse_aut outcomes (texts + results / errors)
    python oracle/gen_golden.py common     # plain-Common-policy outcomes (violations, guards)

Every fixture records the instance (src/act/dst arrays or the generator
recipe), the reference's Priority-policy outputs (block array in leader form,
RunStats) and where applicable the per-round observer snapshots.
"""
from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _ref():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import parbisim  # noqa: F401
    return parbisim


def lts_arrays(lts):
    tr = lts.transitions
    return {
        "n": lts.n,
        "num_actions": len(lts.action_labels),
        "src": [t.source for t in tr],
        "act": [t.action for t in tr],
        "dst": [t.target for t in tr],
    }


def run_bcrp(pb, lts, snaps=False, max_supersteps=None):
    chain = []
    obs = (lambda k, p: chain.append(list(p.block))) if snaps else None
    try:
        part, st = pb.bcrp_run(lts, pb.Priority(), observer=obs, max_supersteps=max_supersteps)
    except pb.SuperstepLimitError:
        return {"guard": True, "snapshots": chain if snaps else None}
    out = {"guard": False, "block": list(part.block), "supersteps": st.supersteps,
           "splits": list(st.splits_per_iteration), "initial_blocks": st.initial_block_count,
           "final_blocks": st.final_block_count}
    if snaps:
        out["snapshots"] = chain
    return out


def run_rcpp(pb, n, edges, pi0_block, snaps=False, max_supersteps=None):
    chain = []
    obs = (lambda k, p: chain.append(list(p.block))) if snaps else None
    rel = pb.RelationInput(n, tuple(edges), pb.Partition(pi0_block))
    try:
        part, st = pb.rcpp_run(rel, pb.Priority(), observer=obs, max_supersteps=max_supersteps)
    except pb.SuperstepLimitError:
        return {"guard": True, "snapshots": chain if snaps else None}
    out = {"guard": False, "block": list(part.block), "supersteps": st.supersteps,
           "splits": list(st.splits_per_iteration), "initial_blocks": st.initial_block_count,
           "final_blocks": st.final_block_count}
    if snaps:
        out["snapshots"] = chain
    return out


def chain_lts(pb, n):
    return pb.lts_from_labeled_edges(n, [(i, "a", i + 1) for i in range(n - 1)])


def cases():
    pb = _ref()
    sys.path.insert(0, REF_TESTS)
    import _support as sup
    from parbisim.cli import gen_fanout
    out = {}

    # preprocessing tables: Fig. 2 instance (test_acceptance.py:239-257) and
    # the no-outgoing-state instance (test_bcrp.py:105-110)
    for name, lts in [("fig2", sup.mixed_label_lts()),
                      ("no_outgoing", pb.lts_from_labeled_edges(3, [(0, "a", 1), (2, "b", 0)])),
                      ("stable_sort", pb.lts_from_labeled_edges(2, [(1, "b", 0), (0, "a", 1),
                                                                    (0, "a", 0)]))]:
        aux = pb.preprocess(lts)
        rec = lts_arrays(lts)
        index = {t: [] for t in set(lts.transitions)}
        # the sorted permutation: k-th sorted transition = original index perm[k]
        used = [False] * lts.m
        perm = []
        for t in aux.lts.transitions:
            for i, u in enumerate(lts.transitions):
                if not used[i] and u == t:
                    used[i] = True
                    perm.append(i)
                    break
        del index
        rec.update(perm=perm, action_switch=list(aux.action_switch), order=list(aux.order),
                   nr_marks=list(aux.nr_marks), off=list(aux.off), mark_length=aux.mark_length,
                   label_partition=list(pb.partition_by_outgoing_labels(lts, pb.Priority()).block),
                   bcrp=run_bcrp(pb, lts, snaps=True))
        out["pre_" + name] = rec

    # Fig. 1 five-state relation (test_rcpp.py:119-136, FIVE_STATE_FINAL)
    rel = sup.five_state_input()
    out["five_state"] = {"n": 5, "src": [e[0] for e in rel.edges], "dst": [e[1] for e in rel.edges],
                         "pi0": list(rel.pi0.block),
                         "rcpp": run_rcpp(pb, 5, rel.edges, rel.pi0.block, snaps=True)}

    # Fan_out family (cli.py:62-75): BCRP and RCPP from the trivial partition
    for n in list(range(3, 65)) + [100, 200]:
        lts = gen_fanout(n)
        rec = lts_arrays(lts)
        rec["bcrp"] = run_bcrp(pb, lts, snaps=(n <= 20))
        edges = [(t.source, t.target) for t in lts.transitions]
        rec["rcpp_trivial"] = run_rcpp(pb, n, edges, [0] * n, snaps=(n <= 20))
        out[f"fanout_{n}"] = rec

    # chains (SURVEY c3 shape): BCRP R = 2n-2, RCPP R = 2n-1
    for n in (2, 3, 10, 100, 200):
        lts = chain_lts(pb, n)
        rec = lts_arrays(lts)
        rec["bcrp"] = run_bcrp(pb, lts)
        edges = [(t.source, t.target) for t in lts.transitions]
        rec["rcpp_trivial"] = run_rcpp(pb, n, edges, [0] * n)
        out[f"chain_{n}"] = rec

    # edge-free (test_rcpp.py:225-231) and label-only instances
    lts = pb.lts_from_labeled_edges(4, [], extra_labels=("a", "b"))
    rec = lts_arrays(lts)
    rec["bcrp"] = run_bcrp(pb, lts)
    rec["rcpp_trivial"] = run_rcpp(pb, 4, [], [0] * 4)
    out["edge_free_4"] = rec

    # guard boundaries: the run completes iff |Act| + R + 1 <= max_supersteps
    guard = []
    for n in (4, 8, 12):
        lts = gen_fanout(n)
        full = run_bcrp(pb, lts)
        A = len(lts.action_labels)
        for g in (0, 1, 2, A, A + full["supersteps"], A + full["supersteps"] + 1):
            guard.append({"kind": "bcrp", "instance": f"fanout_{n}", "max_supersteps": g,
                          "result": run_bcrp(pb, lts, max_supersteps=g)})
        edges = [(t.source, t.target) for t in lts.transitions]
        rfull = run_rcpp(pb, n, edges, [0] * n)
        for g in (0, 1, rfull["supersteps"], rfull["supersteps"] + 1):
            guard.append({"kind": "rcpp_trivial", "instance": f"fanout_{n}", "max_supersteps": g,
                          "result": run_rcpp(pb, n, edges, [0] * n, max_supersteps=g)})
    out["guard"] = guard

    # RCPP with non-canonical pi0 leaders (Partition allows any self-led
    # leader, lts.py:85-95): pi0 is used verbatim (rcpp.py:64)
    rng = random.Random(7)
    noncanon = []
    for idx in range(60):
        n = rng.randint(1, 30)
        m = rng.randint(0, 3 * n)
        edges = [(rng.randrange(n), rng.randrange(n)) for _ in range(m)]
        k = rng.randint(1, max(1, n // 3))
        colour = [rng.randrange(k) for _ in range(n)]
        leader_of = {}
        for s in range(n):  # leader = LARGEST member of its colour class
            leader_of[colour[s]] = s
        pi0 = [leader_of[c] for c in colour]
        noncanon.append({"n": n, "src": [e[0] for e in edges], "dst": [e[1] for e in edges],
                         "pi0": pi0, "rcpp": run_rcpp(pb, n, edges, pi0, snaps=True)})
    out["rcpp_noncanonical"] = noncanon

    # medium random BCRP instances (oracle-finishable, a few seconds each)
    medium = []
    for idx, (n, m, A) in enumerate([(300, 1500, 4), (500, 2500, 3), (400, 4000, 8),
                                     (600, 1800, 1), (250, 2500, 16)]):
        r = random.Random(1000 + idx)
        labels = [f"l{j:02d}" for j in range(A)]
        edges = [(r.randrange(n), labels[r.randrange(A)], r.randrange(n)) for _ in range(m)]
        lts = pb.lts_from_labeled_edges(n, edges, extra_labels=labels)
        rec = lts_arrays(lts)
        rec["bcrp"] = run_bcrp(pb, lts)
        medium.append(rec)
    out["medium_random"] = medium

    with gzip.open(os.path.join(OUT, "cases.json.gz"), "wt") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote cases.json.gz")


def sweep(count=1000):
    """The acceptance sweep generator (test_acceptance.py:114-125,
    _support.py:55-66) with Priority outputs and observer chains."""
    pb = _ref()
    sys.path.insert(0, REF_TESTS)
    import _support as sup
    rng = random.Random(20260814)
    recs = []
    for idx in range(count):
        seed = rng.randrange(2 ** 32)
        lts = sup.random_lts(random.Random(seed))
        rec = lts_arrays(lts)
        rec["seed"] = seed
        rec["bcrp"] = run_bcrp(pb, lts, snaps=True)
        if len(lts.action_labels) == 1:
            edges = [(t.source, t.target) for t in lts.transitions]
            rec["rcpp_trivial"] = run_rcpp(pb, lts.n, edges, [0] * lts.n, snaps=True)
        recs.append(rec)
    with gzip.open(os.path.join(OUT, "sweep.json.gz"), "wt") as fh:
        json.dump(recs, fh, separators=(",", ":"))
    print(f"wrote sweep.json.gz ({count} instances)")


def c1():
    """n=10k, m=50k, |Act|=4, random.Random(1)."""
    pb = _ref()
    n, m = 10_000, 50_000
    rng = random.Random(1)
    labels = ["a0", "a1", "a2", "a3"]
    edges = []
    for _ in range(m):
        s = rng.randrange(n)
        lab = labels[rng.randrange(4)]
        t = rng.randrange(n)
        edges.append((s, lab, t))
    lts = pb.lts_from_labeled_edges(n, edges, extra_labels=labels)
    t0 = time.perf_counter()
    res = run_bcrp(pb, lts)
    res["wall_s"] = time.perf_counter() - t0
    res["recipe"] = "random.Random(1); per edge: s=randrange(n), lab=labels[randrange(4)], t=randrange(n)"
    res["n"], res["m"], res["num_actions"] = n, m, 4
    arrays = lts_arrays(lts)
    np.savez_compressed(os.path.join(OUT, "c1_reference.npz"),
                        src=np.array(arrays["src"], np.int32),
                        act=np.array(arrays["act"], np.int32),
                        dst=np.array(arrays["dst"], np.int32),
                        block=np.array(res["block"], np.int32),
                        splits=np.array(res["splits"], np.int32))
    meta = {k: v for k, v in res.items() if k not in ("block", "splits")}
    with open(os.path.join(OUT, "c1_reference.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("c1:", meta)


def post(count=400):
    """quotient (aut.py:132-152), is_stable (oracle.py:128-141) and
    partition_from_assignment (lts.py:117-128) of the reference, on the first
    `count` sweep instances and the medium instances, each under several
    partitions (the coarsest one, the label partition, trivial, discrete and
    a random one), plus random id assignments."""
    pb = _ref()
    from parbisim.oracle import is_stable as ref_is_stable
    from parbisim.oracle import is_stable_under as ref_is_stable_under
    with gzip.open(os.path.join(OUT, "sweep.json.gz"), "rt") as fh:
        sweep_recs = json.load(fh)[:count]
    with gzip.open(os.path.join(OUT, "cases.json.gz"), "rt") as fh:
        case_recs = json.load(fh)["medium_random"]
    rng = random.Random(31337)
    out = []
    for idx, rec in enumerate(sweep_recs + case_recs):
        n, A = rec["n"], rec["num_actions"]
        init = rng.randrange(n)
        lts = pb.Lts(n=n, action_labels=tuple(f"a{k}" for k in range(A)),
                     transitions=tuple(pb.Transition(s, a, t) for s, a, t in
                                       zip(rec["src"], rec["act"], rec["dst"])),
                     initial_state=init)
        k = rng.randint(1, max(1, n // 2))
        assignment = [rng.randrange(k) * 7 - 3 for _ in range(n)]
        parts = {"coarsest": rec["bcrp"]["block"],
                 "labels": list(pb.partition_by_outgoing_labels(lts, pb.Priority()).block),
                 "trivial": [0] * n, "discrete": list(range(n)),
                 "random": list(pb.partition_from_assignment(assignment).block)}
        res = {}
        for name, blk in parts.items():
            p = pb.Partition(blk)
            q = pb.quotient(lts, p)
            subsets = [sorted(rng.sample(range(n), rng.randint(0, n))) for _ in range(2)]
            # one block of the partition as the target set (the splitter case)
            subsets.append([t for t in range(n) if blk[t] == blk[rng.randrange(n)]])
            res[name] = {"block": blk, "stable": ref_is_stable(lts, p),
                         "under": [[sub, ref_is_stable_under(lts, p, sub)] for sub in subsets],
                         "q_n": q.n, "q_initial": q.initial_state,
                         "q_src": [t.source for t in q.transitions],
                         "q_act": [t.action for t in q.transitions],
                         "q_dst": [t.target for t in q.transitions]}
        out.append({"n": n, "num_actions": A, "initial_state": init, "src": rec["src"],
                    "act": rec["act"], "dst": rec["dst"], "assignment": assignment,
                    "canonical": res["random"]["block"], "partitions": res})
    with gzip.open(os.path.join(OUT, "post.json.gz"), "wt") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print(f"wrote post.json.gz ({len(out)} instances)")


def aut(fuzz=3000):
    """parse_aut (aut.py:79-92) outcomes of the unmodified reference: the
    reference's own test texts (tests/test_aut.py:23-64), hand-written edge
    cases, write_aut round trips of sweep instances with awkward labels, and
    random single-character mutations of small files (error paths)."""
    pb = _ref()
    from parbisim.aut import ParseError, write_aut

    def outcome(text):
        try:
            lts = pb.parse_aut(text)
        except ParseError as e:
            return {"error": str(e), "line": e.line}
        return {"n": lts.n, "initial": lts.initial_state, "labels": list(lts.action_labels),
                "src": [t.source for t in lts.transitions],
                "act": [t.action for t in lts.transitions],
                "dst": [t.target for t in lts.transitions]}

    texts = [
        'des (0,1,2)\n(0,"a",1)', 'des (0,2,2)\n(0,a,1)\n(1,"b c",0)',
        'des (0,1,2)\n(0,"send(x, y)",1)', "des (0,3,2)\n(0,a,1)", "res (0,1,2)\n(0,a,1)",
        "des (0,2,2)\n(0,a,1)\n(0,a,2)", 'des (0,1,2)\n(0,"a,1)', "des (2,0,2)\n",
        "des ( 0 , 1 , 2 )\r\n( 0 , a , 1 )\r\n\r\n", "", "\n", " ", "des (0,0,1)",
        "des (0,0,0)", "des (0, 0, 1)\n\n\n", "des(0,1,1)\n(0,a,0)", "des (0,1,1) x\n(0,a,0)",
        "  des (0,1,1)  \n(0,a,0)", "des (0,1,1)\r(0,a,0)", "des (0,1,1)\x0b(0,a,0)",
        "des (0,1,1)\x0c(0,a,0)\x1c", "des (0,1,1)\x1d(0,a,0)\x1e", "des (0,1,1)\x85(0,a,0)",
        "des (0,1,1)\u2028(0,a,0)\u2029", "des (0,1,1)\n\x1f(0,a,0)\x1f", "des (0,1,1)\n\xa0(0,a,0)",
        "des (0,1,1)\n\u3000(0,\u2003a\u2003,0)", "des (0,1,3)\n(+1,a,2)", "des (0,1,3)\n(007,a,0_2)",
        "des (0,1,3)\n(1_0,a,2)", "des (0,1,3)\n(-1,a,2)", "des (0,1,3)\n(-0,a,2)",
        "des (0,1,3)\n(1__0,a,2)", "des (0,1,3)\n(_1,a,2)", "des (0,1,3)\n(1_,a,2)",
        "des (0,1,3)\n(+,a,2)", "des (0,1,3)\n( ,a,2)", "des (0,1,3)\n(0x1,a,2)",
        "des (0,1,3)\n(99999999999999999999999,a,2)", "des (0,1,3)\n(1,a,99999999999)",
        "des (0,1,3)\n(1,,2)", "des (0,1,3)\n(1, ,2)", 'des (0,1,3)\n(1,"",2)',
        'des (0,1,3)\n(1,",2)', 'des (0,1,3)\n(1,"a"b",2)', 'des (0,1,3)\n(1,a"b,2)',
        "des (0,1,3)\n(1,a(b,2)", "des (0,1,3)\n(1,a)b,2)", "des (0,1,3)\n(1,a,b,2)",
        'des (0,1,3)\n(1,"a,b",2)', "des (0,1,3)\n(1,a 2)", "des (0,1,3)\n(1 a 2)",
        "des (0,1,3)\n1,a,2)", "des (0,1,3)\n(1,a,2", "des (0,1,3)\n()", "des (0,1,3)\n(,)",
        "des (0,1,3)\n(,,)", "des (0,1,3)\n(", "des (0,1,3)\n)", "des (0,1,3)\n(1,a,2) x",
        "des (0,1,3)\n(x,a,y)", "des (0,1,3)\n(x',a,y)", "des (0,1,3)\n(x'\",a,y)",
        "des (0,1,3)\n(\\,a,\t)", "des (0,1,3)\n(\x7f,a,\x01)", "des (0,1,3)\n(\xe9,a,\xad)",
        "des (0,1,3)\n(1,\xe9t\xe9,2)", 'des (0,2,3)\n(1,"z",2)\n(0,"\xe9",1)',
        'des (0,3,3)\n(1,b,2)\n(0,"B",1)\n(2,"a b",0)', "des (0,2,3)\n(0,a,1)\n(0,a,1)",
        "des (1,2,3)\n(0,a,1)\n(1,a,2)\n", "des (00,01,03)\n(0,a,1)", "des (0,1,3)\n\n\n(0,a,1)\n\n",
        "des (0,2,3)\n(0,a,1)", "des (0,0,3)\n(0,a,1)", "des (0,1,3)\n(0,a,1)\n(0,a,1)\n(x)",
        "des (0,1,3)\n(0,a,5)\n(x)", "des (-1,1,3)\n(0,a,1)", "des (0,1,3,4)\n(0,a,1)",
        "DES (0,1,3)\n(0,a,1)", "des (0,1,3\n(0,a,1)", "des 0,1,3)\n(0,a,1)",
        "des (0,99999999999999999999,3)\n(0,a,1)", "des (5,1,99999999999999999999)\n(0,a,1)",
    ]
    recs = [{"text": t, "ref": outcome(t)} for t in texts]
    # write_aut round trips with awkward labels
    with gzip.open(os.path.join(OUT, "sweep.json.gz"), "rt") as fh:
        sweep_recs = json.load(fh)[:200]
    pool = ["a", "b c", "send(x, y)", "\xe9t\xe9", "q\"r", "x,y", "tau", "i", "A", "\u2603"]
    rng = random.Random(4242)
    for rec in sweep_recs:
        A = rec["num_actions"]
        labels = tuple(sorted(rng.sample(pool, A))) if A <= len(pool) else tuple(
            f"l{k}" for k in range(A))
        lts = pb.Lts(n=rec["n"], action_labels=labels,
                     transitions=tuple(pb.Transition(s, a, t) for s, a, t in
                                       zip(rec["src"], rec["act"], rec["dst"])),
                     initial_state=rng.randrange(rec["n"]))
        t = write_aut(lts)
        recs.append({"text": t, "ref": outcome(t)})
    # single-character mutations of small files
    alphabet = list("0123456789,()\" _-+ab\t\r\n\x0b\x0c\x1c\x85\xa0\xe9\u2028")
    bases = [r["text"] for r in recs if len(r["text"]) < 400 and "error" not in r["ref"]][:80]
    for _ in range(fuzz):
        t = rng.choice(bases)
        k = rng.randrange(len(t) + 1)
        op = rng.randrange(3)
        if op == 0 and k < len(t):
            t = t[:k] + t[k + 1:]
        elif op == 1:
            t = t[:k] + rng.choice(alphabet) + t[k:]
        elif k < len(t):
            t = t[:k] + rng.choice(alphabet) + t[k + 1:]
        recs.append({"text": t, "ref": outcome(t)})
    with gzip.open(os.path.join(OUT, "aut.json.gz"), "wt", encoding="utf-8") as fh:
        json.dump(recs, fh, separators=(",", ":"))
    errs = sum("error" in r["ref"] for r in recs)
    print(f"wrote aut.json.gz ({len(recs)} texts, {errs} parse errors)")


def common():
    """Outcomes of the reference under the PLAIN Common policy
    (common_election=False, pram.py:147-152): PolicyViolationError address
    and values, SuperstepLimitError, or the result -- plus the observer calls
    made before -- for BCRP and RCPP instances reaching every branch (label
    round conflicts, the first-select conflict, one-block systems, RCPP
    round-1 splits of 0 / 1 / >= 2 states, non-canonical pi0, guards)."""
    pb = _ref()
    sys.path.insert(0, REF_TESTS)
    import _support as sup
    from parbisim.cli import gen_fanout

    def outcome(run):
        calls = []
        try:
            part, st = run(lambda k, p: calls.append([k, list(p.block)]))
        except pb.PolicyViolationError as e:
            addr = list(e.address) if isinstance(e.address, tuple) else e.address
            return {"raised": "policy", "address": addr, "values": list(e.values),
                    "message": str(e), "observed": calls}
        except pb.SuperstepLimitError as e:
            return {"raised": "guard", "message": str(e), "observed": calls}
        return {"raised": None, "block": list(part.block), "supersteps": st.supersteps,
                "splits": list(st.splits_per_iteration), "initial_blocks": st.initial_block_count,
                "final_blocks": st.final_block_count, "observed": calls}

    def bcrp_case(lts, guards=(None,)):
        rec = lts_arrays(lts)
        rec["common"] = {str(g): outcome(lambda obs, g=g: pb.bcrp_run(
            lts, pb.Common(), common_election=False, observer=obs, max_supersteps=g))
            for g in guards}
        try:
            lp = pb.partition_by_outgoing_labels(lts, pb.Common(), common_election=False)
            rec["label_common"] = {"raised": None, "block": list(lp.block)}
        except pb.PolicyViolationError as e:
            addr = list(e.address) if isinstance(e.address, tuple) else e.address
            rec["label_common"] = {"raised": "policy", "address": addr, "values": list(e.values)}
        return rec

    def rcpp_case(n, edges, pi0, guards=(None,)):
        rel = pb.RelationInput(n, tuple(edges), pb.Partition(pi0))
        rec = {"n": n, "src": [e[0] for e in edges], "dst": [e[1] for e in edges], "pi0": list(pi0)}
        rec["common"] = {str(g): outcome(lambda obs, g=g: pb.rcpp_run(
            rel, pb.Common(), common_election=False, observer=obs, max_supersteps=g))
            for g in guards}
        return rec

    bcrp, rcpp = [], []
    L = pb.lts_from_labeled_edges
    guards = (None, -1, 0, 1, 2, 3, 4, 5)
    # label-round conflicts (most systems), first-select conflicts (chains),
    # one-block systems (cycles, edge-free), hubs
    bcrp.append(bcrp_case(sup.mixed_label_lts(), guards))
    for n in (2, 3, 5, 8):
        bcrp.append(bcrp_case(chain_lts(pb, n), guards))
        bcrp.append(bcrp_case(L(n, [(i, "a", (i + 1) % n) for i in range(n)]), guards))
        bcrp.append(bcrp_case(L(n, [(i, lab, (i + 1) % n) for i in range(n) for lab in "ab"]),
                              guards))
    bcrp.append(bcrp_case(pb.Lts(4, ("a", "b"), ()), guards))
    for n in (3, 4, 6, 10):
        bcrp.append(bcrp_case(gen_fanout(n), guards))
    bcrp.append(bcrp_case(L(4, [(0, "a", 1), (1, "b", 2), (2, "a", 3), (3, "b", 0)]), guards))
    bcrp.append(bcrp_case(L(5, [(0, "a", 1), (2, "a", 1), (3, "b", 4)], extra_labels=["c"]),
                          guards))
    rng = random.Random(777)
    for _ in range(300):
        bcrp.append(bcrp_case(sup.random_lts(random.Random(rng.randrange(2 ** 32))), (None, 1, 3)))
    # RCPP: >= 2 blocks, one block with round-1 split sets of size 0 / 1 / >= 2,
    # non-canonical leaders
    rcpp.append(rcpp_case(3, [(1, 0), (2, 0)], [0, 0, 0], guards))          # test_acceptance.py:361
    rcpp.append(rcpp_case(5, [(0, 3), (1, 4), (1, 2), (2, 1)], [0, 0, 0, 3, 3], guards))
    for n in (2, 3, 4, 7):
        rcpp.append(rcpp_case(n, [(i, i + 1) for i in range(n - 1)], [0] * n, guards))
        rcpp.append(rcpp_case(n, [(i, (i + 1) % n) for i in range(n)], [0] * n, guards))
        rcpp.append(rcpp_case(n, [(i, i + 1) for i in range(n - 1)], [n - 1] * n, guards))
        rcpp.append(rcpp_case(n, [(i, (i + 1) % n) for i in range(n)], [n // 2] * n, guards))
    rcpp.append(rcpp_case(4, [(0, 1)], [2, 2, 2, 2], guards))
    rcpp.append(rcpp_case(4, [(1, 0), (2, 3), (3, 3)], [1, 1, 1, 1], guards))
    rcpp.append(rcpp_case(4, [], [0, 0, 0, 0], guards))
    for _ in range(200):
        r = random.Random(rng.randrange(2 ** 32))
        n = r.randrange(1, 9)
        edges = [(r.randrange(n), r.randrange(n)) for _ in range(r.randrange(0, 3 * n))]
        k = r.randrange(1, 3)
        col = [r.randrange(k) for _ in range(n)]
        lead = {}
        for sidx in r.sample(range(n), n):
            lead.setdefault(col[sidx], sidx)
        rcpp.append(rcpp_case(n, edges, [lead[c] for c in col], (None, 0, 1, 2)))
    with gzip.open(os.path.join(OUT, "common.json.gz"), "wt") as fh:
        json.dump({"bcrp": bcrp, "rcpp": rcpp}, fh, separators=(",", ":"))
    kinds = [o["raised"] for rec in bcrp + rcpp for o in rec["common"].values()]
    print(f"wrote common.json.gz ({len(bcrp)} bcrp, {len(rcpp)} rcpp; outcomes "
          f"{ {k: kinds.count(k) for k in set(kinds)} })")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    what = sys.argv[1] if len(sys.argv) > 1 else "cases"
    {"cases": cases, "sweep": sweep, "c1": c1, "post": post, "aut": aut, "common": common}[what]()
