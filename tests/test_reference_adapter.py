"""The drop-in, end to end: the UNMODIFIED reference package (installed into
baseline/_ref, the reference arm's install target) with its refinement path
swapped to the B200 by `paper_2105_11788_b200.refadapter.install` -- the
reference's own seam, module attributes its CLI calls (cli.py:97-119,
148-218) and its tests monkeypatch (tests/test_cli.py:210).

The stock reference and the adapted one must agree exactly: same Partition
and RunStats objects (the reference's classes), same observer calls, same
exception classes and messages, and the reference's own CLI (`parbisim
stats / reduce / compare`, run through its `main(argv)`) must print and
write the same bytes and return the same exit codes.
"""
import os
import sys

import pytest

import _golden as G

pytestmark = pytest.mark.gpu
REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "parbisim")):
        pytest.skip("reference package not installed in baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import parbisim
    import parbisim.cli  # noqa: F401
    return parbisim


@pytest.fixture
def adapted(ref):
    from paper_2105_11788_b200 import refadapter
    stock = {k: getattr(ref, k) for k in ("bcrp_run", "rcpp_run", "partition_by_outgoing_labels",
                                          "preprocess")}
    refadapter.install(ref)
    yield stock
    refadapter.uninstall(ref)


def _ref_lts(ref, rec):
    n, src, act, dst, A = G.arrays(rec)
    return ref.Lts(n=n, action_labels=tuple(f"a{i}" for i in range(A)),
                   transitions=tuple(ref.Transition(int(s), int(a), int(t))
                                     for s, a, t in zip(src, act, dst)))


def test_install_swaps_the_seam(ref, adapted):
    assert ref.bcrp_run is not adapted["bcrp_run"]
    assert ref.cli.bcrp_run is ref.bcrp_run and ref.cli.rcpp_run is ref.rcpp_run


def test_bcrp_run_equals_stock_reference(ref, adapted):
    recs = [G.cases()[k] for k in ("pre_fig2", "pre_no_outgoing", "pre_stable_sort", "fanout_9",
                                   "chain_10", "edge_free_4")] + G.sweep()[:60]
    for rec in recs:
        lts = _ref_lts(ref, rec)
        for policy in (ref.Priority(), ref.Common()):
            want_calls, got_calls = [], []
            want = adapted["bcrp_run"](lts, policy, observer=lambda k, p: want_calls.append((k, p)))
            got = ref.bcrp_run(lts, policy, observer=lambda k, p: got_calls.append((k, p)))
            assert type(got[0]) is ref.Partition and type(got[1]) is ref.RunStats
            assert got == want
            assert got_calls == want_calls


def test_rcpp_run_equals_stock_reference(ref, adapted):
    rec = G.cases()["five_state"]
    rel = ref.RelationInput(5, tuple(zip(rec["src"], rec["dst"])), ref.Partition(tuple(rec["pi0"])))
    assert ref.rcpp_run(rel, ref.Priority()) == adapted["rcpp_run"](rel, ref.Priority())
    for r in G.cases()["rcpp_noncanonical"][:20]:
        rel = ref.RelationInput(r["n"], tuple(zip(r["src"], r["dst"])), ref.Partition(tuple(r["pi0"])))
        assert ref.rcpp_run(rel, ref.Priority()) == adapted["rcpp_run"](rel, ref.Priority())


def test_preprocess_and_label_partition_equal_stock(ref, adapted):
    for name in ("pre_fig2", "pre_no_outgoing", "pre_stable_sort", "fanout_17"):
        lts = _ref_lts(ref, G.cases()[name])
        assert ref.preprocess(lts) == adapted["preprocess"](lts)
        assert (ref.partition_by_outgoing_labels(lts, ref.Priority())
                == adapted["partition_by_outgoing_labels"](lts, ref.Priority()))


def test_errors_are_the_references_classes(ref, adapted):
    lts = _ref_lts(ref, G.cases()["fanout_12"])
    for g in (0, 3, 10):
        with pytest.raises(ref.SuperstepLimitError) as got:
            ref.bcrp_run(lts, ref.Priority(), max_supersteps=g)
        with pytest.raises(ref.SuperstepLimitError) as want:
            adapted["bcrp_run"](lts, ref.Priority(), max_supersteps=g)
        assert str(got.value) == str(want.value)
    fig2 = _ref_lts(ref, G.cases()["pre_fig2"])
    with pytest.raises(ref.PolicyViolationError) as got:
        ref.bcrp_run(fig2, ref.Common(), common_election=False)
    with pytest.raises(ref.PolicyViolationError) as want:
        adapted["bcrp_run"](fig2, ref.Common(), common_election=False)
    assert (got.value.address, got.value.values, str(got.value)) == \
        (want.value.address, want.value.values, str(want.value))


def _cli(ref, argv, capsys):
    rc = ref.cli.main(argv)
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_reference_cli_output_identical(ref, adapted, tmp_path, capsys):
    """parbisim stats / reduce / compare with the stock path and with the
    B200 path: identical stdout, stderr, exit codes and written files."""
    from paper_2105_11788_b200 import refadapter
    recs = [G.cases()[k] for k in ("pre_fig2", "fanout_9", "chain_10")] + G.sweep()[:8]
    for i, rec in enumerate(recs):
        lts = _ref_lts(ref, rec)
        aut = tmp_path / f"in{i}.aut"
        aut.write_text(ref.write_aut(lts))
        runs = []
        for mode in ("stock", "b200"):
            if mode == "stock":
                refadapter.uninstall(ref)
            else:
                refadapter.install(ref)
            out_aut = tmp_path / f"out{i}_{mode}.aut"
            part = tmp_path / f"part{i}_{mode}.txt"
            r = [_cli(ref, ["stats", str(aut)], capsys),
                 _cli(ref, ["stats", str(aut), "--policy", "common"], capsys),
                 _cli(ref, ["reduce", str(aut), "-o", str(out_aut), "--partition-out", str(part)],
                      capsys),
                 _cli(ref, ["compare", str(aut)], capsys),
                 out_aut.read_text(), part.read_text()]
            if len(lts.action_labels) == 1:
                pi0 = tmp_path / f"pi0_{i}.txt"
                pi0.write_text(ref.write_partition(ref.trivial_partition(lts.n)))
                r.append(_cli(ref, ["stats", str(aut), "--pi0", str(pi0)], capsys))
            runs.append(r)
        assert runs[0] == runs[1], i
