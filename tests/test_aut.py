""".aut ingestion (csrc/aut.cpp via paper_2105_11788_b200.aut) against the
unmodified reference's parse_aut (aut.py:79-92).

Host-only C++ (no GPU needed): every fixture text in tests/golden/aut.json.gz
(made by oracle/gen_golden.py aut) must give the reference's Lts -- n,
initial state, sorted labels, transitions -- or the reference's ParseError
message and line.  Multi-threaded parsing of large texts must agree with the
single-threaded parse, including the line number of an error deep inside.
"""
import functools
import gzip
import json
import os

import re

import numpy as np
import pytest

from paper_2105_11788_b200.aut import ParseError, parse_aut, read_aut

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@functools.lru_cache(maxsize=None)
def aut_cases():
    with gzip.open(os.path.join(GOLDEN, "aut.json.gz"), "rt", encoding="utf-8") as fh:
        return json.load(fh)


def _outcome(text, threads=1):
    try:
        lts = parse_aut(text, threads=threads)
    except ParseError as e:
        return {"error": str(e), "line": e.line}
    s, a, d = lts.columns()
    return {"n": lts.n, "initial": lts.initial_state, "labels": list(lts.action_labels),
            "src": s.tolist(), "act": a.tolist(), "dst": d.tolist()}


def test_fixture_coverage():
    recs = aut_cases()
    assert len(recs) > 3000
    errs = [r for r in recs if "error" in r["ref"]]
    assert len(errs) > 1000 and len(recs) - len(errs) > 500


_HEADER = re.compile(r"des\s*\(\s*(\d+)\s*,\s*(\d+)\s*,\s*(\d+)\s*\)\s*$")


def test_parse_matches_reference_fixtures():
    """Bit-exact outcomes, except the documented limit: a declared state
    count of 2^30 or more is rejected at the header (the C ABI is int32)."""
    bad, limit = [], 0
    for r in aut_cases():
        got = _outcome(r["text"])
        if "exceeds this library's limit" in got.get("error", ""):
            lines = r["text"].splitlines()
            hdr = _HEADER.match(lines[0].strip()) if lines else None
            assert hdr and int(hdr.group(3)) >= 2 ** 30 and int(hdr.group(1)) < int(hdr.group(3))
            limit += 1
            continue
        if got != r["ref"]:
            bad.append((r["text"][:120], r["ref"], got))
    assert not bad, bad[:5]
    assert limit < 50


def test_reference_known_answers():
    # tests/test_aut.py:23-64 of the reference
    lts = parse_aut('des (0,1,2)\n(0,"a",1)')
    assert (lts.n, lts.m, lts.action_labels, lts.initial_state) == (2, 1, ("a",), 0)
    assert lts.transitions[0] == (0, 0, 1)
    with pytest.raises(ParseError, match="expected 3 transitions, found 1"):
        parse_aut("des (0,3,2)\n(0,a,1)")
    with pytest.raises(ParseError, match="line 1"):
        parse_aut("res (0,1,2)\n(0,a,1)")
    with pytest.raises(ParseError, match="line 3"):
        parse_aut("des (0,2,2)\n(0,a,1)\n(0,a,2)")
    with pytest.raises(ParseError, match="unterminated"):
        parse_aut('des (0,1,2)\n(0,"a,1)')
    with pytest.raises(ParseError):
        parse_aut("")
    assert isinstance(ParseError("x", 3), ValueError)


def _big_text(n, m, seed, labels=("a", "b c", "send(x, y)", "tau")):
    g = np.random.default_rng(seed)
    s = g.integers(0, n, m)
    a = g.integers(0, len(labels), m)
    d = g.integers(0, n, m)
    lines = [f"des (3, {m}, {n})"]
    lines += [f'({x}, "{labels[y]}", {z})' for x, y, z in zip(s.tolist(), a.tolist(), d.tolist())]
    return lines, (s, a, d)


def test_multithreaded_parse_matches_single_thread():
    lines, (s, a, d) = _big_text(5000, 300_000, 1)
    text = "\r\n".join(lines) + "\n"
    one = parse_aut(text, threads=1)
    many = parse_aut(text, threads=8)
    assert one == many
    assert len(text) > 4 << 20  # several 1 MiB+ chunks
    assert one.action_labels == ("a", "b c", "send(x, y)", "tau")
    ms, ma, md = many.columns()
    assert np.array_equal(ms, s) and np.array_equal(md, d)
    assert np.array_equal(ma, a)  # labels above are already in sorted order


@pytest.mark.parametrize("where", [1, 123_457, 299_999])
def test_multithreaded_error_line(where):
    lines, _ = _big_text(5000, 300_000, 2)
    lines[where + 1] = lines[where + 1].replace(",", ";", 1)  # breaks one transition
    text = "\n".join(lines) + ("\n\n" if where % 2 else "")
    with pytest.raises(ParseError) as e1:
        parse_aut(text, threads=8)
    with pytest.raises(ParseError) as e2:
        parse_aut(text, threads=1)
    assert e1.value.line == e2.value.line == where + 2
    assert str(e1.value) == str(e2.value)


def test_read_aut_file(tmp_path):
    lines, (s, a, d) = _big_text(100, 2000, 3)
    p = tmp_path / "x.aut"
    p.write_text("\n".join(lines) + "\n", encoding="utf-8")
    lts = read_aut(p)
    assert lts == parse_aut(p.read_text(encoding="utf-8"))
    assert lts.initial_state == 3 and lts.n == 100 and lts.m == 2000
    with pytest.raises(ParseError):
        (tmp_path / "e.aut").write_text("", encoding="utf-8")
        read_aut(tmp_path / "e.aut")


def test_long_labels_parse_from_worker_thread(tmp_path):
    """Labels longer than the std::string inline buffer live on the heap of
    the calling thread's malloc arena (mmapped high addresses off the main
    thread): the label pointer must come back untruncated."""
    import threading
    labels = ["a_rather_long_action_label_%03d" % i for i in range(40)]
    lines = ["des (0, %d, 50)" % len(labels)]
    lines += ['(%d, "%s", %d)' % (i, labels[i], (i * 7 + 3) % 50) for i in range(len(labels))]
    text = "\n".join(lines) + "\n"
    path = tmp_path / "long.aut"
    path.write_text(text)
    out = {}

    def work():
        try:
            out["parse"] = parse_aut(text, threads=2)
            out["read"] = read_aut(path, threads=2)
        except BaseException as e:  # noqa: BLE001
            out["exc"] = e

    t = threading.Thread(target=work)
    t.start()
    t.join()
    assert "exc" not in out, out.get("exc")
    for lts in (out["parse"], out["read"]):
        assert list(lts.action_labels) == sorted(labels)
        assert lts.n == 50
