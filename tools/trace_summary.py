"""Summarise a BISIM_TRACE csv (capi.cu writes it): rounds grouped by kind.

    BISIM_DEV=1 BISIM_TRACE=100000 BISIM_TRACE_FILE=t.csv python tools/run_config.py c5
    python tools/trace_summary.py t.csv

Kinds: solo (CTA 0 alone), one-pass K=1 / wide, two-pass.  Columns are the
mean ns of each stamp interval (-1 entries, i.e. stamps a round did not
take, are left out of that column's mean).
"""
import sys

import numpy as np


def main(path):
    d = np.genfromtxt(path, delimiter=",", names=True, dtype=np.int64)
    if d.size == 0:
        print("empty trace")
        return
    d = d[d["phaseA_ns"] > 0]
    total = d["phaseA_ns"] + d["barrierA_ns"] + d["phaseB_ns"]
    kinds = {
        "solo": d["solo"] == 1,
        "onepass_k1": (d["solo"] == 0) & (d["mode_b"] == 0),
        "onepass_wide": (d["solo"] == 0) & (d["mode_b"] == 1),
        "twopass": (d["solo"] == 0) & (d["mode_b"] == 2),
    }
    cols = ["phaseA_ns", "barrierA_ns", "phaseB_ns", "csize", "n_small", "big_chunks", "n_big",
            "b_tag_ns", "b_sync1_ns", "b_arrive_ns", "b_sync2_ns", "b_place_ns",
            "a_walk0_ns", "a_walkcta_ns", "a_wave_ns"]
    print(f"{len(d)} traced rounds, {total.sum() / 1e6:.2f} ms stamped (round start to end barrier)")
    print("kind           rounds  total_ms  us/round  " + "  ".join(c[:10] for c in cols))
    for k, sel in kinds.items():
        if not sel.any():
            continue
        x = d[sel]
        t = total[sel]
        means = []
        for c in cols:
            v = x[c]
            v = v[v >= 0]
            means.append(f"{(v.mean() if v.size else float('nan')):10.0f}")
        print(f"{k:13s} {sel.sum():7d} {t.sum() / 1e6:9.2f} {t.mean() / 1e3:9.2f}  " + "  ".join(means))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "bisim_trace.csv")
