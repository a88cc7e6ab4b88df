"""Same-process A/B timing of two builds of libbisim.so (developer tool).

    python tools/ab_inproc.py ab/libA.so ab/libB.so c5 c1 ... [--reps 5]

Both libraries are loaded side by side (each keeps its own device buffers);
runs alternate A, B, A, B on the same instance and the medians of the
library's own CUDA-event phase times are printed, with a check that both
produce the same block array and round count.
"""
import argparse
import ctypes
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import make_instance  # noqa: E402
from paper_2105_11788_b200 import _native as N  # noqa: E402


def load(path):
    L = ctypes.CDLL(os.path.abspath(path))
    i32, i64, i32p = ctypes.c_int32, ctypes.c_int64, N.i32p
    L.bisim_bcrp_ex.argtypes = [i32, i64, i32, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                ctypes.POINTER(N.Stats), ctypes.POINTER(N.Options)]
    L.bisim_rcpp_ex.argtypes = [i32, i64, i32p, i32p, i32p, i64, i32p, i32p, i64,
                                ctypes.POINTER(N.Stats), ctypes.POINTER(N.Options)]
    L.bisim_last_error.restype = ctypes.c_char_p
    return L


def run(L, inst, flags=0):
    n = inst.n
    block = np.empty(n, np.int32)
    splits = np.zeros(3 * n + 16, np.int32)
    st = N.Stats()
    o = N.Options()
    o.flags = flags
    if inst.kind == "bcrp":
        rc = L.bisim_bcrp_ex(n, inst.m, inst.num_actions, N.ptr(inst.src), N.ptr(inst.act),
                             N.ptr(inst.dst), N.DEFAULT_GUARD, N.ptr(block), N.ptr(splits),
                             splits.size, ctypes.byref(st), ctypes.byref(o))
    else:
        rc = L.bisim_rcpp_ex(n, inst.m, N.ptr(inst.src), N.ptr(inst.dst), N.ptr(inst.pi0),
                             N.DEFAULT_GUARD, N.ptr(block), N.ptr(splits), splits.size,
                             ctypes.byref(st), ctypes.byref(o))
    if rc:
        raise RuntimeError(L.bisim_last_error().decode())
    return block, st


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs=2)
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    libs = [load(p) for p in a.libs]
    for cfg in a.configs:
        inst, _ = make_instance(cfg, 0)
        res = {0: [], 1: []}
        blocks = {}
        for rep in range(a.reps + 1):
            for k in (0, 1) if rep % 2 == 0 else (1, 0):
                block, st = run(libs[k], inst)
                blocks[k] = (block, st.supersteps)
                if rep:
                    res[k].append((st.t_pre_ms, st.t_label_ms, st.t_alg_ms))
        same = np.array_equal(blocks[0][0], blocks[1][0]) and blocks[0][1] == blocks[1][1]
        line = [cfg, f"R={blocks[0][1]}", "same" if same else "DIFFERENT"]
        for k, tag in ((0, "A"), (1, "B")):
            pre, lab, alg = (statistics.median(x[i] for x in res[k]) for i in range(3))
            line.append(f"{tag}: pre={pre:.2f} label={lab:.2f} alg={alg:.2f} tot={pre + lab + alg:.2f}")
        print("  ".join(line), flush=True)


if __name__ == "__main__":
    main()
