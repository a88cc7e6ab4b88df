"""Throughput of the .aut reader (csrc/aut.cpp) on a generated file.

    python tools/aut_bench.py [m] [n]

Writes an Aldebaran file with m transitions over n states (quoted labels,
32 distinct), parses it with read_aut (all host threads) and with one
thread, and checks the columns against the generator.
"""
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2105_11788_b200.aut import read_aut  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
g = np.random.default_rng(0)
src = g.integers(0, n, m)
act = g.integers(0, 32, m)
dst = g.integers(0, n, m)
labels = [f"act_{k:02d}(x, y)" for k in range(32)]
path = os.path.join(tempfile.gettempdir(), f"bench_{m}.aut")
t = time.perf_counter()
with open(path, "w") as fh:
    fh.write(f"des (0, {m}, {n})\n")
    step = 1_000_000
    lab = np.array([f'"{x}"' for x in labels])
    for i in range(0, m, step):
        rows = np.char.add(np.char.add(np.char.add(np.char.add(
            "(", src[i:i + step].astype(str)), ", "), lab[act[i:i + step]]), ", ")
        rows = np.char.add(np.char.add(rows, dst[i:i + step].astype(str)), ")\n")
        fh.write("".join(rows.tolist()))
size = os.path.getsize(path)
print(f"wrote {size / 1e9:.2f} GB in {time.perf_counter() - t:.1f} s")
for threads in (0, 1):
    t = time.perf_counter()
    lts = read_aut(path, threads=threads)
    dt = time.perf_counter() - t
    s, a, d = lts.columns()
    ok = np.array_equal(s, src) and np.array_equal(d, dst) and np.array_equal(a, act)
    print(f"read_aut threads={threads or os.cpu_count()}: {dt:.2f} s, {m / dt / 1e6:.1f} M transitions/s, "
          f"{size / dt / 1e9:.2f} GB/s, correct={ok}")
os.remove(path)
