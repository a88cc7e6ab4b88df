"""Summarise tools/ab_proc.sh output: median / mean / spread per (config, lib)."""
import collections
import statistics
import sys

runs = collections.defaultdict(list)
for line in open(sys.argv[1]) if len(sys.argv) > 1 else sys.stdin:
    f = line.split()
    if len(f) == 3:
        runs[(f[0], f[1])].append(float(f[2]))
for c in sorted({k[0] for k in runs}):
    a, b = runs.get((c, "A"), []), runs.get((c, "B"), [])
    if a and b:
        ma, mb = statistics.median(a), statistics.median(b)
        print(f"{c:5s} A med {ma:9.2f} (n={len(a)}, {min(a):.1f}-{max(a):.1f})  "
              f"B med {mb:9.2f} (n={len(b)}, {min(b):.1f}-{max(b):.1f})  B/A {mb / ma:.3f}")
