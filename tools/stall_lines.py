"""Top CUDA source lines by warp-stall samples of an ncu report (run here, no GPU).

    python tools/stall_lines.py gpurun_out/x.ncu-rep profiles/out.txt [top]

Reads `ncu -i REP --page source --csv --print-source cuda,sass` (the
kernel must be built with -lineinfo) and prints "share file:line source".
"""
import csv
import io
import os
import subprocess
import sys


def stall_lines(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows, fname, col = [], "?", None
    for r in csv.reader(io.StringIO(out)):
        if not r:
            continue
        if r[0] == "File Path" and len(r) > 1:
            fname = os.path.basename(r[1])
        elif r[0] == "Line No":
            col = r.index("Warp Stall Sampling (All Samples)")
        elif col is not None and r[0].isdigit() and len(r) > col:
            try:
                rows.append((int(r[col]), f"{fname}:{r[0]}", r[1].strip()))
            except ValueError:
                pass
    return rows


if __name__ == "__main__":
    rows = stall_lines(sys.argv[1])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
    total = sum(r[0] for r in rows) or 1
    lines = [f"{100.0 * n / total:5.1f}% {where} {src[:110]}" for n, where, src in sorted(rows, reverse=True)[:top]]
    with open(sys.argv[2], "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))
