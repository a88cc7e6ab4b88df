"""Time the public bcrp_arrays call on c5 with pageable numpy inputs (developer probe)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import make_instance  # noqa: E402
from paper_2105_11788_b200 import bcrp_arrays  # noqa: E402

inst, _ = make_instance(sys.argv[1] if len(sys.argv) > 1 else "c5", 0)
ts = []
for _ in range(6):
    t = time.perf_counter()
    block, st, ns = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
    ts.append((time.perf_counter() - t) * 1e3)
print(os.environ.get("BISIM_STAGE_THREADS", "default"), "ms", sorted(ts)[1:4], "dev", ns["t_pre_ms"] + ns["t_label_ms"] + ns["t_alg_ms"] + ns["t_h2d_ms"])
