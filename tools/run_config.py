"""Run one refinement of a benchmark config once (for ncu captures).

    python tools/run_config.py c1 [sparse|dense] [repeats]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import make_instance  # noqa: E402
from paper_2105_11788_b200 import _native as N  # noqa: E402
from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
mode = {"sparse": N.MODE_AUTO, "dense": N.MODE_DENSE}[sys.argv[2] if len(sys.argv) > 2 else "sparse"]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if cfg.startswith("chain"):  # e.g. chain50000: a smaller c3 for profiling
    from paper_2105_11788_b200 import workloads as W
    inst, desc = W.chain(int(cfg[5:])), cfg
else:
    inst, desc = make_instance(cfg, 0)
for _ in range(reps):
    t = time.perf_counter()
    if inst.kind == "bcrp":
        block, st, ns = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, mode=mode)
    else:
        block, st, ns = rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0, mode=mode)
    print(cfg, desc, f"R={st.supersteps} alg={ns['t_alg_ms']:.2f}ms "
          f"wall={1e3 * (time.perf_counter() - t):.1f}ms bytes={ns['bytes_alg']}")
