"""Time the transition-sharded mode against the single-replica loop.

    python tools/run_sharded.py c5 0,0        # two replicas sharing GPU 0
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from bench import make_instance  # noqa: E402
from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays  # noqa: E402
from paper_2105_11788_b200.sharded import bcrp_sharded_arrays, rcpp_sharded_arrays  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
devices = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,0").split(",")]
inst, desc = make_instance(cfg, 0)
for label, fn in (("single", None), ("sharded", devices)):
    for rep in range(2):
        t = time.perf_counter()
        if inst.kind == "bcrp":
            if fn is None:
                block, st, ns = bcrp_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions)
            else:
                block, st, ns = bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst,
                                                    inst.num_actions, fn, verify=True)
        else:
            if fn is None:
                block, st, ns = rcpp_arrays(inst.n, inst.src, inst.dst, inst.pi0)
            else:
                block, st, ns = rcpp_sharded_arrays(inst.n, inst.src, inst.dst, inst.pi0, fn,
                                                    verify=True)
        ok = None if inst.truth is None else bool(np.array_equal(block, inst.truth))
        print(cfg, label, devices if fn else [0], f"R={st.supersteps} alg={ns['t_alg_ms']:.2f}ms "
              f"us/round={ns['t_alg_ms'] * 1e3 / max(st.supersteps, 1):.2f} "
              f"wall={1e3 * (time.perf_counter() - t):.0f}ms ok={ok}", flush=True)
