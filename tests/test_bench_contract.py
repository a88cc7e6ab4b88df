"""bench.py contract (CPU): both arms print the same config for a workload,
the round counts they use come from CPU-oracle runs to completion (not from
the GPU), and the reference arm runs end to end on a small config."""
import json
import os
import subprocess
import sys

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_oracle_runstats_cover_all_configs():
    for c in ("c1", "c2", "c3", "c4u", "c4l", "c5", "c5s"):
        rec = bench.oracle_runstats(c)
        assert rec is not None and rec["oracle"] == "fast" and rec["config"] == c
    assert bench.oracle_runstats("c3")["supersteps"] == 2 * 200_000 - 2   # chain: 2n-2


def test_c1_runstats_are_the_reference_run():
    import _golden as G
    meta, _ = G.c1()
    rec = bench.oracle_runstats("c1")
    assert (rec["supersteps"], rec["initial_blocks"], rec["final_blocks"]) == \
        (meta["supersteps"], meta["initial_blocks"], meta["final_blocks"])


def test_reference_arm_runs_and_matches_config():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    inst, desc = bench.make_instance("c1", 0)
    assert line["config"] == bench.config_dict("c1", inst, desc, 1)
    assert line["config"]["supersteps"] == 13962
    assert line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "1",
                          "--impl", "reference", "--config", "c1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_gpus_n_self_launches_one_process_per_rank():
    """`bench.py --gpus 2` without a launcher relaunches itself under
    torch.distributed.run; the reference arm then prints one line (rank 0)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
