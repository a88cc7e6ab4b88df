#!/usr/bin/env python
"""Benchmark of the B200 refinement path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl b200|reference]

A step is one complete coarsest-partition computation (preprocessing, label
pre-partition, refinement loop) of one synthetic LTS.  Default workload:
config c5 -- a VLTS-shaped lifted-quotient LTS with n = 10M
states, m = 100M transitions, |Act| = 32, one independent instance per GPU
(seed = rank), so the job weak-scales with no data-path collective.

`value` = (n+m) x K x N / max-over-ranks device time of K steps with inputs
resident in HBM (CUDA events on the library's stream).  `e2e` = the same
metric through the host C-ABI entry point (bisim_bcrp: pinned host arrays
in, H2D + D2H inside the timed region).  `--impl reference` times the CPU
oracle port of the reference algorithm on the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "(n+m)/s to coarsest partition"
UNIT = "(n+m)/s"

# Round counts of the default-seed workloads, measured by the GPU path and
# pinned by tests/test_bench_contract.py; the CPU reference arm extrapolates
# its sampled per-round time with them.
KNOWN_SUPERSTEPS = {"c5": 6113, "c1": 13962, "c2": 1201621, "c3": 399998, "c4u": 5006404,
                    "c4l": 24344}


def make_instance(config: str, rank: int):
    from paper_2105_11788_b200 import workloads as W
    if config == "c5":
        return W.c5_vlts(seed=rank), "c5_vlts: lifted quotient n=10M m=100M |Act|=32 k=5000, one per GPU"
    if config == "c1":
        return W.c1_random(), "c1_random: n=10k m=50k |Act|=4 random.Random(1)"
    if config == "c2":
        return W.c2_kripke(seed=2 + rank), "c2_kripke: RCPP n=1M m=5M out-degree 5, 4-colour pi0"
    if config == "c3":
        return W.chain(200_000), "c3_chain: BCRP chain n=200k (2n-2 rounds)"
    if config == "c4u":
        return W.c4_uniform(seed=4 + rank), "c4_uniform: n=5M m=50M |Act|=256 iid"
    if config == "c4l":
        return W.c4_lifted(seed=44 + rank), "c4_lifted: n=5M m=50M |Act|=256 lifted quotient"
    if config == "c5s":
        return (W.c5_vlts(n=40_000_000, k=20_000, seed=40),
                "c5_sharded: lifted quotient n=40M m=400M |Act|=32 k=20000, one LTS")
    raise SystemExit(f"unknown config {config}")


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def cpu_sample(inst, supersteps: int, budget_s: float = 20.0):
    """Time the oracle port (all host threads) on a bounded sample of the
    workload: preprocessing + label/pi0 setup + K main-loop rounds, then
    extrapolate to R = `supersteps` rounds."""
    from oracle import oracle
    threads = os.cpu_count() or 1
    kw = dict(threads=threads)
    probe = 2
    t0 = time.perf_counter()
    if inst.kind == "bcrp":
        r = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, stop_after=probe, **kw)
    else:
        r = oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, stop_after=probe, **kw)
    wall = time.perf_counter() - t0
    per_round = r.t_loop_s / max(r.supersteps, 1)
    K = max(probe, min(supersteps, int(max(budget_s - wall, 0) / max(per_round, 1e-9))))
    if K > probe:
        if inst.kind == "bcrp":
            r = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions, stop_after=K, **kw)
        else:
            r = oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, stop_after=K, **kw)
        per_round = r.t_loop_s / max(r.supersteps, 1)
    done = r.supersteps
    t_est = r.t_pre_s + r.t_label_s + per_round * supersteps
    exact = done >= supersteps
    sample = (f"oracle port (oracle/bisim_oracle.c, OpenMP {threads} threads): preprocessing + "
              f"{'label pre-partition' if inst.kind == 'bcrp' else 'pi0 setup'} + {done} of "
              f"{supersteps} main-loop rounds timed; "
              + ("complete run" if exact else
                 f"total extrapolated as t_pre + t_label + R x {per_round * 1e3:.3f} ms/round"))
    return (inst.n + inst.m) / t_est, t_est, threads, sample


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    inst, desc = make_instance(args.config, 0)
    R = KNOWN_SUPERSTEPS.get(args.config)
    if R is None:
        from oracle import oracle
        if inst.kind == "bcrp":
            R = oracle.bcrp(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                            threads=os.cpu_count()).supersteps
        else:
            R = oracle.rcpp(inst.n, inst.src, inst.dst, inst.pi0, threads=os.cpu_count()).supersteps
    vals, times = [], []
    for step in range(args.warmup + args.steps):
        v, t, cores, sample = cpu_sample(inst, R, budget_s=args.cpu_budget)
        if step >= args.warmup:
            vals.append(v)
            times.append(t)
    value = statistics.mean(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": {"workload": desc, "n": inst.n, "m": inst.m,
                                            "supersteps": R},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def reduce_max(value: float, device=None) -> float:
    """Max over ranks (identity without a process group); timing rule: the
    job time is the slowest rank's device time."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(units_per_rank: int, steps: int, world: int, ms_max: float) -> float:
    """Whole-job (n+m)/s: every rank refines its own LTS `steps` times."""
    return units_per_rank * steps * world / (ms_max / 1e3)


def empty_round_floor_us(device: int, n: int = 20000) -> float:
    """Latency floor of one refinement round: RCPP on an edge-free system
    with a discrete pi0 runs n rounds whose splitter has no in-edge (pure
    control + barriers); no-op retirement disabled so every round runs."""
    from paper_2105_11788_b200 import rcpp_arrays
    old = os.environ.get("BISIM_NO_SKIP")
    os.environ["BISIM_NO_SKIP"] = "1"
    try:
        empty = np.zeros(0, np.int32)
        _, st, ns = rcpp_arrays(n, empty, empty, np.arange(n, dtype=np.int32), device=device)
    finally:
        if old is None:
            del os.environ["BISIM_NO_SKIP"]
        else:
            os.environ["BISIM_NO_SKIP"] = old
    return ns["t_alg_ms"] * 1e3 / max(st.supersteps, 1)


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2105_11788_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    inst, desc = make_instance(args.config, rank)
    n, m = inst.n, inst.m
    L = N.lib()
    dev = torch.device("cuda", local)
    d_src = torch.from_numpy(inst.src).to(dev)
    d_dst = torch.from_numpy(inst.dst).to(dev)
    d_act = torch.from_numpy(inst.act).to(dev) if inst.kind == "bcrp" else None
    d_pi0 = torch.from_numpy(inst.pi0).to(dev) if inst.kind == "rcpp" else None
    d_block = torch.empty(n, dtype=torch.int32, device=dev)
    cap = 3 * n + 16
    splits = np.zeros(cap, np.int32)
    opt = N.Options()
    opt.device = local
    opt.mode = N.MODE_AUTO
    torch.cuda.synchronize()

    def step_device():
        st = N.Stats()
        if inst.kind == "bcrp":
            rc = L.bisim_bcrp_device(n, m, inst.num_actions, d_src.data_ptr(), d_act.data_ptr(),
                                     d_dst.data_ptr(), N.DEFAULT_GUARD, d_block.data_ptr(),
                                     N.ptr(splits), cap, ctypes.byref(st), ctypes.byref(opt))
        else:
            rc = L.bisim_rcpp_device(n, m, d_src.data_ptr(), d_dst.data_ptr(), d_pi0.data_ptr(),
                                     N.DEFAULT_GUARD, d_block.data_ptr(), N.ptr(splits), cap,
                                     ctypes.byref(st), ctypes.byref(opt))
        N.check(rc)
        return st

    # pinned host buffers for the end-to-end (host C-ABI) measurement
    h_src = torch.from_numpy(inst.src).pin_memory().numpy()
    h_dst = torch.from_numpy(inst.dst).pin_memory().numpy()
    h_act = torch.from_numpy(inst.act).pin_memory().numpy() if inst.kind == "bcrp" else None
    h_pi0 = torch.from_numpy(inst.pi0).pin_memory().numpy() if inst.kind == "rcpp" else None
    h_block = torch.empty(n, dtype=torch.int32).pin_memory().numpy()

    def step_host():
        st = N.Stats()
        if inst.kind == "bcrp":
            rc = L.bisim_bcrp_ex(n, m, inst.num_actions, N.ptr(h_src), N.ptr(h_act), N.ptr(h_dst),
                                 N.DEFAULT_GUARD, N.ptr(h_block), N.ptr(splits), cap,
                                 ctypes.byref(st), ctypes.byref(opt))
        else:
            rc = L.bisim_rcpp_ex(n, m, N.ptr(h_src), N.ptr(h_dst), N.ptr(h_pi0), N.DEFAULT_GUARD,
                                 N.ptr(h_block), N.ptr(splits), cap, ctypes.byref(st),
                                 ctypes.byref(opt))
        N.check(rc)
        return st

    ext = torch.cuda.ExternalStream(L.bisim_stream(local), device=dev)

    def timed(fn, k):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ext)
        sts = [fn() for _ in range(k)]
        e1.record(ext)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return reduce_max(e0.elapsed_time(e1), dev), sts

    # warm-up + correctness check against the known coarsest partition
    first = None
    for _ in range(args.warmup):
        first = step_device()
    if first is None:
        first = step_device()
    blk = d_block.cpu().numpy()
    correct = None
    if inst.truth is not None:
        correct = bool(np.array_equal(blk, inst.truth))
    if inst.expect_supersteps is not None:
        correct = (correct is not False) and first.supersteps == inst.expect_supersteps
    if correct is False:
        raise SystemExit("bench: GPU result differs from the known coarsest partition")

    with ClockSampler(local) as clocks:
        ms, sts = timed(step_device, args.steps)
    clk = clocks.summary()
    for _ in range(1):
        step_host()  # warm the host path (pinned buffers, context)
    ms_e2e, sts_e2e = timed(step_host, args.steps)
    if inst.truth is not None and not np.array_equal(h_block, inst.truth):
        raise SystemExit("bench: host-path result differs from the known coarsest partition")

    floor_us = empty_round_floor_us(local) if rank == 0 else None

    R = sts[0].supersteps
    value = job_throughput(n + m, args.steps, world, ms)
    e2e = job_throughput(n + m, args.steps, world, ms_e2e)
    t_alg = statistics.mean(s.t_alg_ms for s in sts)
    bytes_alg = statistics.mean(s.bytes_alg for s in sts)
    peak, peak_kind = measured_peak_hbm()
    achieved = bytes_alg / (t_alg / 1e3) / 1e9
    launches = sum(s.kernel_launches for s in sts)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            v, t_est, cores, sample = cpu_sample(inst, R, budget_s=args.cpu_budget)
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                   "t_total_s": t_est}
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(prof):
            with open(prof) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": desc, "n": n, "m": m, "num_actions": inst.num_actions,
                       "kind": inst.kind, "supersteps": R,
                       "initial_blocks": sts[0].initial_blocks,
                       "final_blocks": sts[0].final_blocks,
                       "parallelism": f"replicas x{world} (one independent LTS per GPU)",
                       "l2": "inputs (12 B x m = %.2f GB) exceed L2; no flush" % (12 * m / 1e9),
                       "correct_vs_truth": correct},
            "ms_to_partition": ms / args.steps,
            "phase_ms": {"pre": statistics.mean(s.t_pre_ms for s in sts),
                         "label": statistics.mean(s.t_label_ms for s in sts),
                         "alg": t_alg},
            "per_round_us": t_alg * 1e3 / max(R, 1),
            "per_round_floor_us": floor_us,
            "rounds_retired": sts[0].rounds_retired,
            "e2e": {"value": e2e, "unit": UNIT, "ms_per_step": ms_e2e / args.steps,
                    "h2d_bytes_per_step": int(4 * m * (3 if inst.kind == "bcrp" else 2)
                                              + (4 * n if inst.kind == "rcpp" else 0)),
                    "d2h_bytes_per_step": int(4 * n + 4 * R)},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_refine_sparse (persistent refinement loop)",
                         "peak_source": peak_kind,
                         "bytes_per_launch": bytes_alg, "launch_ms": t_alg},
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded_bench(args):
    """One LTS split over the replicas of the transition-sharded mode
    (csrc/kernels_shard.cuh): devices 0..gpus-1, or `--virtual K` replicas
    sharing device 0 (correctness/overhead only).  Under torchrun rank 0
    drives every device and the other ranks only wait."""
    import torch
    import torch.distributed as dist

    from paper_2105_11788_b200.sharded import bcrp_sharded_arrays, rcpp_sharded_arrays

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return 0
    devices = [0] * args.virtual if args.virtual else list(range(args.gpus))
    inst, desc = make_instance(args.config, 0)

    def step():
        if inst.kind == "bcrp":
            return bcrp_sharded_arrays(inst.n, inst.src, inst.act, inst.dst, inst.num_actions,
                                       devices)
        return rcpp_sharded_arrays(inst.n, inst.src, inst.dst, inst.pi0, devices)

    for _ in range(args.warmup):
        block, st, ns = step()
    correct = None if inst.truth is None else bool(np.array_equal(block, inst.truth))
    if correct is False:
        raise SystemExit("bench: sharded result differs from the known coarsest partition")
    dev_ms, wall_ms = [], []
    with ClockSampler(0) as clocks:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            t = time.perf_counter()
            block, st, ns = step()
            wall_ms.append((time.perf_counter() - t) * 1e3)
            dev_ms.append(ns["t_pre_ms"] + ns["t_label_ms"] + ns["t_alg_ms"])
    ms = statistics.mean(dev_ms)
    units = inst.n + inst.m
    line = {
        "metric": METRIC, "value": units / (ms / 1e3), "unit": UNIT, "n_gpus": len(set(devices)),
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": desc, "n": inst.n, "m": inst.m, "supersteps": st.supersteps,
                   "parallelism": f"transition-sharded x{len(devices)} replicas on devices {devices}",
                   "correct_vs_truth": correct},
        "per_round_us": ns["t_alg_ms"] * 1e3 / max(st.supersteps, 1),
        "phase_ms": {"pre": ns["t_pre_ms"], "label": ns["t_label_ms"], "alg": ns["t_alg_ms"]},
        "e2e": {"value": units / (statistics.mean(wall_ms) / 1e3), "unit": UNIT,
                "ms_per_step": statistics.mean(wall_ms),
                "h2d_bytes_per_step": int(12 * inst.m * len(devices)),
                "d2h_bytes_per_step": int(4 * inst.n + 4 * st.supersteps)},
        "clocks": clocks.summary(),
        "gpu_launches": int(ns["kernel_launches"]) * args.steps,  # loop kernels (one per replica)
        "note": "value: device time of preprocessing + label rounds + loop (max over replicas); "
                "inputs copied to every replica inside e2e",
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=["c5", "c1", "c2", "c3", "c4u", "c4l", "c5s"])
    ap.add_argument("--sharded", action="store_true",
                    help="one LTS over --gpus devices (transition-sharded mode)")
    ap.add_argument("--virtual", type=int, default=0,
                    help="with --sharded: this many replicas sharing GPU 0 (testing)")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.sharded:
        return run_sharded_bench(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
