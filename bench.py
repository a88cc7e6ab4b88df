#!/usr/bin/env python
"""Benchmark of the B200 refinement path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl b200|reference]

A step is one complete coarsest-partition computation (preprocessing, label
pre-partition, refinement loop) of one synthetic LTS.  Default workload:
config c5 -- a VLTS-shaped lifted-quotient LTS with n = 10M
states, m = 100M transitions, |Act| = 32, one independent instance per GPU
(seed = rank), so the job weak-scales with no data-path collective.  With
--gpus N > 1 and no launcher, bench.py relaunches itself under
torch.distributed.run (one process per GPU).

`value` = (n+m) x K x N / max-over-ranks device time of K steps with inputs
resident in HBM (CUDA events on the library's stream).  `e2e` = the same
metric through the host C-ABI entry point (bisim_bcrp_ex: pinned host arrays
in, H2D + D2H inside the timed region); `e2e_api` = through the public
Python call bcrp_arrays with ordinary numpy arrays.  The result is checked
against the RunStats and block digest of a CPU-oracle run to completion
(tests/golden/scale/).  `--impl reference` times the CPU oracle port of the
reference algorithm on the same workload (rank 0 only; see CpuSampler).
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

SCALE_FIXTURES = os.path.join(ROOT, "tests", "golden", "scale")


def oracle_runstats(config: str):
    """RunStats of the seed-0 instance of `config` from a CPU-oracle run to
    completion (tests/golden/scale/, oracle/gen_scale.py) -- the round count
    the reference arm extrapolates with, and the GPU result's check."""
    path = os.path.join(SCALE_FIXTURES, f"{config}.fast.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError:
        return None


def config_dict(config: str, inst, desc: str, world: int) -> dict:
    """The `config` object both arms print (identical by construction)."""
    rec = oracle_runstats(config) or {}
    return {"workload": desc, "n": inst.n, "m": inst.m, "num_actions": inst.num_actions,
            "kind": inst.kind, "supersteps": rec.get("supersteps"),
            "initial_blocks": rec.get("initial_blocks"), "final_blocks": rec.get("final_blocks"),
            "parallelism": f"replicas x{world} (one independent LTS per GPU)",
            "l2": _l2_note(inst)}


def _l2_note(inst) -> str:
    w = 12 if inst.kind == "bcrp" else 8
    gb = w * inst.m / 1e9
    if gb > 0.126:
        return "inputs (%d B x m = %.2f GB) exceed the 126 MB L2; no flush" % (w, gb)
    return "inputs (%d B x m = %.1f MB) fit in L2 (small config; no flush)" % (w, gb * 1e3)


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
        # nvidia-smi needs ~0.5-1 s to start: wait for its first sample, so
        # a short timed region (the default 5 steps ~0.45 s) is still sampled
        t0 = time.perf_counter()
        while not self.lines and self.proc.poll() is None and time.perf_counter() - t0 < 10.0:
            time.sleep(0.02)
        self.lines.clear()  # keep only samples taken inside the timed region
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


class CpuSampler:
    """The reference algorithm on the host cores (oracle port, all threads),
    timed on a bounded sample of the workload.

    Setup -- preprocessing and the label pre-partition (BCRP) or pi0 (RCPP)
    -- runs once and is timed once.  Main-loop rounds are timed in `nwin`
    windows of `window` rounds whose starts are spread evenly over the run
    (first round to last): the literal oracle resumes from the program state
    the event-driven oracle reports after round r0 (oracle.fast_states,
    untimed setup).  Per-round cost varies along a run (c5: rounds 1-11 cost
    ~2.5x the rounds of the second half, where the big blocks have already
    split), so the windows are a stratified sample and the estimate of one
    complete run is t_pre + t_label + R x (mean of the windows' ms/round),
    R from the oracle's own complete run (tests/golden/scale/).
    """

    def __init__(self, config: str, inst, window: int, nwin: int):
        from oracle import oracle
        # all host threads, except where OpenMP fork/join per phase would
        # cost more than the phase (small systems run fastest on one core)
        self.threads = max(1, min(os.cpu_count() or 1, (inst.n + inst.m) // 250_000))
        rec = oracle_runstats(config)
        if rec is None:
            raise SystemExit(f"bench: no oracle fixture for {config} (oracle/gen_scale.py)")
        self.R = int(rec["supersteps"])
        self.window = max(1, min(window, self.R))
        self.run = oracle.OracleRun(inst, self.threads)
        block0 = self.run.block()
        unstable0 = np.zeros(inst.n, np.uint8)
        unstable0[block0] = 1
        last = max(self.R - self.window, 0)
        nwin = max(1, min(nwin, last + 1))
        starts = sorted({(k * last) // max(nwin - 1, 1) for k in range(nwin)})
        later = [r for r in starts if r > 0]
        states = oracle.fast_states(inst, later, threads=self.threads) if later else ([], [])
        by_round = {r: (states[0][i], states[1][i]) for i, r in enumerate(later)}
        by_round[0] = (block0, unstable0)
        self.windows = [(r, by_round[r]) for r in starts]
        self.samples = {r: [] for r in starts}  # seconds per round, per window

    def step(self, i: int) -> float:
        """Time one window (cycling through the windows); returns seconds."""
        r0, (block, unstable) = self.windows[i % len(self.windows)]
        self.run.set_state(block, unstable)
        k, sec = self.run.rounds(min(self.window, self.R - r0))
        if k:
            self.samples[r0].append(sec / k)
        return sec

    def estimate(self):
        per = {r: statistics.mean(v) for r, v in self.samples.items() if v}
        per_round = statistics.mean(per.values())
        t = self.run.t_pre_s + self.run.t_label_s + self.R * per_round
        rounds = sum(len(v) for v in self.samples.values()) * self.window
        ms = sorted(x * 1e3 for x in per.values())
        desc = (f"oracle port (oracle/bisim_oracle.c, literal O(n+m) rounds, OpenMP "
                f"{self.threads} threads): setup (preprocessing + "
                f"label pre-partition / pi0) timed once = {self.run.t_pre_s + self.run.t_label_s:.2f} s; "
                f"{rounds} main-loop rounds timed in {len(per)} windows of {self.window} rounds "
                f"starting evenly from round 1 to {self.windows[-1][0] + 1} of R = {self.R} "
                f"({ms[0]:.3f} .. {ms[-1]:.3f} ms/round, mean {per_round * 1e3:.3f}); "
                f"total extrapolated as t_setup + R x mean ms/round")
        return t, per_round, desc

    def close(self):
        self.run.close()


def cpu_baseline(config: str, inst, window: int = 21, nwin: int = 10) -> dict:
    """cpu_baseline of the GPU arm's line (rank 0, N=1): ten windows."""
    cs = CpuSampler(config, inst, window, nwin)
    try:
        for i in range(nwin):
            cs.step(i)
        t, per_round, desc = cs.estimate()
    finally:
        cs.close()
    return {"value": (inst.n + inst.m) / t, "unit": UNIT, "cores": cs.threads, "kind": "port",
            "sample": desc, "t_total_s": t, "ms_per_round": per_round * 1e3}


def run_reference(args):
    """Reference arm: the reference algorithm (oracle port) on the host cores,
    same workload, config and metric as the GPU arm; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    inst, desc = make_instance(args.config, 0)
    steps_total = args.warmup + args.steps
    # one window per timed step (up to 20), >= 210 timed rounds in total
    nwin = max(2, min(args.steps, 20))
    window = max(10, -(-210 // max(args.steps, 1)))
    cs = CpuSampler(args.config, inst, window, nwin)
    try:
        for i in range(steps_total):
            if i == args.warmup:
                for v in cs.samples.values():
                    v.clear()
            cs.step(i - args.warmup)  # timed step k runs window k
        t, per_round, sample = cs.estimate()
    finally:
        cs.close()
    value = (inst.n + inst.m) / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic", "config": config_dict(args.config, inst, desc, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cs.threads, "kind": "port",
                             "sample": sample},
            "ms_per_round": per_round * 1e3,
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


def empty_round_floors_us(device: int, n: int = 20000) -> dict:
    """Latency floor of one refinement round: RCPP on an edge-free system
    with a discrete pi0 runs n rounds whose splitter has no in-edge (pure
    control), one by one (no bulk retirement).  `solo`: such rounds run on
    one CTA with __syncthreads (the schedule small rounds get); `grid`: every
    round on the whole grid with its two grid barriers (the schedule c5's
    rounds pay)."""
    from paper_2105_11788_b200 import _native as N
    from paper_2105_11788_b200 import rcpp_arrays
    empty = np.zeros(0, np.int32)
    out = {}
    for name, flags in (("solo", N.FLAG_NO_SKIP), ("grid", N.FLAG_NO_SKIP | N.FLAG_NO_SOLO)):
        _, st, ns = rcpp_arrays(n, empty, empty, np.arange(n, dtype=np.int32), device=device,
                                flags=flags)
        out[name] = ns["t_alg_ms"] * 1e3 / max(st.supersteps, 1)
    return out


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

    # warm-up + correctness: the coarsest partition and RunStats of the
    # oracle's complete run (tests/golden/scale/) or the analytic truth
    first = None
    for _ in range(args.warmup):
        first = step_device()
    if first is None:
        first = step_device()
    blk = d_block.cpu().numpy()
    parity = {}
    if inst.truth is not None:
        parity["vs_truth"] = bool(np.array_equal(blk, inst.truth))
    rec = oracle_runstats(args.config) if rank == 0 else None
    if rec is not None:
        import hashlib
        sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, dtype="<i4").tobytes()).hexdigest()
        R0 = int(first.supersteps)
        parity["vs_oracle_runstats"] = bool(
            R0 == rec["supersteps"] and first.initial_blocks == rec["initial_blocks"]
            and first.final_blocks == rec["final_blocks"] and sha(blk) == rec["block_sha256"]
            and sha(splits[:R0]) == rec["splits_sha256"])
    if False in parity.values():
        raise SystemExit(f"bench: GPU result differs from the reference program ({parity})")

    with ClockSampler(local) as clocks:
        ms, sts = timed(step_device, args.steps)
    clk = clocks.summary()
    for _ in range(1):
        step_host()  # warm the host path (pinned buffers, context)
    ms_e2e, sts_e2e = timed(step_host, args.steps)
    if inst.truth is not None and not np.array_equal(h_block, inst.truth):
        raise SystemExit("bench: host-path result differs from the known coarsest partition")

    # e2e through the public Python API with ordinary (pageable) numpy arrays
    from paper_2105_11788_b200 import bcrp_arrays, rcpp_arrays

    def step_api():
        if inst.kind == "bcrp":
            return bcrp_arrays(n, inst.src, inst.act, inst.dst, inst.num_actions, device=local)
        return rcpp_arrays(n, inst.src, inst.dst, inst.pi0, device=local)

    step_api()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        blk_api = step_api()[0]
    ms_api = reduce_max((time.perf_counter() - t0) * 1e3, dev)
    if inst.truth is not None and not np.array_equal(blk_api, inst.truth):
        raise SystemExit("bench: public-API result differs from the known coarsest partition")

    floors = empty_round_floors_us(local) if rank == 0 else None

    R = sts[0].supersteps
    value = job_throughput(n + m, args.steps, world, ms)
    e2e = job_throughput(n + m, args.steps, world, ms_e2e)
    t_alg = statistics.mean(s.t_alg_ms for s in sts)
    bytes_alg = statistics.mean(s.bytes_alg for s in sts)
    peak, peak_kind = measured_peak_hbm()
    achieved = bytes_alg / (t_alg / 1e3) / 1e9
    launches = sum(s.kernel_launches for s in sts)
    h2d = int(4 * m * (3 if inst.kind == "bcrp" else 2) + (4 * n if inst.kind == "rcpp" else 0))
    # bytes that cross PCIe: the library narrows the actions of a large
    # labelled system to 1 byte on the host first (capi.cu, pipelined path)
    narrowed = inst.kind == "bcrp" and inst.num_actions <= 256 and m >= (1 << 22)
    pcie = h2d - 3 * m if narrowed else h2d
    d2h = int(4 * n + 4 * R)

    result = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu:
            cpu = cpu_baseline(args.config, inst)
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(prof):
            with open(prof) as fh:
                traffic = json.load(fh).get("dram_bytes_per_launch")
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config_dict(args.config, inst, desc, world),
            "parity": parity,
            "ms_to_partition": ms / args.steps,
            "phase_ms": {"pre": statistics.mean(s.t_pre_ms for s in sts),
                         "label": statistics.mean(s.t_label_ms for s in sts),
                         "alg": t_alg},
            "per_round_us": t_alg * 1e3 / max(R, 1),
            "per_round_floor_us": floors,
            "rounds_retired": sts[0].rounds_retired,
            "e2e": {"value": e2e, "unit": UNIT, "ms_per_step": ms_e2e / args.steps,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "pcie_h2d_bytes_per_step": pcie,
                    "path": "C ABI bisim_bcrp_ex/bisim_rcpp_ex, pinned host arrays, CUDA events"},
            "e2e_api": {"value": job_throughput(n + m, args.steps, world, ms_api), "unit": UNIT,
                        "ms_per_step": ms_api / args.steps, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h,
                        "path": "bcrp_arrays/rcpp_arrays, pageable numpy arrays, wall clock"},
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


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


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
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    args = ap.parse_args()
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1 and not args.sharded:
        # one process per GPU: relaunch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args)
    if args.sharded:
        return run_sharded_bench(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
