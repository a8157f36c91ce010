#!/usr/bin/env python
"""Benchmark: TNRD/TRDPD Poisson-denoising inference on B200 (BASELINE.json metric
"denoised MPix/s (48x7x7, T=8, fp32) at 1/2/4/8 B200; % of FP32 roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4|5|3] [--impl ours|reference]

A step is one full inference pass (T = 8 fused stage launches) over the
workload: by default BASELINE.json configs[3] (C4: 256 independent 512x512
images, 48 7x7 filters, 63 RBFs, T = 8), its images sharded over the ranks
(no data-path collective).  --config 5 runs C5 (one 8192^2 image) as row slabs
with the per-stage NCCL halo exchange.  Both configs fix the total work, so N > 1
is reported as "scaling": "strong".

For N > 1: under torchrun (WORLD_SIZE set) one process per GPU; launched plainly
with --gpus N, bench.py re-launches itself through torch.distributed.run with N
ranks (an error if fewer than N GPUs are visible).  --dry-run runs the same
multi-rank plumbing on CPU with gloo (shards, barriers, max-over-ranks) without
touching a GPU (tests/test_multiproc_gloo.py).  Rank 0 prints one JSON line.
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks.  Inputs (~0.8 GB resident per step) exceed the 126 MB L2,
so no flush is needed.  See DESIGN.md §8.
"""
from __future__ import annotations

import argparse
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

F_ALG = lambda Nk, k, M: 4 * Nk * k * k + 2 * Nk * M + 10  # flop / pixel / stage
# tabulated phi does not claim the RBF work it avoids: one cubic (8 flop) per response
F_TAB = lambda Nk, k, M: 4 * Nk * k * k + 8 * Nk + 10
METRIC = "denoised MPix/s (48x7x7, T=8, fp32) at 1/2/4/8 B200; % of FP32 roofline"


def fp32_peak_tflops(n_sm: int, mhz: float) -> float:
    """FP32 FMA roofline: n_SM x 128 lanes x 2 flop x clock."""
    return n_sm * 128 * 2 * mhz * 1e6 / 1e12


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def reference_arm(args, rank, world):
    """--impl reference: the double-precision oracle (oracle/, as it stands) timed on
    the host cores on bounded samples of the same workload."""
    if rank != 0:
        return 0
    import oracle
    from synth import make_problem
    cfg = args.config
    p = make_problem(cfg)
    cores = oracle.num_threads()
    # calibrate: one 32x32 crop, then size each step's sample to ~2 s
    f0 = p.f[0]
    t = time.perf_counter()
    oracle.denoise(f0[:32, :32], p.model)
    per_px = (time.perf_counter() - t) / (32 * 32)
    side = int(np.clip(np.sqrt(2.0 / max(per_px, 1e-9)), 32, min(f0.shape)))
    rng = np.random.default_rng(0)
    times = []
    for s in range(args.warmup + args.steps):
        b = s % p.f.shape[0]
        y = int(rng.integers(0, p.f.shape[1] - side + 1))
        x = int(rng.integers(0, p.f.shape[2] - side + 1))
        t = time.perf_counter()
        oracle.denoise(p.f[b][y:y + side, x:x + side], p.model)
        dt = time.perf_counter() - t
        if s >= args.warmup:
            times.append(dt)
    mpix = side * side / 1e6
    value = mpix * len(times) / sum(times)
    sample = f"{side}x{side} window of a {p.cfg['name']} image per step (T={p.model.T}, Nk={p.model.Nk}, " \
             f"k={p.model.k}, M={p.model.M}), double precision, OpenMP over rows"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MPix/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(p, world, args),
        "cpu_baseline": {"value": value, "unit": "MPix/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "MPix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def parallelism(config, world):
    if world == 1:
        return "single-gpu (no partition)"
    return ("batch-shard" if config != 5 else "row-slab+nccl-halo") + f"x{world}"


L2_BYTES = 126 * 1024 * 1024
L2_FLUSH_BYTES = 256 * 1024 * 1024


def workload_config(p, world, args):
    c = p.cfg
    return {"workload": f"{c['name']}: {c['B']}x{c['H']}x{c['W']} fp32, peaks {c['peaks']}, T={c['T']}, "
                        f"Nk={c['Nk']}, k={c['k']}, M={c['M']} (BASELINE.json configs[{args.config - 1}])",
            "batch": c["B"], "H": c["H"], "W": c["W"], "T": c["T"], "Nk": c["Nk"], "k": c["k"], "M": c["M"],
            "parallelism": parallelism(args.config, world),
            "l2": ("L2 flushed before every step (256 MB memset outside the per-step events): working set "
                   f"{3 * 4 * c['B'] * c['H'] * c['W'] / 1e6:.1f} MB < 126 MB L2"
                   if 3 * 4 * c["B"] * c["H"] * c["W"] / world < L2_BYTES else
                   "no flush: per-step working set (f, u, scratch) > 126 MB L2"),
            "phi": args.phi,
            "flop_per_px_stage": (F_TAB if args.phi == "table" else F_ALG)(c["Nk"], c["k"], c["M"])}


def cpu_baseline(p, budget_s=12.0):
    """The oracle on a bounded sample (rank 0, N = 1 only): whole-image windows of
    the workload, one after another, until ~budget_s of CPU time has been spent."""
    import oracle
    B, H, W = p.f.shape
    f0 = p.f[0]
    t = time.perf_counter()
    oracle.denoise(f0[:32, :32], p.model)
    per_px = (time.perf_counter() - t) / 1024
    side = int(np.clip(np.sqrt(budget_s / max(per_px, 1e-9)), 32, min(H, W)))
    y, x = (H - side) // 2, (W - side) // 2
    n, px, t0 = 0, 0, time.perf_counter()
    while True:
        oracle.denoise(p.f[n % B][y:y + side, x:x + side], p.model)
        n += 1
        px += side * side
        dt = time.perf_counter() - t0
        if dt >= 0.8 * budget_s or n >= 8:
            break
    return {"value": px / 1e6 / dt, "unit": "MPix/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"{n} centred {side}x{side} window(s) of images 0..{n - 1} (T={p.model.T}, full model), "
                      f"double precision, OpenMP over rows, {dt:.1f} s"}


def relaunch(args):
    """bench.py --gpus N without torchrun: re-launch as N ranks on this node through
    torch.distributed.run (rank 0's JSON line is passed through)."""
    if not args.dry_run:
        import torch
        n_vis = torch.cuda.device_count()
        if args.gpus > n_vis:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {n_vis} GPU(s) are visible\n")
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world):
    """--dry-run: the N > 1 plumbing on CPU (gloo): each rank takes its shard of the
    workload exactly as the GPU path does, the timed region is bracketed by
    barriers, the time is the max over ranks, and rank 0 prints one line listing
    every rank's shard.  No GPU, no kernel: a test of the launcher, not a number."""
    import torch
    import torch.distributed as dist
    from paper_1510_02930_b200.partition import batch_shard, slab_rows
    from synth.generator import CONFIGS
    c = CONFIGS[args.config]
    if world > 1:
        dist.init_process_group("gloo")
    shard = slab_rows(c["H"], rank, world) if args.config == 5 else batch_shard(c["B"], rank, world)
    t0 = time.perf_counter()
    if world > 1:
        dist.barrier()
    ms = torch.tensor([1e3 * (time.perf_counter() - t0)], dtype=torch.float64)
    shards = [None] * world
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_gather_object(shards, (rank, shard))
    else:
        shards = [(rank, shard)]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "config": {"workload": c["name"], "parallelism": parallelism(args.config, world)},
                          "scaling": "strong", "shards": [list(s) for _, s in sorted(shards)],
                          "ms_max_over_ranks": float(ms[0])}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def grad_bench(args):
    """Training gradient: one tnrd_loss_grad call per step on image 0 of the config
    (loss against its clean image), CUDA events around each synchronous call."""
    import torch
    import paper_1510_02930_b200 as P
    from synth import make_problem
    cfg = 3 if args.config == 4 else args.config
    p = make_problem(cfg)
    torch.cuda.set_device(0)
    f = torch.from_numpy(p.f[:1]).cuda()
    gt = torch.from_numpy(p.clean[:1]).cuda()
    eng = P.TNRD(p.model, device=0,
                 engine={"auto": P.ENGINE_AUTO, "fp32": P.ENGINE_FP32, "tensor": P.ENGINE_TENSOR}[args.engine])
    t0 = time.perf_counter()
    for _ in range(args.warmup):
        eng.loss_grad(f, gt)
    torch.cuda.synchronize()
    # at least ~0.5 s of timed steps, so the 100 ms clock sampler sees the region
    est = (time.perf_counter() - t0) / max(args.warmup, 1)
    steps = max(args.steps, int(0.5 / max(est, 1e-4)) + 1)
    n0 = P.tnrd_launch_count(eng.h)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        ev0.record()
        for _ in range(steps):
            eng.loss_grad(f, gt)
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    _, H, W = p.f.shape
    line = {"metric": "training-gradient MPix/s (loss + dl/dTheta, P Eq.14-20, fp32)", "mode": "grad",
            "value": H * W / 1e6 / (ms / 1e3), "unit": "MPix/s", "n_gpus": 1, "steps": steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f32",
            "data": "synthetic", "config": {"workload": f"{p.cfg['name']} image 0 vs its clean image, "
                                                        f"T={p.model.T}, Nk={p.model.Nk}, k={p.model.k}, M={p.model.M}",
                                            "engine": args.engine,
                                            "tape_and_banks": "fp32 engine" if args.engine == "fp32" else
                                            "tensor cores (3xTF32, round-to-nearest split) where (k, N_k) has them"},
            "stage_launches_per_step": (P.tnrd_launch_count(eng.h) - n0) // steps,
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)
    eng.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="infer", choices=["infer", "grad"],
                    help="infer: the inference pass (the headline); grad: the training gradient "
                         "(tnrd_loss_grad, P Eq.14-20) on one image of --config (default C3), reported separately")
    ap.add_argument("--phi", default="exact", choices=["exact", "table"],
                    help="exact RBF sum (the headline) or the tabulated variant (reported separately)")
    ap.add_argument("--engine", default="auto", choices=["auto", "fp32", "tensor"],
                    help="stage engine (tnrd_set_engine): auto = tensor cores where they apply")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--launch-events", default="after", choices=["after", "inline"],
                    help="per-launch CUDA events: 'after' = on up to 3 profiled steps right after the timed "
                         "region (default: an event between two stage kernels would serialise the "
                         "programmatic dependent launch that overlaps one stage's set-up with the previous "
                         "stage's tail), 'inline' = around every launch inside the timed region")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU only: the multi-rank plumbing (launch, shards, barriers, max over ranks) "
                         "over gloo without any GPU work")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    rank, world, local = dist_env()
    if args.dry_run:
        return dry_run(args, rank, world)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    if args.mode == "grad":
        return grad_bench(args)

    import torch
    import torch.distributed as dist
    import paper_1510_02930_b200 as P
    from paper_1510_02930_b200.partition import batch_shard, slab_rows
    from synth import make_problem

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    p = make_problem(args.config)
    model = p.model
    B, H, W = p.f.shape
    eng = P.TNRD(model, device=local, phi_mode=P.PHI_TABLE if args.phi == "table" else P.PHI_EXACT,
                 engine={"auto": P.ENGINE_AUTO, "fp32": P.ENGINE_FP32, "tensor": P.ENGINE_TENSOR}[args.engine])
    stream = torch.cuda.current_stream()

    if args.config == 5:
        # row slabs, NCCL halo exchange per stage
        r0, r1 = slab_rows(H, rank, world)
        f_dev = torch.from_numpy(p.f[0, r0:r1]).to(dev)
        u_dev = torch.empty_like(f_dev)
        if world > 1:
            uid = P.tnrd_nccl_unique_id() if rank == 0 else bytes(128)
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            P.tnrd_comm_init(eng.h, obj[0], rank, world)

        def step():
            if world > 1:
                P.tnrd_denoise_slab(eng.h, f_dev, u_dev, H, r0, float(p.peaks[0]))
            else:
                P.tnrd_denoise(eng.h, f_dev[None], u_dev[None])
        px_rank = (r1 - r0) * W
        shard = (r0, r1)
    else:
        b0, b1 = batch_shard(B, rank, world)
        f_dev = torch.from_numpy(p.f[b0:b1]).to(dev)
        u_dev = torch.empty_like(f_dev)
        peaks = p.peaks[b0:b1]

        def step():
            P.tnrd_denoise(eng.h, f_dev, u_dev, peaks)
        px_rank = (b1 - b0) * H * W
        shard = (b0, b1)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    ws_bytes = 3 * 4 * px_rank   # f, u and the ping-pong scratch resident per rank

    for _ in range(args.warmup):
        step()
    barrier()
    n_launch0 = P.tnrd_launch_count(eng.h)
    P.tnrd_set_profiling(eng.h, args.launch_events == "inline")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # inputs smaller than the 126 MB L2 (C1-C3): flush L2 before every step (a 256 MB
    # memset) and time each step alone; C4 / C5 move > 800 MB per step and need none
    flush = L2_FLUSH_BYTES and ws_bytes < L2_BYTES
    if flush:
        scrub = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for k in range(args.steps):
            if flush:
                scrub.zero_()
                evs[k][0].record(stream)
            step()
            if flush:
                evs[k][1].record(stream)
        ev1.record(stream)
        barrier()
    ms = sum(a.elapsed_time(b) for a, b in evs) if flush else ev0.elapsed_time(ev1)
    launches = P.tnrd_launch_count(eng.h) - n_launch0
    launch_ms = P.tnrd_get_launch_times(eng.h)
    P.tnrd_set_profiling(eng.h, False)
    if args.launch_events == "after":   # per-launch times from profiled steps right after the timed region
        P.tnrd_set_profiling(eng.h, True)
        for _ in range(min(args.steps, 3)):
            step()
        torch.cuda.synchronize()
        launch_ms = P.tnrd_get_launch_times(eng.h)
        P.tnrd_set_profiling(eng.h, False)
    clocks = clk.summary()
    t = torch.tensor([ms, float(launches), float(np.mean(launch_ms)) if len(launch_ms) else 0.0], device=dev)
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms, launches = float(tmax[0]), int(tsum[1])
        mean_launch_ms = float(tmax[2])
    else:
        mean_launch_ms = float(t[2])
    ms_per_step = ms / args.steps
    total_px = B * H * W
    value = total_px / 1e6 / (ms_per_step / 1e3)

    # ---- e2e: public host entry point, pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e and args.config != 5:
        f_host = torch.from_numpy(p.f[shard[0]:shard[1]]).pin_memory()
        u_host = torch.empty_like(f_host).pin_memory()
        nb = shard[1] - shard[0]
        P.tnrd_denoise_host_ptr(eng.h, f_host.data_ptr(), u_host.data_ptr(), nb, H, W)  # warm
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k_e2e = max(1, min(args.steps, 5))
        e0.record(stream)
        for _ in range(k_e2e):
            P.tnrd_denoise_host_ptr(eng.h, f_host.data_ptr(), u_host.data_ptr(), nb, H, W)
        e1.record(stream)
        barrier()
        ems = torch.tensor([e0.elapsed_time(e1) / k_e2e], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": total_px / 1e6 / (float(ems[0]) / 1e3), "unit": "MPix/s",
               "h2d_bytes_per_step": int(f_host.numel() * 4), "d2h_bytes_per_step": int(u_host.numel() * 4),
               "steps": k_e2e, "entry_point": "tnrd_denoise_host"}

    if rank == 0:
        props = torch.cuda.get_device_properties(dev)
        n_sm = props.multi_processor_count
        max_mhz = (clocks or {}).get("sm_max_mhz") or 1965.0
        peak = fp32_peak_tflops(n_sm, max_mhz)
        f_px = (F_TAB if args.phi == "table" else F_ALG)(model.Nk, model.k, model.M)
        flop_launch = f_px * px_rank
        tensor = eng.engine_for(B if args.config != 5 else 1, H if args.config != 5 else shard[1] - shard[0],
                                W) == P.ENGINE_TENSOR
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf):
            try:
                traffic = json.load(open(tf)).get(f"C{args.config}" + ("/tensor" if tensor else ""))
            except Exception:
                traffic = None
        secs = mean_launch_ms / 1e3 if mean_launch_ms > 0 else None
        launch_timing = ("CUDA events around every stage launch on the launching stream, " +
                         ("inside the timed region" if args.launch_events == "inline" else
                          f"over {min(args.steps, 3)} profiled steps right after the timed region (events between "
                          "stage kernels would serialise the programmatic dependent launch the timed steps use)"))
        if not tensor:
            achieved = flop_launch / secs / 1e12 if secs else None
            roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                        "kernel": "stage_kernel (FP32 engine, one fused TNRD stage)",
                        "flop_per_px_stage": f_px, "flop_per_launch": flop_launch, "mean_launch_ms": mean_launch_ms,
                        "launch_timing": launch_timing,
                        "peak_source": f"derived: {n_sm} SM x 128 FP32 lanes x 2 x {max_mhz:.0f} MHz "
                                       "(MEASURED_PEAKS.json has no FP32 figure)"}
        else:
            # tensor-core engine: the two filter banks run on the tensor
            # pipe (3xTF32), everything else on the FP32 pipes.  The bound is the FP32
            # side: its algorithmic work is F_alg minus the conv flops (the RBF MACs + prox).
            f_conv = 4 * model.Nk * model.k * model.k
            f_alu = f_px - f_conv
            achieved = f_alu * px_rank / secs / 1e12 if secs else None
            tf32_peak = None
            mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
            if os.path.exists(mp):
                tf32_peak = json.load(open(mp)).get("bf16_tflops")
                tf32_peak = tf32_peak / 2 if tf32_peak else None
            t_ach = f_conv * px_rank / secs / 1e12 if secs else None
            roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                        "kernel": "tc_stage_kernel (tensor-core engine, one fused TNRD stage)",
                        "flop_per_px_stage": f_alu, "flop_per_launch": f_alu * px_rank,
                        "mean_launch_ms": mean_launch_ms, "launch_timing": launch_timing,
                        "peak_source": f"derived: {n_sm} SM x 128 FP32 lanes x 2 x {max_mhz:.0f} MHz "
                                       "(MEASURED_PEAKS.json has no FP32 figure)",
                        "fp32_equivalent_frac": (flop_launch / secs / 1e12 / peak) if secs else None,
                        "tensor": {"flop_per_px_stage": f_conv, "executed_split": "3xTF32 (3 MMAs per product)",
                                   "achieved": t_ach, "peak": tf32_peak,
                                   "frac": (t_ach / tf32_peak) if (t_ach and tf32_peak) else None,
                                   "peak_source": "MEASURED_PEAKS.json bf16_tflops / 2 (TF32 = half the bf16 rate)"}}
        line = {
            "metric": METRIC, "value": value, "unit": "MPix/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 storage; conv products 3xTF32 (tensor engine)" if tensor else "f32",
            "data": "synthetic",
            "config": dict(workload_config(p, world, args), engine="tensor" if tensor else "fp32",
                           conv_arithmetic=("3xTF32 tcgen05: fp32 operands split hi + lo, three TF32 products "
                                            "per term, fp32 accumulation (products exact to < 2^-20 relative); "
                                            "parity margin equal to the FP32 engine's (DESIGN.md §5.11)")
                           if tensor else "fp32 FFMA2"),
            "roofline": roofline,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "device": props.name,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(p)
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
