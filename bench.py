"""Benchmark: tiled QR fp64 GFLOP/s (flops = 2 n^2 (m - n/3)) on B200.

Workloads (BASELINE.json configs; synthetic seeded inputs, no datasets):
  c3  16384 x 16384, nb=256, Greedy/TT, N(0,1) seed 2          (default, N=1)
  c4   8192 x 4096,  nb=256, Fibonacci/TT, U diag(s) V^T seed 3
  c5  2,097,152 x 2048, nb=256, Greedy local trees + TT merge of the R factors,
      U(-1,1) seed 4, block rows sharded over the ranks         (default, N>1)
  c1     512 x 256,  nb=64,  Greedy/TT, N(0,1) seed 0

A step = one tiled QR of the workload: pack (row-major A -> tile-major, on
device) + the persistent executor (every GEQRT/UNMQR/TTQRT/TTMQR kernel).
`value` times steps with A resident in HBM; `e2e` times the public API call
with the host->device copy of A (pinned) and the device->host copy of R.

`--gpus N` without a torchrun environment relaunches itself under
torch.distributed.run (one rank per GPU, NCCL); N > 1 lines are C5 and carry
rank 0's same-run one-GPU C5 time (`c5_single_gpu`).

`--impl reference` is the reference arm: the reference package's own CPU
path (tiledag.build_tree, qr.py:622-649, imported from baseline/_ref) plus
the numeric work its trace stands for, executed on the host cores by the
LAPACK tile kernels over the reference's hazard DAG (oracle/cpu_baseline.py)
— this process never loads libtqr.so.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(m=512, n=256, nb=64, algo="greedy", family="TT", seed=0, dist="normal"),
    "c3": dict(m=16384, n=16384, nb=256, algo="greedy", family="TT", seed=2, dist="normal"),
    "c4": dict(m=8192, n=4096, nb=256, algo="fibonacci", family="TT", seed=3, dist="svd"),
    "c5": dict(m=2097152, n=2048, nb=256, algo="greedy", family="TT", seed=4, dist="uniform"),
}
METRIC = "tiled QR fp64 GFLOP/s (2n^2(m-n/3))"


def make_matrix(cfg, rows=None, row0=0):
    """Seeded host matrix (float64, C order).  rows/row0 select a block of
    rows of the full matrix (the same draws for any sharding)."""
    m, n = cfg["m"], cfg["n"]
    rng = np.random.default_rng(cfg["seed"])
    if cfg["dist"] == "normal":
        return rng.standard_normal((m, n))
    if cfg["dist"] == "svd":
        U = np.linalg.qr(rng.standard_normal((m, n)))[0]
        V = np.linalg.qr(rng.standard_normal((n, n)))[0]
        return np.ascontiguousarray((U * np.geomspace(1.0, 1e-12, n)) @ V.T)
    # uniform: row chunk c (65536 rows) drawn from default_rng([seed, c]), so
    # any block of rows is generated without the rows before it
    rows = m if rows is None else rows
    out = np.empty((rows, n))
    chunk = 65536
    for c in range(row0 // chunk, (row0 + rows + chunk - 1) // chunk):
        lo, hi = max(c * chunk, row0), min((c + 1) * chunk, row0 + rows, m)
        blk = np.random.default_rng([cfg["seed"], c]).uniform(-1.0, 1.0, (min(chunk, m - c * chunk), n))
        out[lo - row0:hi - row0] = blk[lo - c * chunk:hi - c * chunk]
    return out


def config_dict(name, cfg, world=1):
    """The `config` object both arms print (same keys, same values)."""
    nb = cfg["nb"]
    d = {"workload": name, "m": cfg["m"], "n": cfg["n"], "nb": nb, "ib": 32, "tree": cfg["algo"],
         "family": cfg["family"], "seed": cfg["seed"], "dist": cfg["dist"],
         "tiles": f"{cfg['m'] // nb}x{cfg['n'] // nb}"}
    if name == "c5":
        d["tree"] = f"{cfg['algo']} local trees + TT merges of the R factors"
        d["parallelism"] = f"block rows over {world} GPU(s), NCCL p2p R blocks to rank 0, one TT merge"
    else:
        d["parallelism"] = "1 GPU, persistent dataflow executor"
    bytes_in = 8 * cfg["m"] * cfg["n"]
    d["l2"] = (f"inputs {bytes_in / 2**30:.2f} GiB > 126 MB L2 (no flush needed)" if bytes_in > 126e6
               else "inputs < L2; not flushed (sub-ms step)")
    return d


def flops_of(cfg):
    m, n = cfg["m"], cfg["n"]
    return 2.0 * n * n * (m - n / 3.0)


class Clocks:
    """nvidia-smi sampler for the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU side (the oracle / reference path; never the thing measured on the GPU)


def replay_sample(name, cfg, A=None):
    """(p, q, nb, A, description) of the trace the CPU replays for a
    workload: the workload itself, except C5, whose sample is one G=8 shard
    (1024 x 8 tiles, its local Greedy tree) — the per-rank work at 8 GPUs."""
    nb = cfg["nb"]
    if name == "c5":
        rows = 1024 * nb
        A = A[:rows] if A is not None else make_matrix(cfg, rows=rows)
        return 1024, cfg["n"] // nb, nb, A, "C5 shard: rows 0..262143 (1024x8 tiles, local Greedy/TT tree)"
    A = A if A is not None else make_matrix(cfg)
    return cfg["m"] // nb, cfg["n"] // nb, nb, A, f"{name} ({cfg['m']}x{cfg['n']})"


def cpu_replay(T, name, cfg, warmup, steps, step_s, A=None):
    """Time the reference path on the host: tiledag.build_tree (the
    reference's own CPU path), then the LAPACK tile kernels of its trace over
    its hazard DAG on every core, in `step_s`-second windows that continue
    one factorization (restarted on a fresh copy of A when it completes).
    Returns a dict of measurements."""
    from oracle.cpu_baseline import DagReplay, edges_of, trace_arrays_of
    p, q, nb, A_s, what = replay_sample(name, cfg, A)
    t0 = time.perf_counter()
    b = T.build_tree(p, q, cfg["algo"], family=cfg["family"])
    t_build = time.perf_counter() - t0
    kinds, idx = trace_arrays_of(b)
    edges = edges_of(b, T)
    dr = DagReplay(A_s, p, q, nb, kinds, idx, edges)
    fl = dt = 0.0
    done = 0
    rates = []
    try:
        for s in range(warmup + steps):
            if dr.finished():
                dr.reload(A_s)
            f, d, c = dr.run_for(step_s)
            if s >= warmup:
                fl, dt, done = fl + f, dt + d, done + c
                rates.append(f / d / 1e9)
    finally:
        dr.close()
    return {"gflops": fl / dt / 1e9, "tasks": done, "trace_tasks": len(kinds), "seconds": dt,
            "step_gflops": [round(r, 2) for r in rates], "cores": dr.workers, "build_tree_s": t_build,
            "sample": (f"LAPACK tile kernels (scipy dgeqrt/dgemqrt/dtpqrt/dtpmqrt, 1 thread each) of the "
                       f"reference trace tiledag.build_tree({p}, {q}, {cfg['algo']!r}, {cfg['family']!r}) "
                       f"over its hazard DAG (tiledag.build_from_trace) on {dr.workers} worker processes; "
                       f"{what}; {steps} windows of {step_s:g} s continuing one factorization: "
                       f"{done} of {len(kinds)} tasks, {fl / 1e9:.0f} GFLOP in {dt:.1f} s")}


def run_reference(args, name, cfg):
    """The reference arm (rank 0 only; other ranks exit without work)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    from oracle.cpu_baseline import load_reference
    T = load_reference()
    if T is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference package tiledag not installed"}))
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    r = cpu_replay(T, name, cfg, args.warmup, args.steps, args.ref_step_s)
    v = round(r["gflops"], 3)
    loaded = [ln.split()[-1] for ln in open("/proc/self/maps") if "libtqr" in ln]
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * r["seconds"] / max(args.steps, 1), 3),
        "higher_is_better": True, "scaling": "strong" if name == "c5" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_dict(name, cfg, world),
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": r["cores"], "kind": "port", "sample": r["sample"]},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_build_tree_s": round(r["build_tree_s"], 3), "step_gflops": r["step_gflops"],
        "native_so_loaded": sorted(set(loaded)),
    }))


def cpu_baseline_block(name, cfg, A_host, step_s, dgeqrf=True):
    """The repo arm's cpu_baseline: the reference path on the host (as in
    run_reference, 3 windows) + dgeqrf on the full workload matrix."""
    from oracle.cpu_baseline import load_reference, time_dgeqrf
    T = load_reference()
    if T is None:
        return None
    r = cpu_replay(T, name, cfg, 1, 3, step_s, A=A_host)
    out = {"value": round(r["gflops"], 3), "unit": "GFLOP/s", "cores": r["cores"], "kind": "port",
           "sample": r["sample"], "reference_build_tree_s": round(r["build_tree_s"], 3)}
    if dgeqrf and name != "c5":
        s, g, th = time_dgeqrf(A_host)
        out["dgeqrf"] = {"value": round(g, 3), "unit": "GFLOP/s", "seconds": round(s, 2), "threads": th,
                         "sample": f"numpy.linalg.qr(A, mode='r') (LAPACK dgeqrf, OpenBLAS) on the full "
                                   f"{cfg['m']}x{cfg['n']} matrix"}
    return out


# ---------------------------------------------------------------------------
# GPU arm


def run_single(args, name, cfg):
    import ctypes as C

    import torch

    import paper_1303_3182_b200 as P
    from paper_1303_3182_b200 import _lib
    from paper_1303_3182_b200.engine import Plan, tiled_qr_host

    torch.cuda.set_device(0)
    nb = cfg["nb"]
    p, q = cfg["m"] // nb, cfg["n"] // nb
    t0 = time.perf_counter()
    build = P.build_tree(p, q, cfg["algo"], family=cfg["family"])
    t_build = time.perf_counter() - t0
    plan = Plan(build, nb)
    t_plan = time.perf_counter() - t0
    A_host = make_matrix(cfg)
    A = torch.from_numpy(A_host).cuda()
    tiles, tg, te = plan.alloc()
    stream = torch.cuda.current_stream()

    # live FP64 peak (DMMA loop on every SM), the roofline denominator
    pk = C.c_double()
    _lib.check(_lib.lib().tqr_fp64_peak(C.byref(pk), C.c_void_p(stream.cuda_stream)))
    peak_tf = pk.value

    def step(ev=None):
        plan.pack(A, tiles)
        if ev:
            ev[0].record()
        plan.factor(tiles, tg, te)
        if ev:
            ev[1].record()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clk = Clocks(0).start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record()
    for s in range(args.steps):
        step(evs[s])
    end.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = start.elapsed_time(end) / args.steps
    k_ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
    flops = plan.flops
    value = flops / (ms * 1e-3) / 1e9

    # correctness spot check of the last factorization (cheap, outside timing)
    R = plan.extract_r(tiles)
    d = torch.diagonal(R)
    ok = bool(torch.isfinite(R).all().item()) and bool((d.abs() > 0).all().item())

    e2e = None
    if not args.no_e2e:
        # public API, host in / host out: tiled_qr_host (tqr_qr_host) overlaps
        # the pinned H2D copy of A (arrival units + flags on one copy stream)
        # and the D2H copy of each finished tile row of R with the executor
        plan_io = Plan(build, nb, io=Plan.IO_IN | Plan.IO_OUT)
        A_pin = torch.from_numpy(A_host).pin_memory()
        R_pin = torch.zeros((cfg["n"], cfg["n"]), dtype=torch.float64).pin_memory()
        # one cold call through the public API: schedule compile (build_tree +
        # plan), scratch allocation, transfers and factorization
        from paper_1303_3182_b200 import engine as E
        E._PLAN_CACHE.clear()
        torch.cuda.synchronize()
        t_c = time.perf_counter()
        tiled_qr_host(A_pin, R_pin, nb=nb, algo=cfg["algo"], family=cfg["family"])
        torch.cuda.synchronize()
        cold_ms = (time.perf_counter() - t_c) * 1e3
        bufs = plan_io.stream_buffers()
        tiled_qr_host(A_pin, R_pin, plan=plan_io, buffers=bufs)  # warm-up
        torch.cuda.synchronize()
        ne = max(3, min(args.steps, 5))
        eev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(ne)]
        for a, b in eev:
            a.record()
            tiled_qr_host(A_pin, R_pin, plan=plan_io, buffers=bufs)
            b.record()
        torch.cuda.synchronize()
        each = [a.elapsed_time(b) for a, b in eev]
        e_ms = statistics.mean(each)
        ok = ok and bool(torch.equal(R_pin, R.cpu()))  # same R as the device-resident path
        e2e = {"value": round(flops / (e_ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
               "ms_per_step": round(e_ms, 3), "ms_each": [round(x, 2) for x in each],
               "api": "tiled_qr_host (pinned host A in, pinned host R out)",
               "cold_call_ms": round(cold_ms, 1),
               "cold_call": "first tiled_qr_host call on the shape: + schedule compile, scratch allocation (wall)",
               "h2d_bytes_per_step": int(A_host.nbytes),
               "d2h_bytes_per_step": int(8 * nb * nb * q * (q + 1) // 2)}  # R's upper tile rows
        del bufs

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_block(name, cfg, A_host, args.ref_step_s)
        if cpu is not None:
            cpu["repo_build_tree_s"] = round(t_build, 3)
            cpu["repo_plan_s"] = round(t_plan, 3)

    achieved = flops / (k_ms * 1e-3) / 1e12
    print(json.dumps({
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_dict(name, cfg),
        "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak_tf, 3),
                     "unit": "TFLOP/s", "frac": round(achieved / peak_tf, 4),
                     "traffic": profile_traffic(name),
                     "kernel": "exec_kernel (persistent executor: all tile kernels)",
                     "peak_source": "live DMMA.8x8x4 probe (tqr_fp64_peak); MEASURED_PEAKS.json has no FP64 entry"},
        "kernel_ms": round(k_ms, 3), "kernel_ms_each": [round(a.elapsed_time(b), 3) for a, b in evs],
        "plan_s": round(t_plan, 3), "gpu_launches": 2 * args.steps, "clocks": clocks, "e2e": e2e,
        "cpu_baseline": cpu,
        "check": {"r_finite_nonsingular": ok, "items": plan.info.n_items, "tasks": plan.info.n_tasks},
    }))


def profile_traffic(workload):
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload)
    except (OSError, ValueError):
        return None


def run_c5(args, name, cfg):
    """C5 on N ranks (N=1: the whole matrix on one GPU): local Greedy trees +
    a TT merge of the R factors (one gather merge on rank 0, or binary
    rounds; paper_1303_3182_b200.dist); device time, max over ranks."""
    import ctypes as C

    import torch
    import torch.distributed as td

    from paper_1303_3182_b200 import _lib, dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nb, m, n = cfg["nb"], cfg["m"], cfg["n"]
    p, q = m // nb, n // nb
    flops = flops_of(cfg)

    def measure(G, rank_, A_host, comm):
        """(ms per step, R block on rank 0, backend) for G shards."""
        P = p // G
        A = torch.from_numpy(A_host).to(dev)
        t_p = time.perf_counter()
        be = dist.GpuBackend(P, q, nb, dev, algo=cfg["algo"], family=cfg["family"])
        plan_times[G] = round(time.perf_counter() - t_p, 3)

        def step():
            return dist.tall_skinny_qr(A, be, rank_, G, comm, merge=args.merge)

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if comm:
            comm.barrier()
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        for _ in range(args.steps):
            out = step()
        end.record()
        torch.cuda.synchronize()
        if comm:
            comm.barrier()
        ms = start.elapsed_time(end) / args.steps
        del A
        return ms, out, be

    plan_times = {}
    single = None
    if world > 1 and rank == 0 and not args.no_single:
        # rank 0's same-run one-GPU C5 (the N=1 point of this scaling line);
        # the other ranks wait in the process-group rendezvous meanwhile
        ms1, _, be1 = measure(1, 0, make_matrix(cfg), None)
        single = {"ms_per_step": round(ms1, 3), "value": round(flops / (ms1 * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
                  "what": "the whole C5 matrix on rank 0's GPU alone, same steps/warmup, measured before the "
                          "distributed run"}
        del be1
        torch.cuda.empty_cache()
    nccl = None
    if world > 1:
        td.init_process_group("nccl", device_id=dev)
        nccl = {"backend": td.get_backend(), "world_size": td.get_world_size(),
                "version": ".".join(str(v) for v in torch.cuda.nccl.version())}
    if p % world:
        raise SystemExit(f"p={p} not divisible by world={world}")
    rows = (p // world) * nb
    A_host = make_matrix(cfg, rows=rows, row0=rank * rows)
    clk = Clocks(local).start() if rank == 0 else None
    ms, out, be = measure(world, rank, A_host, td if world > 1 else None)
    clocks = clk.stop() if clk else None
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        td.all_reduce(t, op=td.ReduceOp.MAX)
    ms = float(t.item())
    # e2e through the public API: each rank's shard streams in from
    # (registered, page-locked) host memory during the factorization, R back
    # to the host on rank 0
    e2e = None
    if not args.no_e2e:
        cudart = torch.cuda.cudart()
        host = torch.from_numpy(A_host)
        reg = int(cudart.cudaHostRegister(host.data_ptr(), host.numel() * 8, 0)) == 0
        R_host = torch.empty((n, n), dtype=torch.float64).pin_memory()
        ne = max(1, min(args.steps, 2))

        def e2e_step():
            o = dist.tall_skinny_qr(host if reg else host.to(dev), be, rank, world, td if world > 1 else None,
                                    merge=args.merge)
            if rank == 0:
                R_host.copy_(be.r_matrix(o), non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            td.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(ne):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / ne], dtype=torch.float64, device=dev)
        if world > 1:
            td.all_reduce(te, op=td.ReduceOp.MAX)
        if reg:
            cudart.cudaHostUnregister(host.data_ptr())
        e_ms = float(te.item())
        e2e = {"value": round(flops / (e_ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s", "ms_per_step": round(e_ms, 3),
               "api": "dist.tall_skinny_qr (page-locked host shard streamed in, R to host on rank 0)",
               "h2d_bytes_per_step": int(m) * int(n) * 8, "d2h_bytes_per_step": int(n) * int(n) * 8,
               "host_registered": reg}
    if rank == 0:
        pk = C.c_double()
        _lib.check(_lib.lib().tqr_fp64_peak(C.byref(pk), C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        peak = pk.value * world
        R = be.r_matrix(out)
        ok = bool(torch.isfinite(R).all().item())
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_baseline_block(name, cfg, None, args.ref_step_s, dgeqrf=False)
        achieved = flops / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": round(flops / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(name, cfg, world),
            # per step on rank 0: pack + executor, then the merge executor(s)
            "gpu_launches": (2 + (min(1, world - 1) if args.merge == "gather" else len(dist.merge_rounds(world))))
            * args.steps,
            "merge": args.merge,
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3),
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "exec_kernel (local factorization + merges)",
                         "peak_source": "live DMMA.8x8x4 probe x n_gpus"},
            "clocks": clocks, "cpu_baseline": cpu, "e2e": e2e, "nccl": nccl,
            "plan_s": plan_times.get(world),
            "check": {"r_finite": ok},
        }
        if single is not None:
            line["c5_single_gpu"] = single
        print(json.dumps(line))
    if world > 1:
        td.destroy_process_group()


def run_dry(args, name, cfg):
    """--dry (CPU, no GPU needed): the multi-rank launcher path end to end —
    torchrun ranks, a gloo process group, each rank compiles its local
    Greedy schedule and the merge schedule, and the R blocks travel in the
    merge pattern of dist.tall_skinny_qr — no kernels.  Rank 0 prints a line
    with n_gpus and no value."""
    import torch
    import torch.distributed as td

    import paper_1303_3182_b200 as P
    from paper_1303_3182_b200 import dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    nb, p, q = cfg["nb"], cfg["m"] // cfg["nb"], cfg["n"] // cfg["nb"]
    if world > 1:
        td.init_process_group("gloo")

    class DryBackend:
        def __init__(self):
            self.q = q
            self.build = P.build_tree(p // world, q, "greedy")
            self.merge_kinds, _ = dist.merge_trace(q, world if args.merge == "gather" else 2)

        def factor_local(self, A_local):
            return torch.full((q * q * 4,), float(rank))

        def merge(self, r_a, r_b, key=None):
            return r_a + r_b

        def merge_many(self, rs, key=None):
            return sum(rs[1:], rs[0])

    be = DryBackend()
    t0 = time.perf_counter()
    out = dist.tall_skinny_qr(None, be, rank, world, td if world > 1 else None, merge=args.merge)
    dt = time.perf_counter() - t0
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GFLOP/s", "n_gpus": world, "dry": True,
                          "steps": 0, "warmup": 0, "config": config_dict(name, cfg, world),
                          "check": {"local_tasks": len(be.build.trace_arrays()[0]),
                                    "merge_tasks": int(len(be.merge_kinds)),
                                    "ranks_summed": float(out[0].item()), "exchange_s": round(dt, 4),
                                    "backend": td.get_backend() if world > 1 else None}}))
    if world > 1:
        td.destroy_process_group()


def spawn(args):
    """Relaunch this script under torch.distributed.run with one rank per
    GPU (127.0.0.1 rendezvous); rank 0 prints the line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-single", action="store_true", help="N>1: skip rank 0's one-GPU C5 point")
    ap.add_argument("--ref-step-s", type=float, default=3.0, help="CPU replay window per step (s)")
    ap.add_argument("--dry", action="store_true", help="CPU launcher check: ranks, gloo exchange, no kernels")
    ap.add_argument("--tree", default=None, help="override the workload's elimination tree (e.g. asap, grasap)")
    ap.add_argument("--family", default=None, choices=["TT", "TS"],
                    help="override the workload's kernel family (tiledag family= of tiled_build/build_tree)")
    ap.add_argument("--merge", default="gather", choices=["gather", "binary"],
                    help="C5 R merges: one gather merge on rank 0, or log2 N binary rounds")
    args = ap.parse_args(argv)
    if args.config is None:
        args.config = "c3" if args.gpus == 1 else "c5"
    return args


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    name, cfg = args.config, CONFIGS[args.config]
    if args.tree:
        cfg = dict(cfg, algo=args.tree)
    if args.family:
        cfg = dict(cfg, family=args.family)
    if args.impl == "reference":
        return run_reference(args, name, cfg)
    if args.dry:
        return run_dry(args, name, cfg)
    if name == "c5" or args.gpus > 1:
        if name != "c5":
            raise SystemExit("multi-GPU runs shard the tall-skinny workload: use --config c5")
        return run_c5(args, name, cfg)
    return run_single(args, name, cfg)


if __name__ == "__main__":
    main()
