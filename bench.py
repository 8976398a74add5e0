#!/usr/bin/env python
"""Benchmark of the STMG solve path (BASELINE.json metric: space-time DoF/s of
the operator vmult and the STMG V-cycle, fp64, with the HBM roofline
fraction).

One step = one preconditioned GMRES iteration's operator work on the slab
system: one V-cycle (SpaceTimeMultigrid::apply) followed by one vmult
(SpaceTimeOperator::apply) -- exactly the precond(v) / op(z) pair of
gmres.cpp:45-47. value = N_fine / t_step over K timed steps (inputs resident
in HBM, vectors larger than L2). The e2e figure runs the same step through the
public API with the step's input copied from pinned host memory and its
result read back inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C2]
  python bench.py --impl reference ...   (the reference's CPU implementation)

Multi-GPU (torchrun, N>1): the workload's finest mesh is partitioned into N
z-slabs, one per rank, with NCCL interface exchanges and
allreduces; value = the workload's DoFs over the max-over-ranks step time
("scaling": "strong"). --replicas runs independent copies instead (weak).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "space-time DoF/s: operator vmult & STMG V-cycle, fp64, % of HBM roofline"


def ncu_traffic(kernel_key: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(kernel_key)
    return e["dram_bytes_per_launch"] if e else None


def ncu_flops(kernel_key: str):
    """Executed fp64 flops per launch from the committed SASS instruction
    counts (profiles/ncu_flops.json) and the measured DFMA peak, or None."""
    p = os.path.join(ROOT, "profiles", "ncu_flops.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f)
    e = d.get(kernel_key)
    return (e["flops_per_launch"] if e else None), d.get("fp64_peak_tflops")


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def e2e_pipelined(step, r_dev, y_dev, rh, yh, n_steps):
    """End-to-end time per step (s): every step copies its input from pinned
    host memory (rh) to the device and its result back (yh). The H2D of step
    i+1 and the D2H of step i-1 run on two copy streams while step i
    computes; r_dev / y_dev are two device buffers each (ping-pong)."""
    import torch
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    read = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(h2d):
        r_dev[0].copy_(rh, non_blocking=True)
        ready[0].record(h2d)
    for i in range(n_steps):
        b = i % 2
        if i + 1 < n_steps:
            with torch.cuda.stream(h2d):
                if i >= 1:
                    h2d.wait_event(done[1 - b])  # step i-1 has read r_dev[1-b]
                r_dev[1 - b].copy_(rh, non_blocking=True)
                ready[1 - b].record(h2d)
        comp.wait_event(ready[b])
        if i >= 2:
            comp.wait_event(read[b])  # step i-2's result is on the host
        step(r_dev[b], y_dev[b])
        done[b].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[b])
            yh.copy_(y_dev[b], non_blocking=True)
            read[b].record(d2h)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n_steps


def cpu_baseline(workload: str, budget_s: float = 15.0, refinements: int = 3):
    """The reference's own C++ (oracle/_ref, single-threaded by construction)
    on a bounded, oracle-reachable sample of the workload: the same step
    (V-cycle + vmult) on the same configuration at `refinements`."""
    import numpy as np
    from oracle import refbind
    from paper_2408_04372_b200 import problems
    cfg = problems.config(workload, refinements)
    t0 = time.perf_counter()
    R = refbind.Reference(cfg, with_mg=True)
    setup = time.perf_counter() - t0
    r = problems.uniform_vector(R.n_dofs, seed=1)
    R.apply(R.vcycle(r))  # warm-up
    steps, t0 = 0, time.perf_counter()
    while True:
        R.apply(R.vcycle(r))
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s:
            break
    val = steps * R.n_dofs / el
    return {"value": val, "unit": "DoF/s", "cores": 1, "kind": "reference",
            "sample": f"{workload} at {cfg.cells}^{cfg.dim} cells (N={R.n_dofs}), {steps} steps of V-cycle+vmult "
                      f"in {el:.1f}s, setup {setup:.1f}s excluded; reference proj/src via oracle/_ref, 1 thread"}, cfg


def _ref_replica(workload, refinements, warmup, steps, barrier, out):
    """One single-threaded reference replica (forked worker of run_reference)."""
    try:
        from oracle import refbind
        from paper_2408_04372_b200 import problems
        cfg = problems.config(workload, refinements)
        R = refbind.Reference(cfg, with_mg=True)
        r = problems.uniform_vector(R.n_dofs, seed=1)
        for _ in range(warmup):
            R.apply(R.vcycle(r))
        barrier.wait()
        t0 = time.perf_counter()
        for _ in range(steps):
            R.apply(R.vcycle(r))
        out.put((time.perf_counter() - t0, R.n_dofs, cfg.cells))
    except Exception as e:  # noqa: BLE001
        barrier.abort()
        out.put(("error", str(e)[:200], 0))


def run_reference(args):
    """The reference's own CPU implementation (oracle/_ref: proj/src compiled
    unmodified) on this host. It is single-threaded by construction, so all
    host threads are used as P concurrent replicas of the same bounded sample
    (one process per core, started together, timed to the slowest);
    value = P * steps * N / t. Under torchrun only rank 0 runs."""
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    ncpu = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    # about 0.5 GB per replica at the default sample (ASM block LU factors)
    try:
        import psutil
        mem_cap = max(1, int(psutil.virtual_memory().available / 0.75e9))
    except Exception:  # noqa: BLE001
        mem_cap = 8
    P = max(1, min(ncpu, mem_cap, args.ref_replicas or ncpu))
    ctx = mp.get_context("fork")
    barrier, out = ctx.Barrier(P), ctx.Queue()
    procs = [ctx.Process(target=_ref_replica, args=(args.workload, args.ref_refinements, args.warmup, args.steps,
                                                     barrier, out)) for _ in range(P)]
    for p in procs:
        p.start()
    res = [out.get() for _ in range(P)]
    for p in procs:
        p.join()
    errs = [r for r in res if r[0] == "error"]
    if errs:
        print(json.dumps({"impl": "reference", "unavailable": f"reference replica failed: {errs[0][1]}"}), flush=True)
        return
    el = max(r[0] for r in res)
    n, cells = res[0][1], res[0][2]
    val = P * args.steps * n / el
    sample = (f"{args.workload} at {cells}^3 cells (N={n}), {args.steps} steps of V-cycle+vmult per replica, "
              f"{P} concurrent single-threaded replicas on {ncpu} host threads, timed to the slowest")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "DoF/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "sample_cells": cells, "n_dofs": n, "replicas": P,
                       "note": "reference CPU implementation (single-threaded per solve) on an oracle-reachable size"},
            "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": P, "kind": "reference", "sample": sample},
            "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_partitioned(args, world, rank, local):
    """N > 1: the z-slab partitioned solve of ONE workload over all ranks
    (strong scaling): rank r holds slab r of the finest mesh,
    NCCL carries the interface-plane exchanges and the allreduces."""
    import torch
    import torch.distributed as dist

    from paper_2408_04372_b200 import api, native, problems

    lib = native.load()
    uid = [api.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = api.Comm(world, rank, uid[0])
    cfg = problems.config(args.workload)
    t0 = time.perf_counter()
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    S = api.SlabMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                          cfg.tau, world, first_part=rank, local_parts=1, comm=comm)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    n_local = S.n_local
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    r = torch.rand(n_local, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z, y = torch.empty_like(r), torch.empty_like(r)

    def step(rr=r, yy=y):
        S.vcycle(rr, z)
        S.apply(z, yy)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    zz = torch.zeros_like(r)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        S.asm_add_correction(r, zz)
    e1.record()
    e1.synchronize()
    t_asm = e0.elapsed_time(e1) / 5
    dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.stmg_kernel_launches()
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    launches = lib.stmg_kernel_launches() - launches0
    t = torch.tensor([e0.elapsed_time(e1) / args.steps], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = cfg.n_dofs / (ms * 1e-3)
    # end to end: local slab from pinned host memory, result back, per step
    rh = torch.empty(n_local, dtype=torch.float64).pin_memory()
    rh.copy_(r.cpu())
    yh = torch.empty(n_local, dtype=torch.float64).pin_memory()
    e2e_steps = max(4, min(args.steps, 10))
    dist.barrier()
    e2e_s = e2e_pipelined(step, [r, torch.empty_like(r)], [y, torch.empty_like(y)], rh, yh, e2e_steps)
    tl = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(tl, op=dist.ReduceOp.MAX)
    e2e = {"value": cfg.n_dofs / float(tl.item()), "unit": "DoF/s", "h2d_bytes_per_step": 8 * n_local,
           "d2h_bytes_per_step": 8 * n_local, "note": "per rank: its slab of the step's input and result"}
    peak, peak_kind = measured_peaks()
    n_cells_local = cfg.cells ** cfg.dim // world
    m = (cfg.p + 1) ** cfg.dim
    asm_bytes = n_cells_local * (m * m + m) * 8 + 24 * n_local
    achieved = asm_bytes / (t_asm * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **cfg.describe(), "parallelism": f"z-slab x{world}",
                       "partitioned_levels": S.dist_levels,
                       "step": "1 V-cycle + 1 vmult (one preconditioned GMRES iteration's operator work)",
                       "l2": "vectors larger than L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": (lambda tr: tr / world if tr else None)(ncu_traffic(f"{args.workload}:asm")),
                         "peak_source": peak_kind,
                         "kernel": "asm_apply_fd64_kernel (rank-local fine-level smoother sweep)",
                         "algorithmic_bytes_per_launch": asm_bytes, "launch_ms": t_asm},
            "e2e": e2e, "gpu_launches": int(launches), "setup_s": setup_s, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    del S, comm
    dist.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch

    from paper_2408_04372_b200 import api, native, problems
    from paper_2408_04372_b200 import dist as sdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        if not args.replicas:
            return run_partitioned(args, world, rank, local)
    lib = native.load()

    cfg = problems.config(args.workload)
    t0 = time.perf_counter()
    mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    print(f"[bench] setup {setup_s:.1f}s, levels {M.level_info()}", file=sys.stderr, flush=True)
    op = M.operator_at(0)
    N = op.n_dofs
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    r = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z = torch.empty_like(r)
    y = torch.empty_like(r)

    def step(rr=r, yy=y):
        M.apply(rr, z)
        op.apply(z, yy)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    def timed(fn, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps  # ms

    # per-kernel times (same stream as the launches), for the roofline
    t_vmult = timed(lambda: op.apply(r, y), 10)
    zz = torch.zeros_like(r)
    t_asm = timed(lambda: M.asm_add_correction(0, r, zz), 5)
    t_vcycle = timed(lambda: M.apply(r, z), 5)

    # timed region
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.stmg_kernel_launches()
    with ClockSampler(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    launches = lib.stmg_kernel_launches() - launches0
    # whole-job throughput: units of all ranks over the max-over-ranks time
    value, ms = sdist.aggregate_throughput(N, e0.elapsed_time(e1) / args.steps, device="cuda")
    if dist:
        dist.barrier()

    # one full STMG-preconditioned GMRES solve of the slab system (the
    # paper's "dofs/s" = N / solve time; manufactured RHS assembled on the
    # device, rel. tol 1e-10), reported beside the per-step metric
    solve = None
    try:
        u0 = torch.zeros(op.n_space, dtype=torch.float64, device="cuda")
        v0 = torch.zeros_like(u0) if cfg.equation == problems.WAVE else None
        b = op.assemble_rhs(1, 0.5, 0.0, u0, v0)
        xs = torch.zeros_like(b)
        M.solve(b, xs, rel_tol=1e-10, abs_tol=0.0)  # warm-up: Krylov basis allocated once
        xs.zero_()
        torch.cuda.synchronize()
        ts = time.perf_counter()
        info = M.solve(b, xs, rel_tol=1e-10, abs_tol=0.0)
        torch.cuda.synchronize()
        t_solve = time.perf_counter() - ts
        solve = {"iterations": info["iterations"], "converged": info["converged"], "ms": 1e3 * t_solve,
                 "dofs_per_s": N / t_solve, "rhs": "manufactured source (frequency 0.5), zero entering state",
                 "rel_tol": 1e-10}
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        solve = {"error": str(e)[:200]}

    # end to end through the public API: every step copies its input from
    # pinned host memory to the device and reads its result back
    rh = torch.empty(N, dtype=torch.float64).pin_memory()
    rh.copy_(r.cpu())
    yh = torch.empty(N, dtype=torch.float64).pin_memory()
    e2e_steps = max(4, min(args.steps, 10))
    if dist:
        dist.barrier()
    e2e_s = e2e_pipelined(step, [r, torch.empty_like(r)], [y, torch.empty_like(y)], rh, yh, e2e_steps)
    if dist:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": world * N / e2e_s, "unit": "DoF/s", "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
           "note": "pinned H2D of each step's input and D2H of its result, overlapped with the neighbouring steps"}

    # roofline of the dominant kernel
    peak, peak_kind = measured_peaks()
    cells = cfg.cells ** cfg.dim
    m = (cfg.p + 1) ** cfg.dim
    n_verts = (cfg.cells + 1) ** cfg.dim
    vmult_bytes = 16 * N + (24 * n_verts if cfg.perturb > 0 else 0)
    # records (X + eigenvalues) + 16-byte meta per cell, r read, z read+write
    asm_bytes = cells * (m * m + m) * 8 + 16 * cells + 8 * N + 16 * N
    # fine-level launches per step: vmult 3 (2 residuals in the V-cycle + the
    # outer op), ASM 2 (pre- and post-smoothing)
    share_vmult = 3 * t_vmult / ms
    share_asm = 2 * t_asm / ms
    if share_asm >= share_vmult:
        dom = {"kernel": "asm_apply_fd64_kernel (fine-level exact cell-block smoother)", "key": "asm", "ms": t_asm,
               "bytes": asm_bytes, "share_of_step": share_asm}
    else:
        dom = {"kernel": "st_lines_kernel (fused space-time vmult)", "key": "vmult", "ms": t_vmult,
               "bytes": vmult_bytes, "share_of_step": share_vmult}
    achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic(f"{args.workload}:{dom['key']}"), "peak_source": peak_kind,
                "kernel": dom["kernel"],
                "algorithmic_bytes_per_launch": dom["bytes"], "launch_ms": dom["ms"],
                "share_of_step": dom["share_of_step"]}
    vm_ach = vmult_bytes / (t_vmult * 1e-3) / 1e9
    vc_bytes = M.vcycle_bytes()
    # the vmult is fp64-issue bound, not HBM bound: its fp64 roofline
    vm_flops, fp64_peak = ncu_flops(f"{args.workload}:vmult")
    vmult_fp64 = None
    if vm_flops and fp64_peak:
        tf = vm_flops / (t_vmult * 1e-3) / 1e12
        vmult_fp64 = {"bound": "fp64", "flops_per_launch": vm_flops, "achieved": tf, "peak": fp64_peak,
                      "unit": "TFLOP/s", "frac": tf / fp64_peak,
                      "source": "executed DFMA/DADD/DMUL of one ncu capture (profiles/ncu_flops.json)"}

    line = {"metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **cfg.describe(), "parallelism": f"replicas x{world}",
                       "step": "1 V-cycle + 1 vmult (one preconditioned GMRES iteration's operator work)",
                       "l2": "vectors (8N = %.0f MB) larger than L2; no flush" % (8 * N / 1e6)},
            "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches),
            "kernels": {"vmult_ms": t_vmult, "vmult_dofs_per_s": N / (t_vmult * 1e-3),
                        "vmult_hbm_frac": vm_ach / peak, "vmult_fp64": vmult_fp64, "vcycle_ms": t_vcycle,
                        "vcycle_dofs_per_s": N / (t_vcycle * 1e-3),
                        "vcycle_algorithmic_bytes": vc_bytes,
                        "vcycle_hbm_frac": vc_bytes / (t_vcycle * 1e-3) / 1e9 / peak, "asm_fine_ms": t_asm},
            "solve": solve, "setup_s": setup_s, "mg_levels": M.n_levels, "device_bytes": M.device_bytes()}
    line["clocks"] = clk.summary()

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cb, _ = cpu_baseline(args.workload, budget_s=args.cpu_budget)
            line["cpu_baseline"] = cb
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C2")
    ap.add_argument("--ref-refinements", type=int, default=3)
    ap.add_argument("--ref-replicas", type=int, default=0,
                    help="reference arm: concurrent single-threaded replicas (0: one per host thread)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the z-slab partitioned path even at N = 1 (one slab; exercises the NCCL plumbing)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas per rank instead of the z-slab partitioned solve")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
