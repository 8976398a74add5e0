#!/usr/bin/env python
"""Benchmark of the STMG solve path (BASELINE.json metric: space-time DoF/s of
the operator vmult and the STMG V-cycle, fp64, with the HBM roofline
fraction).

One step = one preconditioned GMRES iteration's operator work on the slab
system: one V-cycle (SpaceTimeMultigrid::apply) followed by one vmult
(SpaceTimeOperator::apply) -- the precond(v) / op(z) pair of gmres.cpp:45-47.
value = N / t_step over K timed steps (inputs resident in HBM, vectors larger
than L2).

Workload (N = 1): C5-128 -- heat 3D, Q4 space, dG(3) time, 128^3 Cartesian
cells, 5.40e8 space-time DoFs: the largest BASELINE configuration whose full
V-cycle (with the reference's Arnoldi relaxation factors) fits one GPU. C2, C3
and C4 are measured in the same run under "per_config".

e2e: the same step through the reference-facing host-buffer C ABI
(stmg_multigrid_apply_host + stmg_st_operator_apply_host, the LinearMap
plug-in of INTEGRATION.md), pageable numpy buffers, H2D + D2H inside every
step.

Multi-GPU (N > 1; launched through torch.distributed.run, or spawned here
when WORLD_SIZE is unset): the C5 weak-scaling study of SURVEY.md 8e -- one
128^3-cell block per GPU (128^3 @ 1 -> 256^3 @ 8, box meshes in between), the
mesh cut into N z-slabs, NCCL interface exchanges and allreduces; value =
total DoFs / max-over-ranks step time ("scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5-128]
  python bench.py --impl reference ...   (the reference's CPU implementation)
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


def profile_entry(key: str, field: str):
    """A per-launch figure of the committed ncu captures (profiles/ncu_*.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_kernels.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    e = d.get(key)
    return e.get(field) if e else None


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs (burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


FP64_PEAK_TFLOPS = 33.2  # measured DFMA peak, scripts/fp64_peak.cu (profiles/round1_fp64_peaks.txt)


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # the timed region starts once the sampler reports
            t0 = time.perf_counter()
            while not self.lines and time.perf_counter() - t0 < 5.0:
                time.sleep(0.01)
            self.skip = len(self.lines)
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
        for ln in self.lines[max(0, getattr(self, "skip", 1) - 1):]:
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


def timed(fn, reps):
    """Device time per call (ms), CUDA events on the launching stream."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):  # untimed: first-launch work (function attributes, the coarse-cycle graph capture)
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def flush_l2():
    """Overwrite a buffer larger than the 126 MB L2."""
    import torch
    global _FLUSH
    try:
        _FLUSH
    except NameError:
        _FLUSH = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    _FLUSH.fill_(1.0)


def algorithmic_bytes(cfg, N):
    """SURVEY.md 8(d) bytes per launch: vmult 16 N (+ 24 n_verts on perturbed
    meshes), residual 24 N, one smoother sweep 24 N (r read, z read + write),
    same geometry term."""
    geo = 24 * (cfg.cells + 1) ** cfg.dim if cfg.perturb > 0 else 0
    return {"vmult": 16 * N + geo, "residual": 24 * N + geo, "asm": 24 * N + geo}


def vcycle_algorithmic_bytes(M, geo_per_pass=0):
    """112 N_l bytes per level above the coarsest (smoothing,
    residuals, transfers), 8 n_c^2 for the coarse dense solve, plus geometry per
    vmult / smoother pass (5 per level: 2 sweeps, 2 residuals, ... counted on
    the finest level only)."""
    info = M.level_info()
    total = 0
    for l, li in enumerate(info):
        n = li["n_dofs"]
        total += 112 * n if l + 1 < len(info) else 8 * n * n
    return total + 4 * geo_per_pass


def kernel_figures(cfg, M, op, r, z, y, peak):
    """Per-kernel device times of the finest level and their roofline
    fractions against SURVEY.md 8(d) bytes (and the smoother's streamed
    bytes, which include any per-cell records)."""
    import torch
    N = op.n_dofs
    ab = algorithmic_bytes(cfg, N)
    f = torch.empty_like(r).uniform_(-1, 1)
    zz = torch.zeros_like(r)
    t_vmult = timed(lambda: op.apply(r, y), 10)
    t_res = timed(lambda: op.residual(f, r, y), 10)
    t_asm = timed(lambda: M.asm_add_correction(0, r, zz), 5)
    t_vc = timed(lambda: M.apply(r, z), 5)
    del f, zz
    geo = ab["vmult"] - 16 * N
    vc_bytes = vcycle_algorithmic_bytes(M, geo)
    streamed = M.smoother_bytes(0) + 24 * N
    gbs = lambda b, ms: b / (ms * 1e-3) / 1e9  # noqa: E731
    return {
        "vmult": {"ms": t_vmult, "dofs_per_s": N / (t_vmult * 1e-3), "algorithmic_bytes": ab["vmult"],
                  "hbm_frac": gbs(ab["vmult"], t_vmult) / peak},
        "residual": {"ms": t_res, "algorithmic_bytes": ab["residual"], "hbm_frac": gbs(ab["residual"], t_res) / peak},
        "asm": {"ms": t_asm, "algorithmic_bytes": ab["asm"], "hbm_frac": gbs(ab["asm"], t_asm) / peak,
                "streamed_bytes": streamed, "streamed_frac": gbs(streamed, t_asm) / peak,
                "smoother_kind": M.smoother_kind(0)},
        "vcycle": {"ms": t_vc, "dofs_per_s": N / (t_vc * 1e-3), "algorithmic_bytes": vc_bytes,
                   "hbm_frac": gbs(vc_bytes, t_vc) / peak},
    }


def build(cfg, box=None):
    from paper_2408_04372_b200 import api
    if box is None:
        mesh = api.Mesh(cfg.dim, (0, 0, 0), (1, 1, 1), cfg.base_cells, cfg.refinements, cfg.vertices())
    else:
        mesh = api.Mesh(cfg.dim, (0, 0, 0), tuple(float(b) for b in box), box, cfg.refinements)
    return mesh


def cpu_baseline(workload: str, budget_s: float = 15.0, refinements: int = 3):
    """The reference's own C++ (oracle/_ref, single-threaded by construction)
    on a bounded, oracle-reachable sample of the workload: the same step
    (V-cycle + vmult) on the same configuration at `refinements`."""
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
                      f"in {el:.1f}s, setup {setup:.1f}s excluded; reference proj/src via oracle/_ref, 1 thread"}


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


def e2e_host_abi(M, op, r_dev, n_steps):
    """End to end through the host-buffer C ABI (the LinearMap plug-in path):
    every step hands pageable host vectors to stmg_multigrid_apply_host and
    stmg_st_operator_apply_host, which copy them in and the results out."""
    import numpy as np
    rh = r_dev.cpu().numpy().copy()
    zh = np.empty_like(rh)
    yh = np.empty_like(rh)
    M.apply_host(rh, zh)
    op.apply_host(zh, yh)  # warm-up: staging buffers allocated once
    t0 = time.perf_counter()
    for _ in range(n_steps):
        M.apply_host(rh, zh)
        op.apply_host(zh, yh)
    return (time.perf_counter() - t0) / n_steps, 2 * rh.nbytes


def e2e_pinned(step, r_dev, y_dev, n_steps):
    """End to end with pinned host buffers: each step's input H2D and result
    D2H on copy streams, overlapped with the neighbouring steps (ping-pong)."""
    import torch
    rh = torch.empty(r_dev.numel(), dtype=torch.float64).pin_memory()
    rh.copy_(r_dev.cpu())
    yh = torch.empty_like(rh).pin_memory()
    rb = [r_dev, torch.empty_like(r_dev)]
    yb = [y_dev, torch.empty_like(y_dev)]
    comp = torch.cuda.current_stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ready = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    read = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(h2d):
        rb[0].copy_(rh, non_blocking=True)
        ready[0].record(h2d)
    for i in range(n_steps):
        b = i % 2
        if i + 1 < n_steps:
            with torch.cuda.stream(h2d):
                if i >= 1:
                    h2d.wait_event(done[1 - b])
                rb[1 - b].copy_(rh, non_blocking=True)
                ready[1 - b].record(h2d)
        comp.wait_event(ready[b])
        if i >= 2:
            comp.wait_event(read[b])
        step(rb[b], yb[b])
        done[b].record(comp)
        with torch.cuda.stream(d2h):
            d2h.wait_event(done[b])
            yh.copy_(yb[b], non_blocking=True)
            read[b].record(d2h)
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n_steps


def measure_config(name, peak, with_solve=True):
    """One BASELINE config: vmult / residual / smoother / V-cycle figures, and
    one STMG-GMRES solve (manufactured RHS, rel. tol 1e-10)."""
    import torch

    from paper_2408_04372_b200 import api, problems
    cfg = problems.config(name)
    t0 = time.perf_counter()
    mesh = build(cfg)
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    op = M.operator_at(0)
    g = torch.Generator(device="cuda").manual_seed(7)
    r = torch.rand(op.n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z, y = torch.empty_like(r), torch.empty_like(r)
    out = {"n_dofs": op.n_dofs, **cfg.describe(), "setup_s": setup, "mg_levels": M.n_levels,
           "kernels": kernel_figures(cfg, M, op, r, z, y, peak)}
    if with_solve:
        out["solve"] = solve_once(cfg, M, op)
    del M, op, mesh, r, z, y
    torch.cuda.empty_cache()
    return out


def solve_once(cfg, M, op):
    import torch

    from paper_2408_04372_b200 import problems
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
        return {"iterations": info["iterations"], "converged": info["converged"], "ms": 1e3 * t_solve,
                "dofs_per_s": op.n_dofs / t_solve, "rhs": "manufactured source (frequency 0.5), zero entering state",
                "rel_tol": 1e-10}
    except Exception as e:  # noqa: BLE001 - reported, not fatal
        return {"error": str(e)[:200]}


def roofline_of(kern, ms_step, workload):
    """The dominant kernel of the step (largest share of the step's device
    time): the fine-level operator kernel (1 apply + 2 residuals per step) or
    the fine-level smoother (2 sweeps per step)."""
    op_share = (kern["vmult"]["ms"] + 2 * kern["residual"]["ms"]) / ms_step
    asm_share = 2 * kern["asm"]["ms"] / ms_step
    peak, peak_src = measured_peaks()
    if op_share >= asm_share:
        k, key, share = kern["vmult"], "vmult", op_share
        name = "st_brick_ws_kernel (fused space-time vmult, owner-computes Cartesian form, warp-specialised)"
    else:
        k, key, share = kern["asm"], "asm", asm_share
        name = "fine-level smoother sweep (ASMSmoother::add_correction)"
    achieved = k["algorithmic_bytes"] / (k["ms"] * 1e-3) / 1e9
    traffic = profile_entry(f"{workload}:{key}", "dram_bytes_per_launch")
    flops = profile_entry(f"{workload}:{key}", "fp64_flops_per_launch")
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": peak_src, "kernel": name, "launch_ms": k["ms"],
            "algorithmic_bytes_per_launch": k["algorithmic_bytes"],
            "bytes_definition": "SURVEY.md 8(d): vmult 16 N (+24 n_verts perturbed); smoother sweep 24 N",
            "share_of_step": share,
            "fp64": None if not flops else {"flops_per_launch": flops, "achieved_tflops": flops / (k["ms"] * 1e-3) / 1e12,
                                            "peak_tflops": FP64_PEAK_TFLOPS,
                                            "frac": flops / (k["ms"] * 1e-3) / 1e12 / FP64_PEAK_TFLOPS,
                                            "source": "executed DFMA/DADD/DMUL of the committed ncu capture"},
            "traffic_source": "profiles/ncu_kernels.json (ncu --set full, dram__bytes_read.sum + write.sum)"}


def run_single(args):
    import torch

    from paper_2408_04372_b200 import api, native, problems
    lib = native.load()
    torch.cuda.set_device(0)
    peak, _ = measured_peaks()
    cfg = problems.config(args.workload)
    t0 = time.perf_counter()
    mesh = build(cfg)
    M = api.SpaceTimeMultigrid(cfg.equation, cfg.scheme, mesh, cfg.rho, cfg.refinements, cfg.p, cfg.k, cfg.n_steps,
                               cfg.tau)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    print(f"[bench] {args.workload}: setup {setup_s:.1f}s, levels {M.level_info()}", file=sys.stderr, flush=True)
    op = M.operator_at(0)
    N = op.n_dofs
    g = torch.Generator(device="cuda").manual_seed(1234)
    r = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z, y = torch.empty_like(r), torch.empty_like(r)

    def step(rr=r, yy=y):
        M.apply(rr, z)
        op.apply(z, yy)

    warm = max(args.warmup, 3)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    launches0 = lib.stmg_kernel_launches()
    with ClockSampler(0) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        e1.synchronize()
    torch.cuda.synchronize()
    launches = (lib.stmg_kernel_launches() - launches0) // args.steps
    ms = e0.elapsed_time(e1) / args.steps
    value = N / (ms * 1e-3)

    kern = kernel_figures(cfg, M, op, r, z, y, peak)
    solve = solve_once(cfg, M, op)
    e2e_s, bytes_each = e2e_host_abi(M, op, r, max(2, min(args.steps, 3)))
    e2e_pin_s = e2e_pinned(step, r, y, max(4, min(args.steps, 10)))
    e2e = {"value": N / e2e_s, "unit": "DoF/s", "h2d_bytes_per_step": bytes_each, "d2h_bytes_per_step": bytes_each,
           "ms_per_step": 1e3 * e2e_s,
           "path": "stmg_multigrid_apply_host + stmg_st_operator_apply_host on pageable numpy buffers "
                   "(the INTEGRATION.md LinearMap plug-in), copies inside each step",
           "pinned_pipelined": {"value": N / e2e_pin_s, "ms_per_step": 1e3 * e2e_pin_s,
                                "path": "pinned torch buffers, H2D/D2H on copy streams overlapped with "
                                        "the neighbouring steps"}}
    line = {"metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": 1, "steps": args.steps, "warmup": warm,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, **cfg.describe(), "parallelism": "single GPU",
                       "step": "1 V-cycle + 1 vmult (one preconditioned GMRES iteration's operator work)",
                       "l2": "vectors (8N = %.0f MB each) larger than the 126 MB L2; no flush" % (8 * N / 1e6)},
            "roofline": roofline_of(kern, ms, args.workload), "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_note": "library kernels launched per timed step (coarse levels replay one CUDA graph)",
            "kernels": kern, "solve": solve, "setup_s": setup_s, "mg_levels": M.n_levels,
            "device_bytes": M.device_bytes(), "clocks": clk.summary()}
    del M, op, mesh, r, z, y
    torch.cuda.empty_cache()
    if not args.no_per_config:
        per = {}
        for name in args.per_config.split(","):
            if name and name != args.workload:
                try:
                    per[name] = measure_config(name, peak)
                except Exception as e:  # noqa: BLE001
                    per[name] = {"error": str(e)[:200]}
        line["per_config"] = per
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.workload, budget_s=args.cpu_budget)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def run_partitioned(args, world, rank, local):
    """N > 1: the C5 weak-scaling study. One 128^3-cell block
    per GPU (dist.weak_box), the box mesh cut into `world` z-slabs, rank r
    holds slab r; NCCL carries the interface-plane exchanges and the
    allreduces. value = total DoFs / max-over-ranks step time."""
    import torch
    import torch.distributed as dist

    from paper_2408_04372_b200 import api, native, problems
    from paper_2408_04372_b200 import dist as sdist

    lib = native.load()
    uid = [api.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = api.Comm(world, rank, uid[0])
    base = problems.config(args.workload)
    box = sdist.weak_box(world)
    t0 = time.perf_counter()
    mesh = build(base, box)
    S = api.SlabMultigrid(base.equation, base.scheme, mesh, None, base.refinements, base.p, base.k, base.n_steps,
                          base.tau, world, first_part=rank, local_parts=1, comm=comm)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    n_total = base.n_steps * base.n_t
    for a in range(3):
        n_total *= (box[a] << base.refinements) * base.p + 1
    n_local = S.n_local
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    r = torch.rand(n_local, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    z, y = torch.empty_like(r), torch.empty_like(r)

    def step(rr=r, yy=y):
        S.vcycle(rr, z)
        S.apply(z, yy)

    warm = max(args.warmup, 3)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    t_apply = timed(lambda: S.apply(r, y), 5)
    t_vc = timed(lambda: S.vcycle(r, z), 3)
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
    launches = (lib.stmg_kernel_launches() - launches0) // args.steps
    t = torch.tensor([e0.elapsed_time(e1) / args.steps, t_apply, t_vc], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms, t_apply, t_vc = (float(v) for v in t.tolist())
    value = n_total / (ms * 1e-3)
    # end to end: the local slab from pinned host memory and back, per step
    e2e_s = e2e_pinned(step, r, y, max(4, min(args.steps, 10)))
    tl = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    dist.all_reduce(tl, op=dist.ReduceOp.MAX)
    e2e = {"value": n_total / float(tl.item()), "unit": "DoF/s", "h2d_bytes_per_step": 8 * n_local,
           "d2h_bytes_per_step": 8 * n_local,
           "note": "per rank: its slab of the step's input H2D and result D2H (pinned, overlapped)"}
    peak, peak_src = measured_peaks()
    vm_bytes = 16 * n_local
    achieved = vm_bytes / (t_apply * 1e-3) / 1e9
    line = {"metric": METRIC, "value": value, "unit": "DoF/s", "n_gpus": world, "steps": args.steps,
            "warmup": warm, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C5 weak: 128^3 cells per GPU, box {box[0]}x{box[1]}x{box[2]} x 128^3",
                       "cells": [b << base.refinements for b in box], "p": base.p, "k": base.k,
                       "n_dofs": n_total, "parallelism": f"z-slab x{world}", "partitioned_levels": S.dist_levels,
                       "step": "1 V-cycle + 1 vmult (one preconditioned GMRES iteration's operator work)",
                       "l2": "vectors larger than L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": profile_entry("C5-128:vmult", "dram_bytes_per_launch"),
                         "peak_source": peak_src, "kernel": "rank-local vmult incl. interface exchange",
                         "algorithmic_bytes_per_launch": vm_bytes, "launch_ms": t_apply},
            "kernels": {"vmult_ms": t_apply, "vcycle_ms": t_vc},
            "e2e": e2e, "gpu_launches": int(launches), "setup_s": setup_s, "clocks": clk.summary()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    del S, comm
    dist.destroy_process_group()


def spawn_ranks(args):
    """--gpus N without a torch.distributed environment: launch N ranks."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or args.partitioned:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        torch.cuda.set_device(local)
        if not dist.is_initialized():
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        return run_partitioned(args, world, rank, local)
    return run_single(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5-128")
    ap.add_argument("--per-config", default="C2,C3,C4")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--ref-refinements", type=int, default=3)
    ap.add_argument("--ref-replicas", type=int, default=0,
                    help="reference arm: concurrent single-threaded replicas (0: one per host thread)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="run the N > 1 partitioned code path even with one rank (plumbing check)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    run_ours(args)


if __name__ == "__main__":
    main()
