#!/usr/bin/env python3
"""Benchmark of the B200 GMG V-cycle hot path (BASELINE.json metric on configs[1] = C2).

One step = one complete solve_outer (multigrid.cpp:210-246) of the C2 problem — 3D Q1
Poisson on 128^3 cells (2,146,689 DOFs), 7 levels from 2^3, f = 3 pi^2 sin sin sin,
g = 0, V(2,2) damped Jacobi omega = 0.8, stop at 1e-10 relative residual — from x0 = 0.
value = DOFs/s = n_global * steps / (device time of the steps), max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

N > 1 runs under torchrun (one process per GPU, NCCL halo exchange and allreduce),
partitioning the same global problem into N boxes (strong scaling).  --impl
reference times the reference's own CPU solver (oracle/_ref, the unmodified
/root/reference/proj library) on the host cores on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(dim=3, n_coarse=2, levels=7, pre=2, post=2, omega=0.8, tol=1e-10)
METRIC = "GMG solve DOFs/s (solve_outer to 1e-10 rel. residual, V(2,2) damped Jacobi w=0.8)"
CONFIG = {
    "workload": "C2: 3D Poisson -Lap u = f, unit cube, 128^3 hex cells (2,146,689 DOFs), conforming "
                "Q1, fp64, 7 levels from 2^3, V(2,2) damped Jacobi w=0.8, coarse GS, stop at 1e-10",
    "n_dofs": 2146689,
    "levels": 7,
    "cells": "128^3",
    "smoother": "damped_jacobi_0.8",
    "l2_flush": "no flush: the finest-level operator (0.69 GB) and the whole hierarchy (~0.8 GB) "
                "exceed the 126 MB L2, so every step streams the matrices from HBM",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling (B200_PROFILING.md clocks line), started before the run and
    filtered to the timed region by timestamp."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"pf_clocks_{os.getpid()}.csv")
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def stop(self):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()

    def window(self, t0, t1):
        self.windows.append((t0, t1))

    def summary(self, first: int = 0, last: int | None = None):
        """Clock samples inside timed windows [first, last) (default: all)."""
        import datetime
        windows = self.windows[first:last]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons, n_all = [], None, set(), 0
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 8 or not f[1].isdigit():
                    continue
                n_all += 1
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                except ValueError:
                    continue
                if not any(t0 - 0.02 <= ts <= t1 + 0.02 for t0, t1 in windows):
                    continue
                sm.append(int(f[1]))
                mx = int(f[2])
                for n, v in zip(names, f[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
        except OSError:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic():
    """(DRAM bytes per finest-level Jacobi launch, where they come from): the committed
    ncu --set full capture of this kernel (profiles/ncu_summary.json, refreshed from the
    current build each round; ncu cannot run inside the timed bench)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f).get("k_jacobi_c2", {})
        return s.get("dram_bytes_per_launch"), s.get("source")
    except Exception:
        return None, None


def cpu_baseline(steps_hint: int = 1):
    """The reference CPU solver (oracle/_ref) on this host, bounded to one solve of C2."""
    from oracle import ref
    ranks = max(1, min(8, os.cpu_count() or 1))
    if ref.available():
        r = ref.bench(3, 2, WORKLOAD["levels"], ranks, smoother=0, damping=WORKLOAD["omega"],
                      pre=2, post=2, outer_tol=WORKLOAD["tol"], warmup=0, steps=steps_hint)
        t = float(min(r["step_seconds"]))
        return {"value": r["n_global"] / t, "unit": "DOF/s", "cores": ranks, "kind": "reference",
                "sample": f"{steps_hint} full solve_outer of C2 (128^3, {r['iterations']} V(2,2) "
                          f"Jacobi cycles) on {ranks} reference ranks (threads); setup "
                          f"{r['setup_seconds']:.1f}s excluded",
                "solve_seconds": t}
    from oracle.restated import Oracle
    from paper_1609_04809_b200.levels import StructuredSetup
    from paper_1609_04809_b200.gmg import MultigridConfig, SmootherConfig
    s = StructuredSetup(3, 2, WORKLOAD["levels"], 1, 0)
    o = Oracle([s.levels])
    cfg = MultigridConfig(smoother=SmootherConfig(kind=0, damping=0.8), pre_smooth=2, post_smooth=2,
                          outer_tol=1e-10)
    t0 = time.perf_counter()
    _, res, st, _ = o.solve_outer([s.x0], [s.b], cfg)
    t = time.perf_counter() - t0
    return {"value": s.n_global / t, "unit": "DOF/s", "cores": 1, "kind": "port",
            "sample": f"1 solve_outer of C2 ({st.iterations} cycles) with the C restatement",
            "solve_seconds": t}


def run_reference(args):
    """--impl reference: the reference's own CPU solver, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.config == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "C5 (512^3, lognormal coefficient): the reference "
                          "assembles constant-coefficient Q1 only and its setup needs ~4 GB and 57 s per 2M "
                          "DOFs (SURVEY.md 8d); C2 is the configuration both arms run (bench.py --config c2)"}))
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparfem_ref.so not built"}))
        return
    ranks = max(1, min(8, os.cpu_count() or 1))
    r = ref.bench(3, 2, WORKLOAD["levels"], ranks, smoother=0, damping=WORKLOAD["omega"], pre=2, post=2,
                  outer_tol=WORKLOAD["tol"], warmup=args.warmup, steps=args.steps)
    total = float(sum(r["step_seconds"]))
    value = r["n_global"] * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic manufactured problem (f = 3 pi^2 sin sin sin, g = 0)",
        "config": dict(CONFIG, parallelism=f"{ranks} reference ranks (std::thread) on host cores"),
        "cycles": r["iterations"],
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": ranks, "kind": "reference",
                         "sample": f"{args.steps} full C2 solves after {args.warmup} warm-up, "
                                   f"setup {r['setup_seconds']:.1f}s excluded"},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def share_host_cores():
    """One process per GPU on a shared host: give this rank its share of the cores for the
    library's OpenMP setup / upload work (torchrun sets OMP_NUM_THREADS=1 for every rank,
    which makes the 512^3 box setup several times slower)."""
    from paper_1609_04809_b200 import gmg
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    return gmg.set_host_threads(max(1, (os.cpu_count() or 1) // max(1, local_world)))


def run_b200(args):
    import numpy as np
    import torch

    from paper_1609_04809_b200 import gmg
    from paper_1609_04809_b200.levels import StructuredSetup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    clk = Clocks(local).start()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # host plumbing only: the data plane is libpf_gpu.so's
        share_host_cores()

    W = WORKLOAD
    t0 = time.time()
    # multi-process: direct halo lists + fused exchanges (one message group per sweep for
    # master/slave + halo1, + halo2 after each smoothing phase; results unchanged), and
    # every rank's bottom levels replicated on each GPU (one allgather per cycle feeds a
    # redundant bottom V-cycle instead of per-sweep exchanges on the tiny levels)
    multi = world > 1
    setup = StructuredSetup(W["dim"], W["n_coarse"], W["levels"], world, rank, direct_halos=multi)
    replicas = (gmg.replica_levels(W["dim"], W["n_coarse"], W["levels"], world, direct_halos=True)
                if multi else None)
    h = gmg.Hierarchy([setup.levels], device=local, rank_base=rank, world_size=world,
                      coarse_replicas=replicas, fused_exchanges=multi)
    used = attach_transport(h, world, rank, args.transport, dist) if world > 1 else None
    setup_s = time.time() - t0
    top = h.finest
    cfg = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, damping=W["omega"]),
                              pre_smooth=W["pre"], post_smooth=W["post"], outer_tol=W["tol"])
    x0 = h.vector(top, setup.x0)
    b = h.vector(top, setup.b)
    x = h.vector(top)
    stream = torch.cuda.ExternalStream(h.stream_handle(), device=torch.device("cuda", local))

    def step(c):
        x.copy_from(x0)
        return gmg.solve_outer(h, x, b, c)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def timed(c, steps):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record(stream)
        st = None
        for _ in range(steps):
            st = step(c)
        e1.record(stream)
        barrier()
        clk.window(w0, time.time())
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, st

    for _ in range(args.warmup):
        st = step(cfg)
    n0 = h.launch_count()
    ms, st = timed(cfg, args.steps)
    launches = h.launch_count() - n0
    value = setup.n_global * args.steps / (ms / 1e3)

    # e2e: the same solve through the host-buffer entry point (pinned host x0/b in,
    # solution out, copies inside the timed region)
    xh = torch.empty(len(setup.x0), dtype=torch.float64).pin_memory().numpy()
    bh = torch.from_numpy(setup.b.copy()).pin_memory().numpy()
    for _ in range(max(1, args.warmup)):
        xh[:] = setup.x0
        gmg.solve_outer_host(h, [xh], [bh], cfg)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_ms = 0.0
    w0 = time.time()
    for _ in range(args.steps):
        # the host-side reset of the in/out start vector is not part of the step (the
        # reference arm resets its start vector outside its timed region too)
        xh[:] = setup.x0
        torch.cuda.synchronize()
        e0.record(stream)
        gmg.solve_outer_host(h, [xh], [bh], cfg)  # H2D x0, b; solve; D2H x
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    barrier()
    clk.window(w0, time.time())
    n_headline_windows = len(clk.windows)
    if dist:
        t = torch.tensor([e2e_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = setup.n_global * args.steps / (e2e_ms / 1e3)

    # dominant kernel: finest-level Jacobi sweep (4 of the ~5.5 matrix passes per cycle)
    sweep_ms, sweep_bytes = h.time_sweep(top, gmg.PF_SMOOTHER_JACOBI, 50)
    sor_ms, _ = h.time_sweep(top, gmg.PF_SMOOTHER_MULTICOLOR_SOR, 20)
    vcycle_ms = h.time_vcycle(x, b, cfg, 20)
    peak, peak_src = peaks()
    # SURVEY.md §8(d)'s algorithmic bytes of one sweep (the canonical roofline figure: fp64
    # CSR, int32 columns and row pointers): 12 z + 4 n + 8 m + 8 n (b) + 8 n (out), n own
    # rows, z their entries, m the distinct columns they touch
    fin = setup.levels[-1]
    z_own = int(fin.row_offsets[fin.n_own])
    m_cols = int(np.unique(fin.cols[:z_own]).size)
    alg_bytes = 12 * z_own + 4 * fin.n_own + 8 * m_cols + 16 * fin.n_own
    achieved = alg_bytes / (sweep_ms / 1e3) / 1e9
    achieved_stored = sweep_bytes / (sweep_ms / 1e3) / 1e9
    traffic, traffic_src = ncu_traffic()

    # multicolour SOR w=1.2 variant of the same config (BASELINE configs[1])
    sor = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=1.2),
                              pre_smooth=2, post_smooth=2, outer_tol=W["tol"])
    for _ in range(2):
        st_sor = step(sor)
    sor_ms_total, st_sor = timed(sor, max(3, args.steps // 2))
    sor_steps = max(3, args.steps // 2)

    # lognormal(0,1) per-cell coefficient on the same grid (BASELINE configs 3-4's
    # coefficient; not in the reference): every operator value distinct, fp64 storage
    logn = None
    if world == 1:
        ls = StructuredSetup(W["dim"], W["n_coarse"], W["levels"], 1, 0, gmg._lib.PF_PROBLEM_LOGNORMAL, seed=2024)
        lh = gmg.Hierarchy([ls.levels], device=local)
        lc = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, damping=W["omega"]),
                                 pre_smooth=W["pre"], post_smooth=W["post"], outer_tol=W["tol"],
                                 outer_max_cycles=200)
        lx, lb = lh.vector(top, ls.x0), lh.vector(top, ls.b)
        lstream = torch.cuda.ExternalStream(lh.stream_handle(), device=torch.device("cuda", local))
        lst = gmg.solve_outer(lh, lx, lb, lc)
        torch.cuda.synchronize()
        l_steps = 3
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record(lstream)
        for _ in range(l_steps):
            lx.upload(ls.x0)
            lst = gmg.solve_outer(lh, lx, lb, lc)
        e1.record(lstream)
        torch.cuda.synchronize()
        clk.window(w0, time.time())
        l_ms = e0.elapsed_time(e1) / l_steps
        l_sweep_ms, l_sweep_bytes = lh.time_sweep(top, gmg.PF_SMOOTHER_JACOBI, 20)
        logn = {"value": ls.n_global / (l_ms / 1e3), "unit": "DOF/s", "cycles": lst.iterations,
                "ms_per_step": l_ms, "sweep_us": l_sweep_ms * 1e3,
                "sweep_gbs": l_sweep_bytes / (l_sweep_ms / 1e3) / 1e9,
                "sweep_frac": l_sweep_bytes / (l_sweep_ms / 1e3) / 1e9 / peak,
                "note": "fp64 SELL-32x4 values (12 B per entry): the finest sweep at the HBM roofline"}
        lh.close()

    # BASELINE configs[2] (Q2, 64^3 cells, 129^3 dofs, 6 levels, V(3,3)) and configs[3]
    # (rotated Q1, 128^3 cells, 6.3M face dofs, lognormal(0,1) coefficient, 7 levels):
    # include/pf_fe.h, direct coarse solve (BASELINE configs[0]'s "coarse direct solve")
    fe = {}
    if world == 1 and not args.no_fe:
        from paper_1609_04809_b200.fe import LOGNORMAL, Q2, ROTATED_Q1, CONSTANT, FESetup

        def fe_variant(family, coef, levels, pp, kind, omega):
            fs = FESetup(family, 2, levels, coef, seed=2024)
            fh = gmg.Hierarchy([fs.levels], device=local).set_coarse_direct()
            fc = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=kind, damping=omega), pre_smooth=pp,
                                     post_smooth=pp, outer_tol=W["tol"], outer_max_cycles=400)
            ftop = levels - 1
            fx, fb = fh.vector(ftop, fs.x0), fh.vector(ftop, fs.b)
            fstream = torch.cuda.ExternalStream(fh.stream_handle(), device=torch.device("cuda", local))
            fst = gmg.solve_outer(fh, fx, fb, fc)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.time()
            e0.record(fstream)
            for _ in range(3):
                fx.upload(fs.x0)
                fst = gmg.solve_outer(fh, fx, fb, fc)
            e1.record(fstream)
            torch.cuda.synchronize()
            clk.window(w0, time.time())
            f_ms = e0.elapsed_time(e1) / 3
            err = float(np.abs(fx.download(0) - fs.exact).max())
            sw_ms, sw_bytes = fh.time_sweep(ftop, gmg.PF_SMOOTHER_JACOBI, 20)
            out = {"value": fs.n_global / (f_ms / 1e3), "unit": "DOF/s", "n_global": fs.n_global,
                   "nnz": int(fs.levels[-1].row_offsets[-1]), "cycles": fst.iterations,
                   "converged": bool(fst.converged), "ms_per_step": f_ms,
                   "vcycle_ms": fh.time_vcycle(fx, fb, fc, 10), "max_error_vs_exact": err,
                   "jacobi_sweep_us": sw_ms * 1e3, "jacobi_sweep_gbs": sw_bytes / (sw_ms / 1e3) / 1e9,
                   "jacobi_sweep_frac": sw_bytes / (sw_ms / 1e3) / 1e9 / peak, "coarse": "direct"}
            fh.close()
            return out

        def fe_k8_colorwise(omega):
            """configs[3] on 8 subdomains ("1 and 8 GPUs"): the partitioned rotated-Q1
            lognormal hierarchy, all 8 subdomains on this GPU, SOR with the colour-wise
            exchange (processor-local smoothing diverges here)."""
            fs = [FESetup(ROTATED_Q1, 2, 7, LOGNORMAL, seed=2024, n_ranks=8, rank=r) for r in range(8)]
            fh = gmg.Hierarchy([f.levels for f in fs], device=local).set_colorwise_exchange()
            fc = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=omega),
                                     pre_smooth=2, post_smooth=2, outer_tol=W["tol"], outer_max_cycles=400)
            fx = fh.vector(6, [f.x0 for f in fs])
            fb = fh.vector(6, [f.b for f in fs])
            fstream = torch.cuda.ExternalStream(fh.stream_handle(), device=torch.device("cuda", local))
            fst = gmg.solve_outer(fh, fx, fb, fc)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.time()
            e0.record(fstream)
            for _ in range(2):
                for r, f in enumerate(fs):
                    fx.upload(f.x0, r)
                fst = gmg.solve_outer(fh, fx, fb, fc)
            e1.record(fstream)
            torch.cuda.synchronize()
            clk.window(w0, time.time())
            f_ms = e0.elapsed_time(e1) / 2
            n_global = 3 * 128 * 128 * 129
            out = {"value": n_global / (f_ms / 1e3), "unit": "DOF/s", "n_global": n_global, "subdomains": 8,
                   "cycles": fst.iterations, "converged": bool(fst.converged), "ms_per_step": f_ms,
                   "vcycle_ms": fh.time_vcycle(fx, fb, fc, 5), "exchange": "colour-wise",
                   "note": "8 box subdomains of the 1-GPU configs[3] problem on one GPU (device-local "
                           "exchanges); the processor-local reference smoothing diverges at K=8"}
            fh.close()
            return out

        fe["q2_c3_jacobi_v33"] = fe_variant(Q2, CONSTANT, 6, 3, gmg.PF_SMOOTHER_JACOBI, W["omega"])
        # omega 1.6: 68 cycles at 128^3 (1.2: 101, 1.4: 81, 1.8: 156; tools/fe_run.py)
        fe["rotated_q1_c4_lognormal_sor_1.6"] = fe_variant(ROTATED_Q1, LOGNORMAL, 7, 2,
                                                          gmg.PF_SMOOTHER_MULTICOLOR_SOR, 1.6)
        fe["rotated_q1_c4_lognormal_sor_1.6_k8_colorwise"] = fe_k8_colorwise(1.6)

    # BASELINE configs[4] (C5: 512^3, lognormal, SOR) on this one GPU: the N = 1 point of the
    # scaling configuration (bench.py --gpus N runs it on N GPUs)
    c5 = None
    if world == 1 and not args.no_c5:
        import types
        h.close()
        c5h, c5s, c5_setup, c5_upload, _ = c5_hierarchy(1, 0, local, args.transport, None)
        m = c5_solve(c5h, c5s, 1, 0, types.SimpleNamespace(steps=2, warmup=1), clk, None, local, "c5")
        c5 = {"value": m["value"], "unit": "DOF/s", "n_global": c5s.n_global, "cycles": m["cycles"],
              "converged": m["converged"], "ms_per_step": m["ms_per_step"], "vcycle_ms": m["vcycle_ms"],
              "e2e": m["e2e"], "sor_sweep_us": m["sor_sweep_ms"] * 1e3,
              "sor_sweep_frac_on_stored_bytes": m["sor_sweep_bytes"] / m["sor_sweep_ms"] / 1e6 / peak,
              "jacobi_sweep_us": m["jacobi_sweep_ms"] * 1e3,
              "jacobi_sweep_frac_on_stored_bytes": m["jacobi_sweep_bytes"] / m["jacobi_sweep_ms"] / 1e6 / peak,
              "setup_seconds": c5_setup, "upload_seconds": c5_upload, "steps": 2,
              "config": C5_CONFIG["workload"]}
        c5h.close()
    clk.stop()
    clocks = clk.summary(0, n_headline_windows)  # the headline's timed region
    clocks["variants"] = clk.summary(n_headline_windows)  # the variants' timed regions
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline()
        except Exception as e:  # reported, never fatal for the GPU number
            cpu = {"value": None, "unit": "DOF/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic manufactured problem (f = 3 pi^2 sin sin sin, g = 0), product setup",
        "config": dict(CONFIG, parallelism=f"{world} box subdomain(s), one per GPU, {used} exchanges" if world > 1
                       else "1 GPU"),
        "cycles": st.iterations, "final_rel_residual": st.final_residual / st.initial_residual,
        "vcycle_ms": vcycle_ms,
        "roofline": {"bound": "hbm", "achieved": achieved_stored, "peak": peak, "unit": "GB/s",
                     "frac": achieved_stored / peak, "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": "k_jacobi (finest-level damped-Jacobi sweep; SELL-32x4, int32 columns, "
                               "8-bit index into the table of distinct fp64 values staged in shared "
                               "memory, row-start L2 prefetch, 48 registers / 5 blocks per SM)",
                     "kernel_us": sweep_ms * 1e3, "bytes_per_launch": sweep_bytes,
                     "bytes_formula": "(4 + 1) z + 4 n + 8 m + 16 n: the bytes the kernel streams (int32 "
                                      "column + 1 B value index per own-row entry, row length, x once, b, out)",
                     "fp64_csr_equivalent": {
                         "bytes_per_launch": alg_bytes,
                         "formula": "SURVEY.md 8(d): 12 z + 4 n + 8 m + 16 n (fp64 CSR)",
                         "achieved": achieved, "note": "work-equivalent rate: the lossless value index "
                         "moves 5 instead of 12 B per entry, so this exceeds the HBM peak"},
                     "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "DOF/s", "h2d_bytes_per_step": 16 * len(setup.x0),
                "d2h_bytes_per_step": 8 * len(setup.x0), "ms_per_step": e2e_ms / args.steps},
        "gpu_launches": launches,
        "clocks": clocks,
        "setup_seconds": setup_s,
        "variants": {"multicolor_sor_1.2": {
            "value": setup.n_global * sor_steps / (sor_ms_total / 1e3), "unit": "DOF/s",
            "cycles": st_sor.iterations, "ms_per_step": sor_ms_total / sor_steps,
            "sweep_us": sor_ms * 1e3,
            "sweep_frac": alg_bytes / (sor_ms / 1e3) / 1e9 / peak,
            "sweep_frac_on_stored_bytes": sweep_bytes / (sor_ms / 1e3) / 1e9 / peak},
            "lognormal_jacobi": logn, **fe, "c5_512cubed_lognormal_sor_1.2_n1": c5},
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


# --config c5: BASELINE configs[4], the north star's scaling configuration — Q1 on 512^3
# cells (135,005,697 DOFs, 9 levels), lognormal(0,1) per-cell coefficient from a seed,
# V(2,2) multicolour SOR, box-partitioned into N subdomains (partition.cpp:104-142), one
# per GPU, exchanges through the peer-memory transport (CUDA IPC over NVLink: each exchange
# one kernel storing into the peer GPUs' memory, recorded into the solve's CUDA graph) or
# NCCL (--transport nccl).  The total problem is fixed, so N = 1, 2, 4, 8 is strong scaling.
C5 = dict(dim=3, n_coarse=2, levels=9, pre=2, post=2, omega=1.2, tol=1e-10, seed=2024)
C5_METRIC = "GMG solve DOFs/s (solve_outer to 1e-10 rel. residual, V(2,2) multicolour SOR w=1.2, lognormal coefficient)"
C5_CONFIG = {
    "workload": "C5: 3D Q1 -div(kappa grad u) = f, unit cube, 512^3 hex cells (135,005,697 DOFs), fp64, "
                "kappa lognormal(0,1) per finest cell (seed 2024), 9 levels from 2^3, V(2,2) multicolour SOR "
                "w=1.2, replicated coarse levels, stop at 1e-10",
    "n_dofs": 135005697, "levels": 9, "cells": "512^3", "smoother": "multicolor_sor_1.2",
    "l2_flush": "no flush: the finest operator (43.6 GB on one GPU, 5.4 GB per GPU at N=8) exceeds the 126 MB L2",
}


def c5_n1_reference():
    """The one-GPU value of THIS configuration, for strong-scaling efficiency: the default
    `python bench.py` (N = 1) headlines C2 and measures C5 on one GPU as a variant, so the
    N = 1 line's `value` is not the denominator of an N > 1 C5 line.  Read from the last
    committed one-GPU bench line (another run, possibly another box: say so)."""
    src = os.path.join("profiles", "r02_bench_c2_latest.json")
    try:
        with open(os.path.join(ROOT, src)) as f:
            v = json.load(f)["variants"]["c5_512cubed_lognormal_sor_1.2_n1"]
        return {"value": v["value"], "unit": "DOF/s", "ms_per_step": v["ms_per_step"], "cycles": v["cycles"],
                "source": f"{src} variants.c5_512cubed_lognormal_sor_1.2_n1 (committed one-GPU run of the same "
                          "configuration; `python bench.py --gpus 1 --config c5` measures it live)"}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "source": f"{src} unreadable ({e}); run `python bench.py --gpus 1 --config c5`"}


def c5_solve(h, setup, world, rank, args, clk, dist, local, label):
    """Time solve_outer of an uploaded C5 hierarchy (device-resident and through host
    buffers); returns the measurement dict (rank-local figures, max-over-ranks times)."""
    import torch

    from paper_1609_04809_b200 import gmg
    W = C5
    top = h.finest
    cfg = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_MULTICOLOR_SOR, damping=W["omega"]),
                              pre_smooth=W["pre"], post_smooth=W["post"], outer_tol=W["tol"], outer_max_cycles=400)
    x0 = h.vector(top, setup.x0)
    b = h.vector(top, setup.b)
    x = h.vector(top)
    stream = torch.cuda.ExternalStream(h.stream_handle(), device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(v):
        if not dist:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    st = None
    for _ in range(args.warmup):
        x.copy_from(x0)
        st = gmg.solve_outer(h, x, b, cfg)
    barrier()
    n0 = h.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        x.copy_from(x0)
        st = gmg.solve_outer(h, x, b, cfg)
    e1.record(stream)
    barrier()
    clk.window(w0, time.time())
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = h.launch_count() - n0
    # e2e: pinned host x0 / b in, solution out, through the host-buffer entry point
    xh = torch.empty(len(setup.x0), dtype=torch.float64).pin_memory().numpy()
    bh = torch.from_numpy(setup.b.copy()).pin_memory().numpy()
    e2e_ms = 0.0
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(e2e_steps):
        xh[:] = setup.x0
        barrier()
        e0.record(stream)
        gmg.solve_outer_host(h, [xh], [bh], cfg)
        e1.record(stream)
        e1.synchronize()
        e2e_ms += e0.elapsed_time(e1)
    barrier()
    e2e_ms = max_over_ranks(e2e_ms)
    vc_ms = max_over_ranks(h.time_vcycle(x, b, cfg, 3))
    sor_ms, sor_bytes = h.time_sweep(top, gmg.PF_SMOOTHER_MULTICOLOR_SOR, 5)
    jac_ms, jac_bytes = h.time_sweep(top, gmg.PF_SMOOTHER_JACOBI, 5)
    n = setup.n_global
    return {"value": n * args.steps / (ms / 1e3), "ms_per_step": ms / args.steps, "cycles": st.iterations,
            "converged": bool(st.converged), "final_rel_residual": st.final_residual / st.initial_residual,
            "vcycle_ms": vc_ms, "launches": launches,
            "e2e": {"value": n * e2e_steps / (e2e_ms / 1e3), "unit": "DOF/s",
                    "h2d_bytes_per_step": 16 * len(setup.x0), "d2h_bytes_per_step": 8 * len(setup.x0),
                    "ms_per_step": e2e_ms / e2e_steps},
            "sor_sweep_ms": sor_ms, "sor_sweep_bytes": sor_bytes, "jacobi_sweep_ms": jac_ms,
            "jacobi_sweep_bytes": jac_bytes, "x0": x0, "b": b, "x": x}


def attach_transport(h, world, rank, transport, dist):
    """The multi-GPU data plane of hierarchy h: peer-memory exchanges (CUDA IPC over NVLink,
    pf_peer.cu) by default — if any rank cannot map its peers, every rank falls back to
    NCCL together — or NCCL.  Returns what was attached."""
    from paper_1609_04809_b200 import dist as pdist
    from paper_1609_04809_b200 import gmg
    used = None
    if transport == "peer":
        err = None
        try:
            pdist.init_peer_transport(h, pdist.allgather_blobs_torch)
        except Exception as e:  # noqa: BLE001
            err = f"{type(e).__name__}: {e}"
        errs = [None] * world
        dist.all_gather_object(errs, err)
        failed = [(r, e) for r, e in enumerate(errs) if e]
        if not failed:
            return "peer"
        h.drop_transport()
        used = f"nccl (peer transport failed on rank {failed[0][0]}: {failed[0][1]})"
    uid = [gmg.Hierarchy.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, 0)
    h.init_nccl(uid[0])
    return used or "nccl"


def c5_hierarchy(world, rank, local, transport, dist):
    """Rank `rank`'s box of the C5 problem on its GPU (replicated bottom levels gathered from
    their owners, no other rank's setup built), with its transport attached."""
    from paper_1609_04809_b200 import dist as pdist
    from paper_1609_04809_b200 import gmg
    from paper_1609_04809_b200.levels import StructuredSetup
    W = C5
    t0 = time.time()
    setup = StructuredSetup(W["dim"], W["n_coarse"], W["levels"], world, rank, gmg._lib.PF_PROBLEM_LOGNORMAL,
                            seed=W["seed"], direct_halos=world > 1, materialize=False)
    setup_s = time.time() - t0
    replicas = None
    if world > 1:
        def gather(obj):
            out = [None] * world
            dist.all_gather_object(out, obj)
            return out
        replicas = gmg.gather_replica_levels(setup, gather)
    t0 = time.time()
    h = gmg.Hierarchy.from_setups([setup], device=local, rank_base=rank, world_size=world,
                                  coarse_replicas=replicas, fused_exchanges=world > 1)
    upload_s = time.time() - t0
    used = attach_transport(h, world, rank, transport, dist) if world > 1 else None
    return h, setup, setup_s, upload_s, used


def run_c5(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional checks of the multi-process path on a one-GPU box: PF_BENCH_DEVICE=0 puts
    # every rank on device 0 (CUDA IPC between processes); PF_BENCH_C5_LEVELS shrinks the grid
    if os.environ.get("PF_BENCH_DEVICE") is not None:
        local = int(os.environ["PF_BENCH_DEVICE"])
    if os.environ.get("PF_BENCH_C5_LEVELS"):
        C5["levels"] = int(os.environ["PF_BENCH_C5_LEVELS"])
        C5_CONFIG["workload"] += f" [REDUCED: {C5['levels']} levels]"
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    clk = Clocks(local).start()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")  # host plumbing only: the data plane is libpf_gpu.so's
    host_threads = share_host_cores()
    h, setup, setup_s, upload_s, used = c5_hierarchy(world, rank, local, args.transport, dist)
    m = c5_solve(h, setup, world, rank, args, clk, dist, local, "c5")
    clk.stop()
    peak, peak_src = peaks()
    # per-GPU finest-level sweeps on the bytes they move (fp64 SELL-32x4: 12 B per stored
    # entry + row lengths + x gather + b): the multicolour SOR sweep is the dominant kernel
    sor_gbs = m["sor_sweep_bytes"] / m["sor_sweep_ms"] / 1e6
    jac_gbs = m["jacobi_sweep_bytes"] / m["jacobi_sweep_ms"] / 1e6
    fracs = [sor_gbs / peak, jac_gbs / peak]
    if dist:
        t = torch.tensor(fracs, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        fracs = t.tolist()
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": C5_METRIC, "value": m["value"], "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": m["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic manufactured problem (f = 3 pi^2 sin sin sin, g = 0, seeded lognormal kappa), "
                    "product setup",
            "config": dict(C5_CONFIG, parallelism=(f"{world} box subdomains (coordinate bisection), one per GPU, "
                                                   f"{used} exchanges" if world > 1 else "1 GPU"),
                           transport=used),
            "cycles": m["cycles"], "converged": m["converged"], "final_rel_residual": m["final_rel_residual"],
            "vcycle_ms": m["vcycle_ms"],
            "roofline": {"bound": "hbm", "achieved": sor_gbs, "peak": peak, "unit": "GB/s", "frac": sor_gbs / peak,
                         "traffic": None, "kernel": "k_color_sweep (finest multicolour SOR sweep, 8 colours, "
                         "fp64 SELL-32x4), rank 0",
                         "kernel_us": m["sor_sweep_ms"] * 1e3, "stored_bytes_per_launch": m["sor_sweep_bytes"],
                         "min_frac_over_ranks": fracs[0], "peak_source": peak_src},
            "finest_jacobi_sweep": {"us": m["jacobi_sweep_ms"] * 1e3, "gbs": jac_gbs, "frac": jac_gbs / peak,
                                    "min_frac_over_ranks": fracs[1]},
            "cpu_baseline": None,
            "cpu_baseline_note": "the reference CPU solver cannot hold 512^3 (57 s and 4.2 GB at 128^3; "
                                 "SURVEY.md 8d): not run",
            "e2e": m["e2e"], "gpu_launches": m["launches"], "clocks": clocks,
            "setup_seconds": setup_s, "upload_seconds": upload_s, "host_threads_per_rank": host_threads,
        }
        if world > 1:
            line["n1_same_config"] = c5_n1_reference()
        print(json.dumps(line), flush=True)
    h.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


# --workload heat: the reference's model problem (app.cpp:146-230), Crank-Nicolson on the
# C2 grid; one step = one time step (device load assembly, CN right-hand side, solve_outer).
HEAT = dict(dim=3, n_coarse=2, levels=7, dt=0.01, pre=2, post=2, omega=0.8, tol=1e-10)
HEAT_METRIC = "CN heat time steps DOF-steps/s (load + rhs + solve_outer to 1e-10, V(2,2) Jacobi w=0.8)"
HEAT_CONFIG = {
    "workload": "heat: u_t - Lap u = f, u = exp(-t/10) sin(pi x) cos(pi y) cos(pi z), unit cube, "
                "128^3 Q1 cells (2,146,689 DOFs), Crank-Nicolson dt = 0.01, 7 levels, V(2,2) damped "
                "Jacobi w=0.8, stop at 1e-10 (the reference's run_heat at C2 size)",
    "n_dofs": 2146689, "levels": 7, "cells": "128^3", "dt": 0.01,
    "l2_flush": "no flush: operator + rhs operator + hierarchy (~1.5 GB) exceed the 126 MB L2",
}


def run_reference_heat(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libparfem_ref.so not built"}))
        return
    ranks = max(1, min(8, os.cpu_count() or 1))
    H = HEAT
    steps = min(args.steps, 3)
    r = ref.heat_bench(H["dim"], H["n_coarse"], H["levels"], ranks, dt=H["dt"], damping=H["omega"],
                       pre=H["pre"], post=H["post"], outer_tol=H["tol"], warmup=1, steps=steps)
    total = float(sum(r["step_seconds"]))
    value = r["n_global"] * steps / total
    line = {
        "impl": "reference", "metric": HEAT_METRIC, "value": value, "unit": "DOF-steps/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": 1, "ms_per_step": 1e3 * total / steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "manufactured heat problem of the reference (model.cpp:19-31)",
        "config": dict(HEAT_CONFIG, parallelism=f"{ranks} reference ranks (std::thread) on host cores"),
        "cycles_last_step": r["iterations"],
        "cpu_baseline": {"value": value, "unit": "DOF-steps/s", "cores": ranks, "kind": "reference",
                         "sample": f"{steps} CN steps at C2 after 1 warm-up step, setup "
                                   f"{r['setup_seconds']:.1f}s excluded"},
        "e2e": {"value": value, "unit": "DOF-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_heat(args):
    import torch

    from paper_1609_04809_b200 import gmg
    from paper_1609_04809_b200.heat import HeatRun

    if int(os.environ.get("WORLD_SIZE", "1")) != 1:
        raise SystemExit("--workload heat runs on one GPU")
    clk = Clocks(0).start()
    torch.cuda.set_device(0)
    H = HEAT
    t0 = time.time()
    run = HeatRun(H["dim"], H["n_coarse"], H["levels"], H["dt"])
    setup_s = time.time() - t0
    cfg = gmg.MultigridConfig(smoother=gmg.SmootherConfig(kind=gmg.PF_SMOOTHER_JACOBI, damping=H["omega"]),
                              pre_smooth=H["pre"], post_smooth=H["post"], outer_tol=H["tol"])
    stream = torch.cuda.ExternalStream(run.h.stream_handle(), device=torch.device("cuda", 0))
    n_global = run.setups[0].n_global
    run.run(args.warmup, cfg)
    run.reset()
    torch.cuda.synchronize()
    n0 = run.h.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.time()
    e0.record(stream)
    st = run.run(args.steps, cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    clk.window(w0, time.time())
    ms = e0.elapsed_time(e1)
    launches = run.h.launch_count() - n0
    value = n_global * args.steps / (ms / 1e3)

    # e2e: u(0) and load(0) from pinned host memory, every step's solution back to the host
    u0 = torch.from_numpy(run.setups[0].x0.copy()).pin_memory().numpy()
    l0 = torch.from_numpy(run.setups[0].b.copy()).pin_memory().numpy()
    out = torch.empty(len(u0), dtype=torch.float64).pin_memory().numpy()
    torch.cuda.synchronize()
    e0.record(stream)
    run.u.upload(u0)
    run.load_now.upload(l0)
    run.t, run.step = 0.0, 0
    for _ in range(args.steps):
        run.run(1, cfg)
        run.u.download(0, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    clk.stop()

    # the time step's kernels besides the solve: load assembly and the fused CN rhs
    from paper_1609_04809_b200.heat import assemble_load, cn_rhs
    v, b = run.h.vector(), run.h.vector()
    s, has, g = run.setups[0].scales(H["dt"])
    for _ in range(3):
        assemble_load(run.load, s, v)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(20):
        assemble_load(run.load, s, v)
    e1.record(stream)
    torch.cuda.synchronize()
    load_us = e0.elapsed_time(e1) / 20 * 1e3
    e0.record(stream)
    for _ in range(20):
        cn_rhs(run.op, run.load, run.u, run.load_now, v, 0.5 * H["dt"], has, g, b)
    e1.record(stream)
    torch.cuda.synchronize()
    rhs_us = e0.elapsed_time(e1) / 20 * 1e3
    # fused CN rhs: algorithmic bytes = rhs operator values + columns (own + other rows,
    # SELL-stored) + u gather (once) + ln, lnx, is_dir, b
    nnz = int(run.setups[0].levels[-1].row_offsets[-1])
    n = len(u0)
    rhs_bytes = 12 * nnz + 8 * n + 8 * 3 * n + n
    # ... and the bytes the kernel streams: 4 B column + the stored value width (the rhs
    # operator M - dt/2 K of the constant-coefficient problem has few distinct values, so it
    # is index-encoded like the level operators: 1 or 2 B per entry)
    import numpy as np
    distinct = int(np.unique(np.asarray(run.setups[0].rhs_op)).size)
    vbytes = 1 if distinct <= 256 else 2 if distinct <= 65536 else 8
    rhs_stored = (4 + vbytes) * nnz + 8 * n + 8 * 3 * n + n
    peak, peak_src = peaks()
    achieved = rhs_stored / (rhs_us / 1e6) / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle import ref
            ranks = max(1, min(8, os.cpu_count() or 1))
            r = ref.heat_bench(3, 2, H["levels"], ranks, dt=H["dt"], warmup=0, steps=1)
            t = float(r["step_seconds"][0])
            cpu = {"value": n_global / t, "unit": "DOF-steps/s", "cores": ranks, "kind": "reference",
                   "sample": f"1 CN step at C2 ({r['iterations']} cycles) on {ranks} reference ranks; "
                             f"setup {r['setup_seconds']:.1f}s excluded", "step_seconds": t}
        except Exception as e:
            cpu = {"value": None, "unit": "DOF-steps/s", "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    line = {
        "metric": HEAT_METRIC, "value": value, "unit": "DOF-steps/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "manufactured heat problem of the reference, product setup",
        "config": dict(HEAT_CONFIG, parallelism="1 GPU"),
        "cycles_last_step": st.iterations,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None, "kernel": "k_cn_rhs (+ k_dirichlet): b = (M - dt/2 K) u + dt/2 (ln + lnx)",
                     "kernel_us": rhs_us, "bytes_per_launch": rhs_stored,
                     "bytes_formula": f"(4 + {vbytes}) z_all + 8 n (u) + 24 n (ln, lnx, b) + n (mask): the bytes the "
                                      f"kernel streams ({distinct} distinct operator values: {vbytes} B value index)"
                                      if vbytes < 8 else "12 z_all + 8 n + 24 n + n (fp64 values)",
                     "fp64_csr_equivalent": {"bytes_per_launch": rhs_bytes,
                                             "achieved": rhs_bytes / (rhs_us / 1e6) / 1e9,
                                             "note": "SURVEY.md 8(d) work-equivalent rate (12 B per entry), not "
                                                     "bytes moved"},
                     "peak_source": peak_src,
                     "note": "the solve's dominant kernel is k_jacobi as in the default workload"},
        "load_assembly_us": load_us,
        "cpu_baseline": cpu,
        "e2e": {"value": n_global * args.steps / (e2e_ms / 1e3), "unit": "DOF-steps/s",
                "h2d_bytes_per_step": 16 * n / args.steps, "d2h_bytes_per_step": 8 * n,
                "ms_per_step": e2e_ms / args.steps},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "setup_seconds": setup_s,
    }
    print(json.dumps(line), flush=True)
    run.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fe", action="store_true", help="skip the Q2 / rotated-Q1 variants")
    ap.add_argument("--no-c5", action="store_true", help="skip the one-GPU C5 (512^3) variant of the default run")
    ap.add_argument("--workload", choices=["poisson", "heat"], default="poisson",
                    help="poisson: BASELINE configs[1] (default); heat: the reference's CN run at C2")
    ap.add_argument("--config", choices=["c2", "c5"], default=None,
                    help="c2: BASELINE configs[1] (default on 1 GPU); c5: configs[4], 512^3 lognormal SOR "
                         "(default on N > 1 GPUs: the scaling configuration)")
    ap.add_argument("--transport", choices=["peer", "nccl"], default="peer",
                    help="multi-GPU exchanges: peer-memory stores (CUDA IPC/NVLink, default) or NCCL")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.config is None:
        args.config = "c2" if args.gpus == 1 else "c5"
    if args.workload == "heat":
        (run_reference_heat if args.impl == "reference" else run_b200_heat)(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.config == "c5":
        run_c5(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
