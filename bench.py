#!/usr/bin/env python
"""Benchmark of the B200 PCGM hot path (BASELINE.json metric: PCGM steps/s and achieved
HBM GB/s at K=N=256, T=200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

A "step" is one PCGM iteration (pcg.py:98-131): Delta-apply + curvature, x/r update +
||r||_inf, S x L nested-block-Jacobi sweeps + q.r, direction update.  Default workload is
BASELINE config 4 (mass-spring-damper 256 x 256 grid, T=200, n=2, m=1, S=L=2; seeded
synthetic data, no dataset involved).  Every vector is 210.8 MB, larger than the 126 MB
L2, so no L2 flush is needed between timed steps.

Multi-GPU (torchrun): by default N > 1 ranks run the stage-slab sharded solve of the ONE
problem (paper_2304_04980_b200/slab.py): one slab of stages per rank, halos
and the step's scalars over NCCL, value = steps of the global solve / max-over-ranks device
time ("strong" scaling).  --replicas runs N independent replicas of the one-context graph
solve instead ("weak"); N = 1 always runs the one-context graph solve.  (--slabs at N = 1
runs the sharded driver with a single slab.)  The slab solver (paper_2304_04980_b200/slab.py,
SURVEY.md 8(e)/(f)4): one slab per rank, halos and scalars over NCCL, value = steps of the
one global solve / max-over-ranks time ("strong" scaling).

--impl reference times the CPU restatement of the reference algorithm (oracle/, the
reference itself is pure Python + NumPy and cannot run at this size: SURVEY.md 6) on
the host cores for a bounded number of steps of the same workload.
"""

from __future__ import annotations

import argparse
import ctypes
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "PCGM steps/s"
UNIT = "steps/s"
CONFIG_NAMES = {1: "config1 random 4x4 T=20 n=2", 2: "config2 msd 16x16 T=50 n=2",
                3: "config3 random 64x64 T=100 n=4", 4: "config4 msd 256x256 T=200 n=2",
                5: "config5 random 32x1024 T=500 n=8"}


def c_factor(S, L):
    """canonical full-vector passes per step, C(S,L)."""
    return 10 + (3 * L - 1) + (S - 1) * (4 * L - 1)


def kernel_passes(name, S=2, L=2):
    """Algorithmic full-vector reads+writes of one launch of each step kernel."""
    if name == "delta":
        return 2                       # read d, write y (+ y.d)
    if name == "update":
        return 3                       # read r, y; write r (+ max|r|)
    if name == "update_x":
        return 3                       # read x, d; write x (parallel graph branch)
    if name == "dirupdate":
        return 3                       # read q, d; write d
    if name == "dirupdate_x":
        return 5                       # read q, d, x; write d, x (x update fused)
    if name == "dot":
        return 2
    if name.startswith("outer_rhs"):
        return 3                       # read delta, r; write r + Xi~ delta
    if name.startswith("sweep_s"):
        # read rhs, write the sweep output; + theta for inner sweeps; + r for the q.r dot
        # fused into the last sweep; + delta for the v1 path's on-the-fly Xi~ delta
        s_ = int(name[len("sweep_s"):].split("_")[0])
        l_ = int(name.split("_l")[1].split("_")[0])
        last = s_ == S - 1 and l_ == L - 1
        return (2 + (1 if l_ > 0 else 0) + (1 if last else 0) + (1 if name.endswith("_xi") else 0)
                + (2 if name.endswith("_r") else 0))   # _r: + read y, write r (r update fused)
    return 0


def kernel_flops(name, cnt, dim, S=2, L=2):
    """Algorithmic fp64 flops of one launch (2 x the reference's multiply counters,
    counts.py / SURVEY.md Appendix A; 2 flops per element for the CG vector kernels)."""
    if name == "delta":
        return 2.0 * cnt["matvec_flops"]
    if name.startswith("outer_rhs"):
        return 2.0 * cnt["outer_coupling_flops"]
    if name.startswith("sweep_s"):
        l_ = int(name.split("_l")[1].split("_")[0])
        f = 2.0 * cnt["pair_solve_flops"] + (2.0 * cnt["inner_coupling_flops"] if l_ > 0 else 0.0)
        s_ = int(name[len("sweep_s"):].split("_")[0])
        if s_ == S - 1 and l_ == L - 1:
            f += 2.0 * dim                    # q.r fused into the last sweep
        if name.endswith("_r"):
            f += 2.0 * dim                    # r -= alpha y fused into the first sweep
        return f
    if name in ("update", "update_x", "dirupdate", "dot"):
        return 2.0 * dim
    if name == "dirupdate_x":
        return 4.0 * dim
    return 0.0


def kernel_pipe(name):
    """fp64 pipe a kernel family runs on: DMMA (tensor, m8n8k4 f64) or DFMA."""
    return "dmma" if name.startswith("sweep_s") else "dfma"


def load_fp64_peaks():
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_peaks.json")) as fh:
            pk = json.load(fh)
        return {"dfma": float(pk["dfma_tflops"]), "dmma": float(pk["dmma_tflops"])}
    except Exception:
        return {"dfma": 34.0, "dmma": 36.8}


def kernel_family(name):
    """Step-kernel name -> the compiled kernel it launches (launches of one family share
    code and differ only in their operands)."""
    if name.startswith("sweep_s"):
        l_ = int(name.split("_l")[1].split("_")[0])
        if l_ > 0:
            return "pair-chain inner sweep (k_chainm / k_chain)"
        return ("pair-chain outer sweep + r update (k_chainm / k_chain)" if name.endswith("_r")
                else "pair-chain outer sweep (k_chain)")
    if name.startswith("outer_rhs"):
        return "outer rhs (k_rstep / k_grid)"
    if name == "delta":
        return "delta (k_dstep / k_grid)"
    return name


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(value, device, ws):
    """Replica timing: every rank times its own solve; the job's time is the slowest rank
    (device-timed values reduced with MAX over the process group)."""
    if ws <= 1:
        return float(value)
    import torch
    import torch.distributed as dist

    t = torch.tensor([float(value)], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def traffic_from_profiles(kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            data = json.load(fh)
        return data.get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------------------


def run_ours(args, ws, rank, local):
    import torch
    import torch.distributed as dist

    from paper_2304_04980_b200 import (GpuNestedJacobiPreconditioner, GpuSchurOperator,
                                       MaxIterationsExceeded, _lib, generators, pcg_solve)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    S, L = args.S, args.L
    ga = generators.CONFIGS[args.config](args.seed)
    t0 = time.perf_counter()
    op = GpuSchurOperator(ga, L, S)
    pc = GpuNestedJacobiPreconditioner(op, L, S)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ctx = op._ctx
    lib = ctx.lib
    stream = torch.cuda.Stream(device=dev)
    _lib.check(lib.gq_set_stream(ctx.h, ctypes.c_void_p(stream.cuda_stream)))
    rhs = torch.tensor(ga.offset, device=dev, dtype=torch.float64)
    tol = 1e-300            # fixed-step run (BASELINE config 4: fixed 100 steps)
    steps = ctypes.c_int64()
    conv = ctypes.c_int32()
    _lib.check(lib.gq_pcg_start(ctx.h, ctypes.c_void_p(rhs.data_ptr()), None, 1))
    W, K = args.warmup, args.steps
    rc = lib.gq_pcg_run(ctx.h, tol, W, ctypes.byref(steps), ctypes.byref(conv))
    assert rc in (_lib.GQ_OK, _lib.GQ_MAX_ITER), _lib.last_error()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        rc = lib.gq_pcg_run(ctx.h, tol, W + K, ctypes.byref(steps), ctypes.byref(conv))
        e1.record(stream)
        torch.cuda.synchronize()
    assert rc in (_lib.GQ_OK, _lib.GQ_MAX_ITER), _lib.last_error()
    assert steps.value == W + K, (steps.value, W + K)
    ms = max_over_ranks(e0.elapsed_time(e1), dev, ws)
    if ws > 1:
        dist.barrier()
    hist = np.empty(W + K)
    _lib.check(lib.gq_pcg_history(ctx.h, hist.ctypes.data, W + K))

    # per-kernel device times (CUDA events on the launch stream, individual launches)
    nk = lib.gq_launches_per_step(ctx.h)
    prof_steps = 3
    buf = (ctypes.c_float * nk)()
    got = lib.gq_profile_steps(ctx.h, prof_steps, buf, nk)
    assert got == nk, _lib.last_error()
    names = [lib.gq_kernel_name(ctx.h, i).decode() for i in range(nk)]
    kms = {nm: buf[i] / prof_steps for i, nm in enumerate(names)}
    dim = op.dim
    vec_bytes = 8 * dim
    peak, peak_src = load_peaks()
    fp64_peaks = load_fp64_peaks()
    from paper_2304_04980_b200.counts import counters
    cnt = counters(ga, L, S)
    # dominant kernel = the kernel (one compiled kernel, possibly several launches per step)
    # with the largest total device time per step; its roofline uses the per-launch averages
    fams = {}
    for nm, t in kms.items():
        fams.setdefault(kernel_family(nm), []).append(nm)
    top_fam = max(fams, key=lambda f: sum(kms[n] for n in fams[f]))
    members = fams[top_fam]
    top = top_fam + " (" + ", ".join(members) + ")"
    top_bytes = sum(kernel_passes(n, S, L) for n in members) * vec_bytes / len(members)
    top_ms = sum(kms[n] for n in members) / len(members)
    achieved = top_bytes / (top_ms * 1e-3) / 1e9
    trs = [traffic_from_profiles(n) for n in members]
    top_traffic = sum(trs) / len(trs) if all(t is not None for t in trs) else None
    step_bytes = 8 * dim * c_factor(S, L)
    step_ms = ms / K
    step_gbs = step_bytes / (step_ms * 1e-3) / 1e9
    total_ms = sum(kms.values())

    # end to end through the public API with host buffers (H2D rhs, D2H x + history)
    rhs_host = torch.from_numpy(ga.offset.copy()).pin_memory().numpy()
    try:        # warm-up solve of W steps through the same path (not timed)
        pcg_solve(op, pc, rhs_host, tol=tol, max_steps=max(W, 1))
    except MaxIterationsExceeded:
        pass
    gc.collect()    # the warm-up's result is gone: its page-locked buffer is back in the pool
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        pcg_solve(op, pc, rhs_host, tol=tol, max_steps=K)
        raise RuntimeError("unexpected convergence in a fixed-step run")
    except MaxIterationsExceeded as exc:
        x_out = exc.iterate
    e2e_s = time.perf_counter() - t0
    assert x_out.shape == (dim,)
    e2e_s = max_over_ranks(e2e_s, dev, ws)

    line = {
        "metric": METRIC,
        "value": K * ws / (ms * 1e-3),
        "unit": UNIT,
        "n_gpus": ws,
        "steps": K,
        "warmup": W,
        "ms_per_step": ms / K,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, no dataset)",
        "config": workload_config(args, ga, S, L, f"replicas x{ws}" if ws > 1 else "single GPU"),
        "run": {"setup_s": round(setup_s, 3),
                "layout": "stage-inner, stage stride padded to a multiple of 8 (128-byte records)"},
        "roofline": {
            "bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak,
            "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak,
            "traffic": top_traffic,
            "algorithmic_bytes_per_launch": top_bytes, "launches_per_step": len(members),
            "ms_per_launch": top_ms,
            "fp64_tflops": sum(kernel_flops(n, cnt, dim, S, L) for n in members) / len(members)
                           / (top_ms * 1e-3) / 1e12,
            "fp64_peak_tflops": fp64_peaks[kernel_pipe(members[0])],
            "fp64_frac": sum(kernel_flops(n, cnt, dim, S, L) for n in members) / len(members)
                         / (top_ms * 1e-3) / 1e12 / fp64_peaks[kernel_pipe(members[0])],
        },
        "step_roofline": {
            "bytes_per_step": step_bytes, "C(S,L)": c_factor(S, L), "achieved": step_gbs,
            "peak": peak, "unit": "GB/s", "frac": step_gbs / peak,
            "model": "SURVEY.md 8(d): 8*dim*C(S,L) canonical full-vector traffic",
            "fp64_flops_per_step": 2.0 * (cnt["matvec_flops"] + cnt["apply_flops"]) + 12.0 * dim,
            "fp64_tflops": (2.0 * (cnt["matvec_flops"] + cnt["apply_flops"]) + 12.0 * dim)
                           / (step_ms * 1e-3) / 1e12,
        },
        "kernel_ms": {k: round(v, 4) for k, v in kms.items()},
        # per kernel: HBM GB/s and fraction (algorithmic passes), fp64 TF/s and fraction of
        # the measured pipe peak (algorithmic flops; profiles/fp64_peaks.json)
        "kernel_roofline": {
            k: {"gbs": round(kernel_passes(k, S, L) * vec_bytes / (v * 1e-3) / 1e9, 1),
                "hbm_frac": round(kernel_passes(k, S, L) * vec_bytes / (v * 1e-3) / 1e9 / peak, 3),
                "tflops": round(kernel_flops(k, cnt, dim, S, L) / (v * 1e-3) / 1e12, 2),
                "fp64_pipe": kernel_pipe(k),
                "fp64_frac": round(kernel_flops(k, cnt, dim, S, L) / (v * 1e-3) / 1e12
                                   / fp64_peaks[kernel_pipe(k)], 3)}
            for k, v in kms.items()},
        "kernel_share": {k: round(v / total_ms, 4) for k, v in kms.items()},
        "gpu_launches": K * nk,
        "residual_inf": [float(hist[0]), float(hist[-1])],
        "e2e": {
            "value": K * ws / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": vec_bytes / K, "d2h_bytes_per_step": (vec_bytes + 8 * K) / K,
            "includes": "pcg_solve() on host numpy rhs: H2D rhs + layout transpose, "
                        "initial preconditioner apply, K steps, D2H x + history",
        },
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, ga)
    return line


def run_slabs(args, ws, rank, local):
    """Stage-slab sharded PCGM: one slab per rank, native stage-slab phases (slab.py)."""
    import torch

    from paper_2304_04980_b200 import MaxIterationsExceeded, generators
    from paper_2304_04980_b200.slab import SlabComm, SlabPcg

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ga = generators.CONFIGS[args.config](args.seed)
    t0 = time.perf_counter()
    solver = SlabPcg(ga, inner_sweeps=args.L, outer_sweeps=args.S,
                     comm=SlabComm.from_env(ws, device=dev))
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    rhs = torch.tensor(ga.offset, device=dev, dtype=torch.float64)
    W, K = args.warmup, args.steps

    def run(steps):
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()
        try:
            solver.solve(rhs, tol=1e-300, max_steps=steps)
        except MaxIterationsExceeded:
            pass
        torch.cuda.synchronize()

    run(W + 2)                   # captures the step graph (one slab per process: eager)
    solver.time_from = W         # CUDA events around steps W .. W+K-1 of the next solve
    with ClockSampler(local) as clk:
        run(W + K)
    solver.time_from = None
    k_timed, ms = solver.last_timed
    assert k_timed == K, (k_timed, K)
    ms = max_over_ranks(ms, dev, ws)
    sl = solver.slabs
    # per-rank communication time of a step (halo exchanges + scalar collectives), from CUDA
    # events around each of them in a few extra eager steps (not part of the timed region)
    comm_ms = None
    if ws > 1:
        solver.comm_events = []
        graph_was, solver.graph = solver.graph, False
        run(3)
        solver.graph = graph_was
        torch.cuda.synchronize()
        evs, solver.comm_events = solver.comm_events, None
        mine = sum(e0.elapsed_time(e1) for e0, e1 in evs) / 3.0
        import torch.distributed as dist

        allc = [None] * ws
        dist.all_gather_object(allc, mine)
        comm_ms = [round(float(c), 4) for c in allc]

    # end to end through the public API: host numpy rhs in, host x out (gathered), K steps
    rhs_host = torch.from_numpy(ga.offset.copy()).pin_memory().numpy()
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    try:
        solver.solve(rhs_host, tol=1e-300, max_steps=K)
    except MaxIterationsExceeded as exc:
        assert exc.iterate.shape == (ga.dim,)
    e2e_s = max_over_ranks(time.perf_counter() - t0, dev, ws)

    # kernels of ours per step and slab: the step kernels of the one-context graph, the three
    # scalar fix-ups the slab phases enqueue (k_slab_alpha in UPDATE, k_slab_savemu in the
    # last OUTER, k_slab_conv_beta in DIRECTION: gq_slab_phase), and a pack + unpack per halo
    # stage per exchange (S exchanges per step)
    lib = solver.nat[solver.comm.local[0]].ctx.lib
    per_slab = lib.gq_launches_per_step(solver.nat[solver.comm.local[0]].ctx.h) + 3
    halos = sum((x.lo > 0) + (x.hi < ga.T + 1) for x in sl) / len(sl)
    launches = int(round(K * (per_slab + 2 * halos * args.S)))
    return {
        "metric": METRIC, "value": K / (ms * 1e-3), "unit": UNIT, "n_gpus": ws, "steps": K,
        "warmup": W, "ms_per_step": ms / K, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, no dataset)",
        "config": workload_config(args, ga, args.S, args.L, parallelism_label(args, ws)),
        "run": {"comm_ms_per_step_by_rank": comm_ms,
                "slabs": [[x.lo, x.hi] for x in sl], "setup_s": round(setup_s, 3),
                "timing": "CUDA events on the solver stream around steps W..W+K-1 of one solve"},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "e2e": {
            "value": K / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": 8 * ga.dim / K, "d2h_bytes_per_step": 8 * ga.dim / K,
            "includes": "SlabPcg.solve on host numpy rhs: H2D + scatter, slab start and "
                        "initial preconditioner, K steps, gather + D2H of x",
        },
    }


def _oracle_steps(ga, S, L, steps, threads, budget_s=None):
    """Time PCGM steps of the C oracle (oracle/gridlq_oracle.c, restating pcg.py's loop);
    setup and the initial preconditioner apply are excluded.  Returns (seconds per
    step, setup seconds, steps timed, threads)."""
    from oracle.coracle import COracle
    from oracle.gridlq_oracle import Oracle

    t0 = time.perf_counter()
    orc = COracle(Oracle(ga, L, S), threads=threads)
    setup = time.perf_counter() - t0
    if budget_s is not None:
        # one probe step, then as many as fit in the budget (at least 2, at most `steps`)
        _, _, _, _, _, secs = orc.pcg(ga.offset, tol=1e-300, max_steps=2)
        per = secs[1] - secs[0]
        steps = int(max(2, min(steps, budget_s / max(per, 1e-9))))
    _, _, k, _, _, secs = orc.pcg(ga.offset, tol=1e-300, max_steps=max(2, steps))
    per_step = (secs[k - 1] - secs[0]) / (k - 1)
    return per_step, setup, k - 1, orc.threads


def reference_python_leg(steps=8):
    """The unmodified reference package (baseline/_ref, pure Python + NumPy) timed on this
    host at a size it can hold: BASELINE config 2 (MSD 16x16, T=50, S=L=2), its own pcg_solve
    with pool=None and with its --threads executor (cli.py:285).  The headline size is out of
    its reach (>100 GB, hours of setup: SURVEY.md 6).  None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gridlq")):
        return None
    from concurrent.futures import ThreadPoolExecutor

    from paper_2304_04980_b200 import generators
    from paper_2304_04980_b200.problem import arrays_to_problem

    sys.path.insert(0, ref)
    try:
        import gridlq
    finally:
        sys.path.remove(ref)
    ga = generators.config2(0)
    t0 = time.perf_counter()
    st = gridlq.build_stacked(arrays_to_problem(ga))
    sc = gridlq.build_schur(st)
    pc = gridlq.NestedJacobiPreconditioner(sc, inner_sweeps=2, outer_sweeps=2)
    setup = time.perf_counter() - t0
    out = {"workload": "config2 msd 16x16 T=50 n=2, S=L=2", "dim": int(sc.dim),
           "setup_s": round(setup, 2), "steps": steps, "unit": UNIT}
    threads = os.cpu_count() or 1
    for key, pool in (("pool_none", None), (f"threads_{threads}", ThreadPoolExecutor(threads))):
        stamps = []
        try:
            gridlq.pcg_solve(sc, pc, st.offset, tol=1e-300, max_steps=steps, pool=pool,
                             callback=lambda k, x, r: stamps.append(time.perf_counter()))
        except gridlq.MaxIterationsExceeded:
            pass
        if pool is not None:
            pool.shutdown()
        out[key] = (len(stamps) - 1) / (stamps[-1] - stamps[0])
    return out


def cpu_baseline(args, ga):
    per_step, setup, k, th = _oracle_steps(ga, args.S, args.L, args.cpu_steps + 1, 1)
    line = {
        "value": 1.0 / per_step, "unit": UNIT, "cores": th, "kind": "port",
        "sample": f"{k} PCGM step(s) of the same workload with the C restatement of the "
                  f"reference loop (oracle/gridlq_oracle.c), 1 thread; setup {setup:.1f}s "
                  "and the initial preconditioner apply excluded",
        "host_cpus": os.cpu_count(),
    }
    try:
        ref = reference_python_leg()
    except Exception as exc:   # the reference leg is informational; never fail the bench on it
        ref = {"error": str(exc)[:200]}
    if ref is not None:
        line["reference_python"] = ref
    return line


def workload_config(args, ga, S, L, parallelism):
    """The `config` object every arm prints for one workload (identical across the product and
    reference arms, so the driver's config comparison sees the same keys and values)."""
    return {"workload": CONFIG_NAMES.get(args.config, str(args.config)),
            "K": ga.K, "N": ga.N, "T": ga.T, "n": ga.n, "m": ga.m,
            "outer_sweeps_S": S, "inner_sweeps_L": L, "dim": ga.dim,
            "parallelism": parallelism,
            "l2": ("inputs larger than L2 (one vector = %.1f MB)" % (8 * ga.dim / 1e6)
                   if 8 * ga.dim > 126e6 else
                   "working set of %.1f MB per vector fits in L2: launch/latency-bound "
                   "configuration, not an HBM measurement" % (8 * ga.dim / 1e6))}


def parallelism_label(args, ws):
    if ws == 1:
        return "single GPU"
    return f"replicas x{ws}" if getattr(args, "replicas", False) else f"stage slabs x{ws}"


def run_reference(args, ws, rank):
    from paper_2304_04980_b200 import generators

    ga = generators.CONFIGS[args.config](args.seed)
    threads = os.cpu_count() or 1
    per_step, setup, k, th = _oracle_steps(ga, args.S, args.L, args.steps + 1, threads,
                                           budget_s=args.ref_budget_s)
    value = 1.0 / per_step
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator, no dataset)", "impl": "reference",
        "config": workload_config(args, ga, args.S, args.L, parallelism_label(args, ws)),
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": th, "kind": "port",
            "sample": f"{k} of {args.steps} PCGM steps of the same workload, C/OpenMP "
                      "restatement of the reference loop (oracle/gridlq_oracle.c; the "
                      "reference itself is pure Python/NumPy, ~530 s/step here per "
                      f"SURVEY.md 6); setup {setup:.1f}s excluded",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--S", type=int, default=None)
    ap.add_argument("--L", type=int, default=None)
    ap.add_argument("--cpu-steps", type=int, default=1)
    ap.add_argument("--ref-budget-s", type=float, default=90.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--slabs", action="store_true",
                    help="stage-slab sharded solve, one slab per rank (strong scaling; the "
                         "default for N > 1)")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: independent replicas of the one-context solve (weak scaling)")
    args = ap.parse_args()
    if args.S is None:
        args.S = 3 if args.config == 3 else 2
    if args.L is None:
        args.L = 2
    ws, rank, local = dist_env()
    if args.impl == "reference":
        if rank != 0:
            return
        print(json.dumps(run_reference(args, ws, rank)), flush=True)
        return
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    try:
        slabs = args.slabs or (ws > 1 and not args.replicas)
        line = (run_slabs if slabs else run_ours)(args, ws, rank, local)
        if rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        if ws > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
