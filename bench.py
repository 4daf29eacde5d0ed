#!/usr/bin/env python
"""Benchmark of the CG hot path of arXiv 1505.07630 on B200 (BASELINE.json metric:
"CG iter/s & effective HBM GB/s, 256^3 Poisson LDU, at 1/2/4/8 B200").

One step = one ``pcg_solve`` (or ``pipecg_solve``) of ``--iters`` fixed iterations (tol = 0) on
the resident config-3 system: laplacianFoam 3-D 256^3 Poisson, FV Dirichlet walls, hot-face
RHS, x0 = 0.  With N ranks the same global system is split into N contiguous z-slabs (halo
exchange + reductions over NVLink), so the work is fixed as N grows ("strong").  value = global
CG iterations per second (max over ranks of the device time).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--solver pcg|pipecg] [--impl reference]

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")  # keep NCCL's version banner off stdout (one JSON line)

METRIC = "CG iter/s & effective HBM GB/s, 256³ Poisson LDU, at 1/2/4/8 B200"
UNIT = "iter/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--solver", default="pipecg", choices=["pcg", "pipecg"],
                   help="headline solver; the other one is measured too (key 'secondary')")
    p.add_argument("--no-secondary", action="store_true")
    p.add_argument("--cube", "--n", dest="n", type=int, default=256,
                   help="mesh is n^3 (config 3: 256; config 4: 512)")
    p.add_argument("--iters", type=int, default=200, help="fixed CG iterations per step")
    p.add_argument("--batch", type=int, default=0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-profile", action="store_true", help="skip per-pass event timing")
    p.add_argument("--no-amg", action="store_true", help="skip the AMG-PCG time-to-solution leg")
    p.add_argument("--amg-tol", type=float, default=1e-8)
    p.add_argument("--no-c5", action="store_true",
                   help="skip the c5 irregular (SELL-32) evidence leg")
    p.add_argument("--c5-n", type=int, default=184,
                   help="c5 leg: irregular mesh base n^3 (184^3 = 6.2M cells: one GPU's share of "
                        "config 5's 50M cells on 8 GPUs)")
    return p.parse_args()


# ------------------------------------------------------------------------------------------
# byte model
# ------------------------------------------------------------------------------------------
def model_bytes(solver, N, F, P):
    """Algorithmic bytes per iteration, LDU model: fp64 values, int32 addressing."""
    if solver == "pcg":
        return 88 * N + 16 * F + 28 * P
    return 136 * N + 16 * F + 28 * P


def pass_model_bytes(solver, N, F, fused=False):
    """Dominant kernel per launch, §8(d): classical pass A = 56N + 16F; pipelined pass U = 112N
    (single rank: S and U fused into one pass = the whole iteration, 136N + 16F)."""
    if solver == "pcg":
        return 56 * N + 16 * F
    return 136 * N + 16 * F if fused else 112 * N


def pass_format_bytes(solver, info, N):
    """Bytes the dominant kernel(s) must move in the layout actually streamed.
    Classical pass A with variant 7 is two kernels: A1 (r, rD, p_old, x in; p, x out: 48N) and
    A2 (p, rD, coefficients in; q out)."""
    if solver == "pipecg":
        if not info.get("pipeFused"):
            return 112 * N
        if info["layout_name"] == "DIA_SYM":  # w, rD, z, s, r, p, x, U_k in; z, s, p, x, r, w out
            return (13 + info["nDiagonals"]) * 8 * N
        return 104 * N + 12 * info["storedEntries"] + 12 * ((N + 31) // 32)
    split = info.get("variant") == 7
    if info["layout_name"] == "DIA_SYM":
        if split:
            return 48 * N + (24 + 8 * info["nDiagonals"]) * N
        return 56 * N + 8 * info["nDiagonals"] * N  # r, rD, p_old, x in; p, q, x out; U_k once
    base = 48 * N + 24 * N if split else 56 * N
    return base + 12 * info["storedEntries"] + 12 * ((N + 31) // 32)


def iter_format_bytes(solver, info, N, P):
    """Bytes one iteration must move in the layout and pass structure actually run: the fused
    pipelined pass alone; classical = pass A (A1 + A2) + pass B (r, q, rD in; r out: 32N);
    plus the halo (faceCells 4 + coeffs 8 + send 8 + recv 8 per interface face)."""
    b = pass_format_bytes(solver, info, N)
    if solver == "pcg":
        b += 32 * N
    elif not info.get("pipeFused"):
        b += 24 * N + 8 * (info["nDiagonals"] if info["layout_name"] == "DIA_SYM" else 0) * N
    return b + 28 * P


def host_cpu():
    """The host the CPU oracle runs on (record nproc and the lscpu model)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"model": model, "nproc": os.cpu_count()}


def pinned_to_one_core(fn):
    """Run fn with this process pinned to one core (the `taskset -c <core>` of SURVEY §8(d))."""
    try:
        old = os.sched_getaffinity(0)
        core = min(old)
        os.sched_setaffinity(0, {core})
    except Exception:
        old, core = None, None
    try:
        return fn(), core
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)


def vcycle_bytes(amg, info):
    """Bytes one V-cycle must move in the layouts it streams: level 0 on the
    handle's DIA layout (nd coefficient arrays), coarser levels and every P / R as CSR (12 B per
    entry + 4 B row pointer), each vector touched once per kernel, the coarsest dense inverse."""
    n, nA, nP, L = amg["n"], amg["nnzA"], amg["nnzP"], amg["nLevels"]
    tot = 0
    for l in range(L):
        N, Nc = n[l], n[l + 1]
        if l == 0 and info["layout_name"] == "DIA_SYM":
            a = 8 * info["nDiagonals"] * N + 8 * N        # U_k and diag
        else:
            a = 12 * nA[l] + 4 * N
        tot += a + 8 * N + 16 * N                         # K1: A, x_pre (gathered), f in, r out
        tot += 12 * nP[l] + 4 * Nc + 8 * N + 16 * Nc      # K2: R, r in; f_c, x_pre,c out
        tot += 12 * nP[l] + 4 * N + 8 * Nc + (24 if l == 0 else 16) * N  # K3: P, x_c (+ rD, f) in; x
        tot += a + 8 * N + 24 * N                         # K4: A, x, f, rD in; z out
    nc = amg["coarsestN"]
    return tot + 8 * nc * nc + 16 * nc


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(solver, n, world):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed `ncu --set full` capture summary (profiles/ncu_traffic.json), if it matches."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(f"{solver}_n{n}_p{world}")
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


# ------------------------------------------------------------------------------------------
# clocks during the timed region
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
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
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------------
# CPU oracle baseline (tests/bench only may call oracle/)
# ------------------------------------------------------------------------------------------
def oracle_iter_rate(sys_, b, solver, k1, k2):
    """Oracle per-iteration time from fixed-iteration runs (t(k2) - t(k1)) / (k2 - k1)."""
    import oracle
    fn = oracle.pcg if solver == "pcg" else oracle.pipecg
    ts = []
    for k in (k1, k2):
        t0 = time.perf_counter()
        fn(sys_, b, tol=0.0, maxIter=k)
        ts.append(time.perf_counter() - t0)
    per = (ts[1] - ts[0]) / (k2 - k1)
    return 1.0 / per, per


def build_global(n):
    import meshgen
    sys_ = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
    return sys_, sys_.b


def config_dict(args, world, info=None):
    d = {"workload": f"c3: laplacianFoam 3-D {args.n}^3 Poisson ({args.n ** 3:,} cells), FV "
                     f"Dirichlet walls, hot-face RHS, x0 = 0, {'Jacobi-PCG' if args.solver == 'pcg' else 'pipelined CG (Ghysels-Vanroose, Jacobi)'}, "
                     f"{args.iters} fixed iterations per step (tol = 0)",
         "cells": args.n ** 3, "solver": args.solver, "iters_per_step": args.iters,
         "decomposition": f"{world} contiguous z-slab(s)",
         "l2": "inputs larger than L2 (working set >= 1.9 GB vs 126 MB L2); no flush needed"}
    if info is not None:
        d["layout"] = info["layout_name"]
    return d


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle as it stands
# ------------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    sys_, b = build_global(args.n)
    fn = oracle.pcg if args.solver == "pcg" else oracle.pipecg
    k = 2  # bounded sample per step: 2 oracle iterations of the same 256^3 workload
    for _ in range(args.warmup):
        fn(sys_, b, tol=0.0, maxIter=k)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn(sys_, b, tol=0.0, maxIter=k)
    dt = time.perf_counter() - t0
    value = args.steps * k / dt
    sample = (f"each step = oracle {args.solver} (C, fp64, 1 thread) for {k} iterations on the "
              f"full {args.n}^3 system incl. r0 setup")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": config_dict(args, 1),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch

    import meshgen
    import paper_1505_07630_b200 as ldu

    # LDU_DIST_BOOT=host: gloo + ldu_comm_init_host (no NCCL; ranks may share GPUs -- used to
    # exercise more ranks than the box has GPUs; timings are then not a scaling measurement)
    host_boot = os.environ.get("LDU_DIST_BOOT", "nccl") == "host" and world > 1
    if host_boot:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    comm = None
    if world > 1:
        import torch.distributed as dist
        if host_boot:
            dist.init_process_group("gloo")
            comm = ldu.Comm.host(rank, world, local)
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            uid = [ldu.Comm.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = ldu.Comm(rank, world, uid[0], local)

    n = args.n
    if world == 1:
        sys_ = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
    else:
        sys_ = meshgen.hex_laplacian_slab(n, n, n, world, rank, dirichlet=dict(x0=1.0))
    N, F = sys_.nCells, sys_.nFaces
    P = sum(len(i.faceCells) for i in sys_.interfaces)
    A = ldu.LduMatrix.from_system(sys_, comm)
    info = A.info()
    stream = torch.cuda.current_stream()
    A.set_stream(stream.cuda_stream)
    b = torch.from_numpy(sys_.b).cuda()
    x = torch.zeros_like(b)
    kw = dict(tol=0.0, maxIter=args.iters, batch=args.batch)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce_(t, op=None):
        """in-place all-reduce of a small CUDA tensor (through the host under gloo)"""
        kw = {} if op is None else {"op": op}
        if host_boot:
            c = t.cpu()
            dist.all_reduce(c, **kw)
            t.copy_(c)
        else:
            dist.all_reduce(t, **kw)

    # global byte model
    tot = torch.tensor([N, F, P], dtype=torch.float64, device="cuda")
    if dist is not None:
        allreduce_(tot)
    Ng, Fg, Pg = (float(v) for v in tot.tolist())
    peak, peak_src = hbm_peak()
    # the paper's STREAM-measured roofline: our fp64 triad, same run, same device
    triad = ldu.stream_triad(local, 1 << 28, 5)

    def timed(solver, sample_clocks):
        """W warm-up solves, then K timed solves bracketed by barrier + synchronize; device time
        by CUDA events on the caller's stream, max over ranks.  The headline value comes from a
        region without per-pass event nodes; a second timed region of K solves with the event
        nodes (profile) gives the dominant kernel's live per-launch time for the roofline."""
        fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
        for _ in range(max(3, args.warmup)):
            x.zero_()
            fn(b, x, **kw)
        barrier()
        prof = {"pass_ms": 0.0, "pass_n": 0, "elapsed": None}
        if not args.no_profile:
            slot = 0 if solver == "pcg" else 1
            p0 = torch.cuda.Event(enable_timing=True)
            p1 = torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            for _ in range(args.steps):
                x.zero_()
                fn(b, x, profile=True, **kw)
                s = A.stats()
                prof["pass_ms"] += s["passMs"][slot]
                prof["pass_n"] += s["passLaunches"][slot]
            p1.record(stream)
            barrier()
            prof["elapsed"] = p0.elapsed_time(p1) / 1e3
        clocks = ClockSampler(local) if sample_clocks else None
        if clocks:
            clocks.start()
            time.sleep(0.3)
        kernels = 0
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            x.zero_()
            st, it, res = fn(b, x, **kw)
            s = A.stats()
            kernels += s["kernels"]
        e1.record(stream)
        barrier()
        elapsed = e0.elapsed_time(e1) / 1e3
        clk = clocks.stop() if clocks else None
        t = torch.tensor([elapsed], dtype=torch.float64, device="cuda")
        if dist is not None:
            allreduce_(t, dist.ReduceOp.MAX)
        elapsed = float(t.item())
        value = args.steps * args.iters / elapsed
        # roofline of the dominant kernel (this rank), timed live with CUDA event nodes
        roof = None
        pass_ms, pass_n = prof["pass_ms"], prof["pass_n"]
        if pass_n:
            t_launch = pass_ms / pass_n / 1e3
            fused = bool(info.get("pipeFused")) and solver == "pipecg"
            mb = pass_model_bytes(solver, N, F, fused)
            fb = pass_format_bytes(solver, info, N)
            kname = ("k_cg_passA1+k_cg_passA2" if info.get("variant") == 7 else "k_cg_passA")
            # achieved / frac: the bytes the layout must move per launch over the
            # live launch time; the §8(d) LDU-model figure is reported only as the labelled
            # "model-equivalent" rate (it counts int32 addressing and unfused passes the DIA
            # layout and the fused pass never move, so it can exceed the copy peak)
            pk = ("k_pipe_SU_mr" if world > 1 else "k_pipe_SU") if fused else "k_pipe_U"
            roof = {"kernel": kname if solver == "pcg" else pk,
                    "bound": "hbm", "achieved": fb / t_launch / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": fb / t_launch / 1e9 / peak, "traffic": ncu_traffic(solver, n, world),
                    "bytes_per_launch": fb, "launch_us": t_launch * 1e6,
                    "triad_frac": (fb / t_launch / 1e9 / triad) if triad else None,
                    "model_bytes_per_launch": mb,
                    "model_equivalent_gbps": mb / t_launch / 1e9, "peak_source": peak_src,
                    "share_of_step": pass_ms / 1e3 / prof["elapsed"],
                    "timed_with_event_nodes_ms_per_step": 1e3 * prof["elapsed"] / args.steps}
        bytes_iter = model_bytes(solver, Ng, Fg, Pg)
        fb_iter = torch.tensor([float(iter_format_bytes(solver, info, N, P))], dtype=torch.float64,
                               device="cuda")
        if dist is not None:
            allreduce_(fb_iter)
        fb_iter = float(fb_iter.item())
        return dict(value=value, elapsed=elapsed, kernels=kernels, roof=roof, clk=clk,
                    status=int(st), iters=it, bytes_iter=bytes_iter, fb_iter=fb_iter,
                    eff=value * fb_iter / 1e9, model_eff=value * bytes_iter / 1e9)

    main_r = timed(args.solver, True)
    value, elapsed, kernels = main_r["value"], main_r["elapsed"], main_r["kernels"]
    roof, clk, bytes_iter = main_r["roof"], main_r["clk"], main_r["bytes_iter"]
    st, it = main_r["status"], main_r["iters"]
    secondary = None
    if not args.no_secondary:
        other = "pcg" if args.solver == "pipecg" else "pipecg"
        r2 = timed(other, False)
        secondary = {"solver": other, "value": r2["value"], "unit": UNIT,
                     "ms_per_step": 1e3 * r2["elapsed"] / args.steps,
                     "effective_gbps": r2["eff"], "bytes_per_iter": r2["fb_iter"],
                     "effective_frac_of_hbm": r2["eff"] / (peak * world),
                     "model_bytes_per_iter": r2["bytes_iter"],
                     "model_equivalent_gbps": r2["model_eff"], "roofline": r2["roof"]}
    solve = A.pcg_solve if args.solver == "pcg" else A.pipecg_solve

    # end to end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        bh = torch.from_numpy(sys_.b).pin_memory()
        xh = torch.zeros(N, dtype=torch.float64).pin_memory()
        for _ in range(2):
            xh.zero_()
            solve(bh, xh, **kw)
        # one pre-zeroed pinned x0 per timed step: the user's input preparation (a host memset of
        # the 134 MB x0) stays outside the timed region, the H2D / solve / D2H of every call inside
        ne = min(args.steps, 16)
        xs = [torch.zeros(N, dtype=torch.float64).pin_memory() for _ in range(ne)]
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        h2d = d2h = 0
        for i in range(ne):
            solve(bh, xs[i], **kw)
            s = A.stats()
            h2d += s["h2dBytes"]
            d2h += s["d2hBytes"]
        f1.record(stream)
        barrier()
        te = torch.tensor([f0.elapsed_time(f1) / 1e3], dtype=torch.float64, device="cuda")
        if dist is not None:
            allreduce_(te, dist.ReduceOp.MAX)
        e2e = {"value": ne * args.iters / float(te.item()), "unit": UNIT,
               "h2d_bytes_per_step": h2d // ne, "d2h_bytes_per_step": d2h // ne, "steps": ne}
        del xs

    # AMG-PCG (NEXT-2): time to solution at --amg-tol vs Jacobi-PCG on the same system
    amg = None
    if world == 1 and not args.no_amg:
        ai = A.amg_setup()
        setup_cold = ai["setupMs"]
        warm = []  # again: the first build in a process also pays the allocator's first touch;
        for _ in range(3):  # the median of 3 warm builds (allocator latency varies box to box)
            ai = A.amg_setup()
            warm.append(ai["setupMs"])
        setup_warm = sorted(warm)[1]
        tol = args.amg_tol
        for _ in range(2):
            x.zero_()
            A.amg_pcg_solve(b, x, tol=tol, maxIter=1000)
        barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        akern = 0
        for _ in range(args.steps):
            x.zero_()
            ast, ait, ares = A.amg_pcg_solve(b, x, tol=tol, maxIter=1000)
            akern += A.stats()["kernels"]
        a1.record(stream)
        barrier()
        t_amg = a0.elapsed_time(a1) / 1e3 / args.steps
        x.zero_()
        A.amg_pcg_solve(b, x, tol=tol, maxIter=1000, profile=True)
        ps = A.stats()
        vc_ms = ps["passMs"][0] / max(1, ps["passLaunches"][0])
        kr_ms = ps["passMs"][1] / max(1, ps["passLaunches"][1])
        x.zero_()
        A.pcg_solve(b, x, tol=tol, maxIter=20000)
        barrier()
        j0 = torch.cuda.Event(enable_timing=True)
        j1 = torch.cuda.Event(enable_timing=True)
        j0.record(stream)
        x.zero_()
        jst, jit, jres = A.pcg_solve(b, x, tol=tol, maxIter=20000)
        j1.record(stream)
        barrier()
        t_jac = j0.elapsed_time(j1) / 1e3
        vb = vcycle_bytes(ai, info)
        amg = {"solver": "amg_pcg (smoothed-aggregation AMG V-cycle, Jacobi w-smoother; P:236)",
               "tol": tol, "status": int(ast), "iterations": ait, "final_res": ares,
               "ms_per_solve": 1e3 * t_amg, "ms_per_iter": 1e3 * t_amg / max(1, ait),
               "setup_ms": setup_warm, "setup_ms_warm_runs": warm, "levels": ai["n"],
               "operator_complexity": ai["operatorComplexity"],
               "jacobi_pcg": {"iterations": jit, "ms_per_solve": 1e3 * t_jac, "status": int(jst)},
               "time_to_solution_speedup_vs_jacobi_pcg": t_jac / t_amg,
               "setup_ms_first_in_process": setup_cold,
               "setup_plus_solve_ms": setup_warm + 1e3 * t_amg,
               "setup_over_solve": setup_warm / (1e3 * t_amg),
               "speedup_vs_jacobi_pcg_incl_setup": t_jac / (t_amg + setup_warm / 1e3),
               "gpu_launches_per_solve": akern // args.steps,
               "vcycle": {"ms": vc_ms, "krylov_passes_ms": kr_ms, "bytes": vb,
                          "achieved": vb / (vc_ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                          "frac": vb / (vc_ms / 1e3) / 1e9 / peak, "bound": "hbm",
                          "peak_source": peak_src}}

    # c5 evidence leg (SURVEY §8(d) config 5 recipe at one GPU's share of its 50M cells): the irregular
    # RCM mesh on the SELL-32 layout, fixed iterations, live per-launch time of the fused pass
    # against the bytes the SELL-32 layout must move (12 B per stored entry incl. padding)
    c5 = None
    if world == 1 and not args.no_c5:
        g5 = meshgen.irregular_mesh(args.c5_n, seed=1505)
        A5 = ldu.LduMatrix.from_system(g5)
        A5.set_stream(stream.cuda_stream)
        i5 = A5.info()
        b5 = torch.from_numpy(g5.b).cuda()
        x5 = torch.zeros_like(b5)
        c5 = {"workload": f"c5 recipe, irregular {args.c5_n}^3 base ({g5.nCells:,} cells, "
                          f"{g5.nFaces:,} faces), RCM order; config 5 is 50M cells on 8 GPUs, "
                          f"i.e. 6.25M per GPU", "layout": i5["layout_name"],
              "stored_entries_per_row": i5["storedEntries"] / g5.nCells}
        for solver in ("pipecg", "pcg"):
            fn5 = A5.pcg_solve if solver == "pcg" else A5.pipecg_solve
            for _ in range(2):
                x5.zero_()
                fn5(b5, x5, tol=0.0, maxIter=args.iters)
            barrier()
            c0 = torch.cuda.Event(enable_timing=True)
            c1 = torch.cuda.Event(enable_timing=True)
            c0.record(stream)
            for _ in range(3):
                x5.zero_()
                fn5(b5, x5, tol=0.0, maxIter=args.iters)
            c1.record(stream)
            barrier()
            rate = 3 * args.iters / (c0.elapsed_time(c1) / 1e3)
            x5.zero_()
            fn5(b5, x5, tol=0.0, maxIter=args.iters, profile=True)
            s5 = A5.stats()
            slot = 1 if solver == "pipecg" else 0
            us = s5["passMs"][slot] / max(1, s5["passLaunches"][slot]) * 1e3
            fb5 = pass_format_bytes(solver, i5, g5.nCells)
            c5[solver] = {"iter_per_s": rate, "pass_us": us, "pass_bytes": fb5,
                          "pass_gbps": fb5 / us / 1e3, "pass_frac": fb5 / us / 1e3 / peak}
        A5.close()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k1, k2 = 3, 15
        (rate, per), core = pinned_to_one_core(
            lambda: oracle_iter_rate(sys_, sys_.b, args.solver, k1, k2))
        cpu = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"oracle {args.solver} (C, fp64, -O2, 1 thread, pinned to core {core}) on "
                         f"the same {n}^3 system: (t({k2} it) - t({k1} it)) / {k2 - k1}",
               "host": host_cpu(), "pinned_core": core,
               "model_equivalent_gbps": rate * bytes_iter / 1e9}

    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
               "steps": args.steps, "warmup": max(3, args.warmup),
               "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
               "config": config_dict(args, world, info),
               "effective_gbps": main_r["eff"],
               "effective_frac_of_hbm": main_r["eff"] / (peak * world),
               "bytes_per_iter": main_r["fb_iter"],
               "model_bytes_per_iter": bytes_iter, "model_equivalent_gbps": main_r["model_eff"],
               "stream_triad_gbps": triad, "hbm_peak_gbps": peak, "hbm_peak_source": peak_src,
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": kernels,
               "secondary": secondary, "amg": amg, "c5_irregular": c5,
               "clocks": clk, "last_status": int(st), "iterations_per_step": it}
        print(json.dumps(out), flush=True)
    A.close()
    if comm is not None:
        comm.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
