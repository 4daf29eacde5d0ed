#!/usr/bin/env python
"""Measurements of the BASELINE.json configs other than the bench.py headline (config 3).

    python scripts/bench_configs.py c1|c2|c5|c2amg|c5amg (1 GPU)
    torchrun --nproc-per-node N scripts/bench_configs.py c4   (512^3 z-slabs over N GPUs)

Prints one JSON line per measurement (rank 0).  Times are device times (CUDA events on the
caller's stream, max over ranks); every solve goes through the C ABI.  The oracle is used only
to check the GPU's iteration counts / iterates on the same inputs (test-infrastructure use).
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402


def ev_time(stream, fn, reps=1):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    out = None
    for _ in range(reps):
        out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3, out


def c1(ldu):
    """16^3 Poisson to tol 1e-10, both solvers, vs oracle iteration counts."""
    import oracle
    s = meshgen.hex_laplacian(16, 16, 16, dirichlet=dict(x0=1.0))
    A = ldu.LduMatrix.from_system(s)
    st = torch.cuda.current_stream()
    A.set_stream(st.cuda_stream)
    b = torch.from_numpy(s.b).cuda()
    for name in ("pcg", "pipecg"):
        fn = A.pcg_solve if name == "pcg" else A.pipecg_solve
        x = torch.zeros_like(b)
        fn(b, x, tol=1e-10, maxIter=10000)
        reps = 50

        def run():
            x.zero_()
            return fn(b, x, tol=1e-10, maxIter=10000)
        t, (stt, it, res) = ev_time(st, run, reps)
        oit = (oracle.pcg if name == "pcg" else oracle.pipecg)(s, s.b, tol=1e-10, maxIter=10000)[2]
        print(json.dumps({"config": "c1 16^3 tol 1e-10", "solver": name, "iters": it,
                          "oracle_iters": oit, "solve_us": 1e6 * t / reps,
                          "iter_per_s": it * reps / t}), flush=True)


def c2(ldu):
    """icoFoam cavity pressure 1024^2: 20 PISO steps x 2 correctors = 40 warm-started solves,
    rel-L2 1e-6 (hot path) and the OpenFOAM normFactor criterion."""
    nx = ny = 1024
    s = meshgen.cavity_pressure_2d(nx, ny)
    A = ldu.LduMatrix.from_system(s)
    st = torch.cuda.current_stream()
    A.set_stream(st.cuda_stream)
    rhs = [torch.from_numpy(meshgen.cavity_rhs(nx, ny, t)).cuda() for t in range(20)]
    for name in ("pcg", "pipecg"):
        fn = A.pcg_solve if name == "pcg" else A.pipecg_solve
        for norm, tol in ((ldu.NORM_L2, 1e-6), (ldu.NORM_OPENFOAM, 1e-6)):
            x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
            its = []

            def seq():
                x.zero_()
                for t in range(20):
                    for corr in range(2):
                        _, it, _ = fn(rhs[t], x, tol=tol, maxIter=100000, norm=norm)
                        its.append(it)
            seq()
            its.clear()
            t, _ = ev_time(st, seq)
            print(json.dumps({"config": "c2 cavity 1024^2, 40 warm-started solves", "solver": name,
                              "norm": "L2" if norm == ldu.NORM_L2 else "OpenFOAM", "tol": tol,
                              "total_iters": int(sum(its)), "first_solve_iters": its[0],
                              "seconds": t, "iter_per_s": sum(its) / t}), flush=True)
        # icoFoam p / pFinal (NEXT-1): OpenFOAM norm, tol 1e-6, relTol 0.05 then 0 (reading Z26)
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        its = []

        def piso():
            x.zero_()
            for t in range(20):
                for corr, rt in ((0, 0.05), (1, 0.0)):
                    _, it, _ = fn(rhs[t], x, tol=1e-6, maxIter=100000, norm=ldu.NORM_OPENFOAM,
                                  relTol=rt)
                    its.append(it)
        piso()
        its.clear()
        t, _ = ev_time(st, piso)
        print(json.dumps({"config": "c2 cavity 1024^2, icoFoam p (relTol 0.05) / pFinal (relTol 0)",
                          "solver": name, "norm": "OpenFOAM", "tol": 1e-6,
                          "total_iters": int(sum(its)), "iters_p_pFinal_step0": its[:2],
                          "seconds": t, "iter_per_s": sum(its) / t}), flush=True)


def c5(ldu, n=200, iters=300):
    """Irregular (perturbed, RCM-renumbered) mesh on the SELL-32 path, fixed iterations."""
    import oracle
    t0 = time.time()
    s = meshgen.irregular_mesh(n, seed=1505)
    gen = time.time() - t0
    A = ldu.LduMatrix.from_system(s)
    info = A.info()
    st = torch.cuda.current_stream()
    A.set_stream(st.cuda_stream)
    b = torch.from_numpy(s.b).cuda()
    N, F = s.nCells, s.nFaces
    for name in ("pcg", "pipecg"):
        fn = A.pcg_solve if name == "pcg" else A.pipecg_solve
        x = torch.zeros_like(b)
        fn(b, x, tol=0.0, maxIter=iters)

        def run():
            x.zero_()
            return fn(b, x, tol=0.0, maxIter=iters)
        t, _ = ev_time(st, run, 3)
        rate = 3 * iters / t
        model = (88 if name == "pcg" else 136) * N + 16 * F
        # parity sample: 5 fixed iterations vs the oracle
        xs = torch.zeros_like(b)
        fn(b, xs, tol=0.0, maxIter=5)
        ox = (oracle.pcg if name == "pcg" else oracle.pipecg)(s, s.b, tol=0.0, maxIter=5)[1]
        rel = float(np.linalg.norm(xs.cpu().numpy() - ox) / np.linalg.norm(ox))
        print(json.dumps({"config": f"c5-like irregular {n}^3 base ({N:,} cells, {F:,} faces), RCM",
                          "layout": info["layout_name"], "solver": name, "iter_per_s": rate,
                          "effective_gbps_model": rate * model / 1e9, "rel_err_5it_vs_oracle": rel,
                          "generation_s": gen}), flush=True)


def amg_vs_jacobi(ldu, A, s, b, label, tol=1e-8, extra=None):
    """Time to solution (device) of Jacobi-PCG vs AMG-PCG / AMG-PipeCG, x0 = 0, and the AMG setup."""
    st = torch.cuda.current_stream()
    t0 = time.time()
    info = A.amg_setup()
    wall = time.time() - t0
    for name, fn in (("jacobi_pcg", A.pcg_solve), ("amg_pcg", A.amg_pcg_solve),
                     ("amg_pipecg", A.amg_pipecg_solve)):
        x = torch.zeros_like(b)
        fn(b, x, tol=tol, maxIter=100000)
        its = []

        def run():
            x.zero_()
            _, it, _ = fn(b, x, tol=tol, maxIter=100000)
            its.append(it)
        t, _ = ev_time(st, run, 3)
        y = torch.empty_like(x)
        A.amul(x, y)
        true = float(torch.linalg.norm(b - y) / torch.linalg.norm(b))
        d = {"config": label, "solver": name, "tol": tol, "iters": its[-1], "ms": 1e3 * t / 3,
             "true_res": true}
        if name.startswith("amg"):
            d.update({"setup_ms": info["setupMs"], "setup_wall_s": wall, "levels": info["n"],
                      "operator_complexity": info["operatorComplexity"]})
        if extra:
            d.update(extra)
        print(json.dumps(d), flush=True)


def c5amg(ldu, n=200):
    """NEXT-2 on the irregular mesh (SELL-32 layout): AMG-PCG vs Jacobi-PCG to tol 1e-8."""
    t0 = time.time()
    s = meshgen.irregular_mesh(n, seed=1505)
    gen = time.time() - t0
    A = ldu.LduMatrix.from_system(s)
    A.set_stream(torch.cuda.current_stream().cuda_stream)
    b = torch.from_numpy(s.b).cuda()
    amg_vs_jacobi(ldu, A, s, b, f"c5-like irregular {n}^3 base ({s.nCells:,} cells), RCM, "
                  f"{A.info()['layout_name']}", extra={"generation_s": gen})


def c2amg(ldu):
    """icoFoam p / pFinal sequence (c2, 1024^2) with AMG-PCG: one setup for the constant pressure
    matrix, 40 warm-started solves (OpenFOAM norm, tol 1e-6, relTol 0.05 then 0)."""
    nx = ny = 1024
    s = meshgen.cavity_pressure_2d(nx, ny)
    A = ldu.LduMatrix.from_system(s)
    st = torch.cuda.current_stream()
    A.set_stream(st.cuda_stream)
    info = A.amg_setup()
    rhs = [torch.from_numpy(meshgen.cavity_rhs(nx, ny, t)).cuda() for t in range(20)]
    for name, fn in (("jacobi_pcg", A.pcg_solve), ("amg_pcg", A.amg_pcg_solve)):
        x = torch.zeros(s.nCells, dtype=torch.float64, device="cuda")
        its = []

        def piso():
            x.zero_()
            for t in range(20):
                for rt in (0.05, 0.0):
                    _, it, _ = fn(rhs[t], x, tol=1e-6, maxIter=100000, norm=ldu.NORM_OPENFOAM,
                                  relTol=rt)
                    its.append(it)
        piso()
        its.clear()
        t, _ = ev_time(st, piso)
        print(json.dumps({"config": "c2 cavity 1024^2, icoFoam p (relTol 0.05) / pFinal (relTol 0)",
                          "solver": name, "norm": "OpenFOAM", "tol": 1e-6,
                          "total_iters": int(sum(its)), "seconds_40_solves": t,
                          "amg_setup_ms": info["setupMs"] if name == "amg_pcg" else None,
                          "amg_levels": info["n"] if name == "amg_pcg" else None}), flush=True)


def accuracy(ldu, sizes=(128, 256, 512)):
    """NEXT-4's condition: is the attainable accuracy of plain Ghysels-Vanroose
    pipelined CG (no residual replacement, reading Z7) a limit?  True residual ||b - A x|| / ||b||
    (library SpMV) vs the recurrence residual at tight tolerances, both solvers, hot-face RHS."""
    for n in sizes:
        s = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
        A = ldu.LduMatrix.from_system(s)
        b = torch.from_numpy(s.b).cuda()
        for tol in (1e-10, 1e-12, 1e-14):
            for name, fn, kw in (("pcg", A.pcg_solve, {}), ("pipecg", A.pipecg_solve, {}),
                                 ("pipecg_rr50", A.pipecg_solve, {"replaceEvery": 50})):
                x = torch.zeros_like(b)
                fn(b, x, tol=tol, maxIter=20000, **kw)
                x = torch.zeros_like(b)
                st, it, res = fn(b, x, tol=tol, maxIter=20000, **kw)
                ms = A.stats()["solveMs"]
                y = torch.empty_like(x)
                A.amul(x, y)
                true = float(torch.linalg.norm(b - y) / torch.linalg.norm(b))
                print(json.dumps({"config": f"accuracy {n}^3 hot face", "solver": name, "tol": tol,
                                  "status": int(st), "iters": it, "recurrence_res": res,
                                  "true_res": true, "solve_ms": ms,
                                  "ms_per_iter": ms / max(1, it)}), flush=True)
        A.close()


def c4(ldu, iters=300):
    """512^3 z-slabs over N GPUs (torchrun), fixed iterations, both solvers."""
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [ldu.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ldu.Comm(rank, world, uid[0], local)
    s = meshgen.hex_laplacian_slab(512, 512, 512, world, rank, dirichlet=dict(x0=1.0))
    A = ldu.LduMatrix.from_system(s, comm)
    st = torch.cuda.current_stream()
    A.set_stream(st.cuda_stream)
    b = torch.from_numpy(s.b).cuda()
    del s
    for name in ("pipecg", "pcg"):
        fn = A.pcg_solve if name == "pcg" else A.pipecg_solve
        x = torch.zeros_like(b)
        fn(b, x, tol=0.0, maxIter=20)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

        def run():
            x.zero_()
            return fn(b, x, tol=0.0, maxIter=iters)
        t, _ = ev_time(st, run, 2)
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"config": "c4 512^3 z-slabs", "n_gpus": world, "solver": name,
                              "iter_per_s": 2 * iters / float(tt.item())}), flush=True)
    A.close()
    if comm is not None:
        comm.close()
        dist.destroy_process_group()


def c5dist(ldu, n=None, iters=200, slow_rank_sms=None):
    """NEXT-3 (Eq 5-8): the irregular mesh over N GPUs with (a) equal-cell
    slabs, (b) nnz-balanced slabs, (c) the paper's measured re-decomposition: per-rank speed
    s_i = (n_i + 2 o_i) / T_i from each rank's own kernel time T_i with the equal slabs (Eq 5),
    r_i = s_i / sum s (Eq 6), n_i,new = N r_i (Eq 7-8), re-slab, measure again."""
    import torch.distributed as dist
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [ldu.Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = ldu.Comm(rank, world, uid[0], local)
    n = n or int(os.environ.get("C5_N", "160"))
    g = meshgen.irregular_mesh(n, seed=1505)
    st = torch.cuda.current_stream()
    if slow_rank_sms and rank == 0:
        # emulated heterogeneous node (the paper's Table 2 cluster): rank 0's kernels get only
        # `slow_rank_sms` SMs (read by ldu_setup when the matrix is configured)
        os.environ["LDU_RESERVE_SMS"] = str(torch.cuda.get_device_properties(local).multi_processor_count
                                            - slow_rank_sms)
    tag = f", rank 0 limited to {slow_rank_sms} SMs" if slow_rank_sms else ""

    def run(bounds, label):
        part = meshgen.slab_partition(g, world, bounds=bounds)[rank]
        A = ldu.LduMatrix.from_system(part, comm)
        A.set_stream(st.cuda_stream)
        b = torch.from_numpy(part.b).cuda()
        x = torch.zeros_like(b)
        A.pipecg_solve(b, x, tol=0.0, maxIter=20)
        dist.barrier()
        x.zero_()
        kms = []
        for _ in range(2):
            x.zero_()
            A.pipecg_solve(b, x, tol=0.0, maxIter=iters, profile=True)
            stt = A.stats()
            kms.append((stt["passMs"][1], stt["passLaunches"][1]))
        if os.environ.get("C5_DEBUG"):
            print(f"[rank {rank}] {label}: passMs/launches {kms}", flush=True)
        kern_ms = kms[-1][0]  # this rank's own fused-pass time
        dist.barrier()
        torch.cuda.synchronize()

        def solve():
            x.zero_()
            return A.pipecg_solve(b, x, tol=0.0, maxIter=iters)
        t, _ = ev_time(st, solve, 2)
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ks = [None] * world
        dist.all_gather_object(ks, (kern_ms, part.nCells, part.nFaces))
        A.close()
        if rank == 0:
            km = [k[0] for k in ks]
            print(json.dumps({"config": f"c5-like irregular {n}^3 base, pipelined CG, {world} GPUs{tag}",
                              "slabs": label, "iter_per_s": 2 * iters / float(tt.item()),
                              "rank_kernel_ms": [round(v, 2) for v in km],
                              "kernel_max_over_min": max(km) / min(km),
                              "rank_cells": [k[1] for k in ks]}), flush=True)
        return ks

    ks = run(meshgen.slab_bounds(g.nCells, world), "equal cells")
    run(meshgen.nnz_balanced_bounds(g, world), "equal non-zeros (static)")
    # Eq 5-8 from the measured kernel times of the equal-cell run
    s = [meshgen.speed(nc, nf, kms) for kms, nc, nf in ks]
    r = meshgen.relative_speeds(s)
    ks2 = run(meshgen.slab_bounds_weighted(g.nCells, r), "Eq 5-8 measured re-decomposition")
    # a second application of Eq 5-8 from the re-decomposed run's own times
    s = [meshgen.speed(nc, nf, kms) for kms, nc, nf in ks2]
    run(meshgen.slab_bounds_weighted(g.nCells, meshgen.relative_speeds(s)), "Eq 5-8, second pass")
    # functional performance model (FuPerMod): T_i(n) = a_i + b_i n fitted per rank from
    # its two measured sizes (equal cells, Eq 5-8), then equal predicted times (meshgen.fpm_partition)
    models = [meshgen.fit_time_model([k1[1], k2[1]], [k1[0], k2[0]]) for k1, k2 in zip(ks, ks2)]
    n_fpm = meshgen.fpm_partition(g.nCells, models)
    run(np.concatenate([[0], np.cumsum(n_fpm)]).astype(np.int64), "FPM fitted T(n) = a + b n (2 points)")
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import paper_1505_07630_b200 as ldu
    which = sys.argv[1] if len(sys.argv) > 1 else "c1"
    if which not in ("c4", "c5dist", "c5het"):
        torch.cuda.set_device(0)
    if which == "c5het":
        c5dist(ldu, slow_rank_sms=int(sys.argv[2]) if len(sys.argv) > 2 else 40)
    else:
        {"c1": c1, "c2": c2, "c4": c4, "c5": c5, "c5dist": c5dist, "c5amg": c5amg,
         "c2amg": c2amg, "accuracy": accuracy}[which](ldu)
