"""AMG-CG / AMG-PipeCG vs Jacobi-PCG / PipeCG time to solution (NEXT-2, Table 2).

One JSON line per (mesh, solver): setup ms, iterations, device solve ms, ms per iteration, per-pass
split (V-cycle vs Krylov passes, profile run), hierarchy sizes.  Usage:
    python scripts/amg_bench.py [--n 64 128 256] [--tol 1e-8] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--jacobi", type=int, default=1)
    ap.add_argument("--only", default="", help="comma-separated solver names")
    ap.add_argument("--setups", type=int, default=2, help="hierarchy builds (timed)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for n in a.n:
        sys_ = meshgen.hex_laplacian(n, n, n)
        b = torch.from_numpy(meshgen.rhs_hot_face(n, n, n)).cuda()
        with ldu.LduMatrix.from_system(sys_) as A:
            t0 = time.perf_counter()
            info = A.amg_setup()
            wall = (time.perf_counter() - t0) * 1e3
            walls = []
            for _ in range(a.setups - 1):  # rebuilds: no first-touch / module-load effects
                t0 = time.perf_counter()
                info = A.amg_setup()
                walls.append((time.perf_counter() - t0) * 1e3)
            wall2 = float(np.median(walls)) if walls else wall
            solvers = [("amg_pcg", A.amg_pcg_solve), ("amg_pipecg", A.amg_pipecg_solve)]
            if a.jacobi:
                solvers += [("jacobi_pcg", A.pcg_solve), ("jacobi_pipecg", A.pipecg_solve)]
            if a.only:
                solvers = [sv for sv in solvers if sv[0] in a.only.split(",")]
            for name, fn in solvers:
                ms, its = [], []
                for r in range(a.reps + 1):
                    x = torch.zeros_like(b)
                    st, it, res = fn(b, x, tol=a.tol, maxIter=20000)
                    if r:
                        ms.append(A.stats()["solveMs"])
                        its.append(it)
                x = torch.zeros_like(b)
                fn(b, x, tol=a.tol, maxIter=20000, profile=True)
                prof = A.stats()
                y = torch.empty_like(x)
                A.amul(x, y)
                true = (torch.linalg.norm(b - y) / torch.linalg.norm(b)).item()
                line = {"n": n, "cells": sys_.nCells, "solver": name, "tol": a.tol, "status": st,
                        "iters": its[-1], "solve_ms": float(np.median(ms)),
                        "ms_per_iter": float(np.median(ms)) / max(1, its[-1]),
                        "final_res": res, "true_res": true,
                        "pass_ms_per_iter": [p / max(1, l) for p, l in zip(prof["passMs"], prof["passLaunches"])],
                        "kernels": prof["kernels"]}
                if name.startswith("amg"):
                    line.update({"setup_ms_device": info["setupMs"], "setup_ms_wall_first": wall,
                                 "setup_ms_wall": wall2, "levels": info["n"],
                                 "operator_complexity": info["operatorComplexity"],
                                 "omega": info["omega"], "hierarchy_bytes": info["deviceBytes"]})
                print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
