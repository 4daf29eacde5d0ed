"""DIC-PCG / DIC-PipeCG (NEXT-1, readings Z35-Z36) against Jacobi-PCG and AMG-PCG on the
laplacianFoam hex Poisson (c3 recipe) and the icoFoam cavity pressure matrix (c2): iterations and
device time to tol, setup time, time per preconditioner apply.  One JSON line per case.

usage: python scripts/bench_dic.py [n ...]     (n = cube edge; default 128 256)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402


def timed_solve(A, fn, b, tol, reps=2):
    best = None
    for _ in range(reps):
        x = torch.zeros_like(b)
        st, it, res = fn(b, x, tol=tol, maxIter=20000)
        s = A.stats()
        if best is None or s["solveMs"] < best[3]:
            best = (st, it, res, s["solveMs"], s["iterMs"])
    st, it, res, ms, ims = best
    return {"status": st, "iterations": it, "final_res": res, "ms_per_solve": ms,
            "ms_per_iter": ims / max(1, it)}


def main():
    torch.cuda.set_device(0)
    sizes = [int(a) for a in sys.argv[1:]] or [128, 256]
    tol = 1e-8
    cases = [(f"hex{n}^3", lambda n=n: (meshgen.hex_laplacian(n, n, n), meshgen.rhs_hot_face(n, n, n)))
             for n in sizes]
    cases.append(("cavity1024^2", lambda: (meshgen.cavity_pressure_2d(1024, 1024),
                                           meshgen.cavity_rhs(1024, 1024, 1))))
    for name, mk in cases:
        sys_, bh = mk()
        b = torch.from_numpy(bh).cuda()
        out = {"case": name, "cells": sys_.nCells, "tol": tol}
        with ldu.LduMatrix.from_system(sys_) as A:
            out["jacobi_pcg"] = timed_solve(A, A.pcg_solve, b, tol)
            info = A.dic_setup()
            out["dic_info"] = info
            z = torch.empty_like(b)
            A.dic_apply(b, z)
            A.dic_apply(b, z)
            out["dic_apply_ms"] = A.stats()["solveMs"]
            out["dic_pcg"] = timed_solve(A, A.dic_pcg_solve, b, tol)
            out["dic_pipecg"] = timed_solve(A, A.dic_pipecg_solve, b, tol)
            A.amg_setup()
            out["amg_pcg"] = timed_solve(A, A.amg_pcg_solve, b, tol)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
