"""c5 (irregular, RCM, SELL-32) kernel measurement: live per-launch time of the dominant passes
(profile event nodes) against the bytes the SELL-32 layout must move.
    python scripts/c5_profile.py [n=200] [iters=100]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402
from bench import pass_format_bytes, hbm_peak  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
t0 = time.time()
s = meshgen.irregular_mesh(n, seed=1505)
gen = time.time() - t0
A = ldu.LduMatrix.from_system(s)
info = A.info()
b = torch.from_numpy(s.b).cuda()
N = s.nCells
peak, _ = hbm_peak()
out = {"n": n, "cells": N, "faces": s.nFaces, "layout": info["layout_name"],
       "storedEntries": info["storedEntries"], "entries_per_row": info["storedEntries"] / N,
       "gen_s": gen}
for solver in ("pipecg", "pcg"):
    fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
    x = torch.zeros_like(b)
    fn(b, x, tol=0.0, maxIter=iters)
    x.zero_()
    fn(b, x, tol=0.0, maxIter=iters, profile=True)
    st = A.stats()
    slot = 1 if solver == "pipecg" else 0
    us = st["passMs"][slot] / st["passLaunches"][slot] * 1e3
    fb = pass_format_bytes(solver, info, N)
    x.zero_()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(b, x, tol=0.0, maxIter=iters)
    e1.record()
    torch.cuda.synchronize()
    it_s = iters / (e0.elapsed_time(e1) / 1e3)
    out[solver] = {"iter_per_s": it_s, "pass_us": us, "pass_bytes": fb,
                   "pass_gbps": fb / us / 1e3, "pass_frac": fb / us / 1e3 / peak}
print(json.dumps(out), flush=True)
