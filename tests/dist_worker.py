"""Multi-rank worker for the distributed parity test (launched by torchrun, one rank per GPU).

Every rank builds the same global system, takes its contiguous slab (meshgen.slab_partition),
sets up the NCCL comm (unique id broadcast over torch.distributed), and runs ldu_amul, pcg_solve
and pipecg_solve through the C ABI.  Rank 0 gathers the slabs and compares with the CPU oracle on
the global system.  Prints "DIST_OK <json>" on success; exits non-zero on failure.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import meshgen  # noqa: E402


def decoupled_boxes():
    a = meshgen.hex_laplacian(12, 10, 16, dirichlet=dict(x0=1.0))
    b = meshgen.hex_laplacian(12, 10, 16, conductance_sigma=0.5, seed=4, dirichlet=dict(x0=2.0))
    n = a.nCells
    return meshgen.LduSystem(2 * n, np.concatenate([a.lowerAddr, b.lowerAddr + n]).astype(np.int32),
                             np.concatenate([a.upperAddr, b.upperAddr + n]).astype(np.int32),
                             np.concatenate([a.diag, b.diag]), np.concatenate([a.upper, b.upper]),
                             None, np.concatenate([a.b, b.b]))


def slab_bounds_for(g, world):
    """LDU_DIST_BOUNDS: equal (default) cell slabs, Eq 5-8 weighted slabs (work
    fractions proportional to 1, 2, .., world -- a heterogeneous set of speeds), or slabs with
    equal non-zeros (meshgen.nnz_balanced_bounds, NEXT-3)."""
    mode = os.environ.get("LDU_DIST_BOUNDS", "equal")
    if mode == "weighted":
        r = meshgen.relative_speeds(np.arange(1, world + 1, dtype=float))
        return meshgen.slab_bounds_weighted(g.nCells, r)
    if mode == "nnz":
        return meshgen.nnz_balanced_bounds(g, world)
    return meshgen.slab_bounds(g.nCells, world)


def stress(rank, world, comm, ldu):
    """Repeated fused pipelined solves (>= 10^4 iterations in total on two mesh sizes): every
    repeat bitwise equal to the first, the first equal to the oracle."""
    ok = True
    out = {}
    total = 0
    for name, g, reps in (("hex24", meshgen.hex_laplacian(24, 20, 32, dirichlet=dict(x0=1.0)), 50),
                          ("hex40", meshgen.hex_laplacian(40, 36, 48, dirichlet=dict(x0=1.0)), 30)):
        parts = meshgen.slab_partition(g, world)
        bounds = meshgen.slab_bounds(g.nCells, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        A = ldu.LduMatrix.from_system(parts[rank], comm)
        b = torch.from_numpy(g.b[lo:hi].copy()).cuda()
        x0 = None
        its = set()
        same = True
        for k in range(reps):
            x = torch.zeros_like(b)
            st, it, _ = A.pipecg_solve(b, x, tol=1e-10, maxIter=5000)
            its.add((st, it))
            total += it
            if x0 is None:
                x0 = x.clone()
            else:
                same &= bool(torch.equal(x, x0))
        A.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, (sorted(its), same, x0.cpu().numpy()))
        if rank == 0:
            import oracle
            ost, ox, oit, _ = oracle.pipecg(g, g.b, tol=1e-10, maxIter=5000)
            x_all = np.concatenate([o[2] for o in gathered])
            rel = float(np.linalg.norm(x_all - ox) / np.linalg.norm(ox))
            its_all = {tuple(t) for o in gathered for t in o[0]}
            good = (all(o[1] for o in gathered) and len(its_all) == 1 and rel <= 1e-8
                    and abs(next(iter(its_all))[1] - oit) <= max(1, round(0.02 * oit)))
            out[name] = dict(iters=sorted(its_all), oracle_iters=oit, rel=rel,
                             repeats_bitwise=all(o[1] for o in gathered), reps=reps)
            ok &= good
    tot = [None] * world
    dist.all_gather_object(tot, total)
    if rank == 0:
        out["total_iterations_per_rank"] = tot[0]
        ok &= tot[0] >= 10000
    return ok, out


def main():
    from dist_boot import boot
    rank, world, comm = boot()
    import paper_1505_07630_b200 as ldu
    if len(sys.argv) > 1 and sys.argv[1] == "stress":
        ok, out = stress(rank, world, comm, ldu)
        comm.close()
        dist.barrier()
        dist.destroy_process_group()
        if rank == 0:
            print(("DIST_STRESS_OK " if ok else "DIST_STRESS_FAIL ") + json.dumps(out), flush=True)
            sys.exit(0 if ok else 1)
        return
    results = {}
    cases = {
        "hex": lambda: meshgen.hex_laplacian(24, 20, 32, dirichlet=dict(x0=1.0)),
        "hex_sigma": lambda: meshgen.hex_laplacian(17, 13, 19, conductance_sigma=0.8, seed=3,
                                                   dirichlet=dict(x0=1.0)),
        "irregular": lambda: meshgen.irregular_mesh(14, seed=7),
        # two disconnected boxes: with 2 ranks each rank owns one and has NO interface (a rank
        # of a multi-rank comm with nothing to exchange); with 4 ranks each box is cut once
        "decoupled": lambda: decoupled_boxes(),
    }
    ok = True
    for name, mk in cases.items():
        g = mk()
        bounds = slab_bounds_for(g, world)
        parts = meshgen.slab_partition(g, world, bounds=bounds)
        me = parts[rank]
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        A = ldu.LduMatrix.from_system(me, comm)
        xg = np.random.default_rng(5).uniform(-1, 1, g.nCells)
        y = torch.empty(me.nCells, dtype=torch.float64, device="cuda")
        A.amul(torch.from_numpy(xg[lo:hi].copy()).cuda(), y)
        out = {"amul": y.cpu().numpy()}
        b = torch.from_numpy(g.b[lo:hi].copy()).cuda()
        for solver in ("pcg", "pipecg"):
            fn = A.pcg_solve if solver == "pcg" else A.pipecg_solve
            # back-to-back solves on one handle (fixed-iteration, converged, warm restart)
            xw = torch.zeros_like(b)
            fn(b, xw, tol=0.0, maxIter=7)
            fn(b, xw, tol=1e-10, maxIter=5000)
            x = torch.zeros_like(b)
            st, it, res = fn(b, x, tol=1e-10, maxIter=5000)
            stats = A.stats()
            x2 = torch.zeros_like(b)
            st2, it2, _ = fn(b, x2, tol=1e-10, maxIter=5000)
            if not (st2 == st and it2 == it and torch.equal(x2, x)):
                print(f"[rank {rank}] {name} {solver}: repeat solve differs: status {st}/{st2} "
                      f"iters {it}/{it2} max|dx| {float((x2 - x).abs().max()):.3e}", flush=True)
                out.setdefault("repeat_bad", []).append(solver)
            out[solver] = (st, it, res, x.cpu().numpy(), stats["allreduces"], stats["reductions"])
            # OpenFOAM normFactor + relTol + minIter + residual history across ranks (Z1, Z26)
            xo = torch.zeros_like(b)
            sto, ito, reso = fn(b, xo, tol=1e-6, maxIter=5000, norm=ldu.NORM_OPENFOAM,
                                relTol=0.01, minIter=3, record_history=True)
            out[solver + "_of"] = (sto, ito, reso, xo.cpu().numpy(), A.history())
            if (solver == "pipecg" and os.environ.get("LDU_PIPE_FUSE", "1") != "0"
                    and os.environ.get("LDU_P2P", "1") != "0"):
                # residual replacement every 25 iterations across ranks (NEXT-4, reading Z7)
                xr = torch.zeros_like(b)
                str_, itr, resr = fn(b, xr, tol=1e-10, maxIter=5000, replaceEvery=25,
                                     record_history=True)
                out["pipecg_rr"] = (str_, itr, resr, xr.cpu().numpy(), A.history())
        A.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            import oracle
            bad = sorted({s_ for o in gathered for s_ in o.get("repeat_bad", [])})
            if bad:
                print(f"{name}: repeat solve differs for {bad}", flush=True)
                ok = False
            y_all = np.concatenate([o["amul"] for o in gathered])
            yo = oracle.amul(g, xg)
            r = {"amul_rel": float(np.linalg.norm(y_all - yo) / np.linalg.norm(yo))}
            ok &= r["amul_rel"] <= 1e-12
            for solver in ("pcg", "pipecg"):
                ofn = oracle.pcg if solver == "pcg" else oracle.pipecg
                ost, ox, oit, ores = ofn(g, g.b, tol=1e-10, maxIter=5000)
                sts = {o[solver][0] for o in gathered}
                its = {o[solver][1] for o in gathered}
                x_all = np.concatenate([o[solver][3] for o in gathered])
                rel = float(np.linalg.norm(x_all - ox) / np.linalg.norm(ox))
                it = gathered[0][solver][1]
                reds = gathered[0][solver][4]
                r[solver] = dict(status=sorted(sts), iters=sorted(its), oracle_iters=oit,
                                 rel=rel, allreduces=reds)
                ok &= sts == {0} and len(its) == 1 and abs(it - oit) <= max(1, round(0.02 * oit))
                ok &= rel <= 1e-8
                # device-counted cross-rank reductions (reading Z4 / P:97): classical = the r0
                # reduction + 2 per iteration; pipelined = r0 + (gamma, delta, rr) of r0 + ONE per
                # iteration (the trip that finds r_it converged consumes the last one)
                expect = 1 + 2 * it if solver == "pcg" else 2 + it
                r[solver]["expected_allreduces"] = expect
                ok &= reds == expect and gathered[0][solver][5] == expect
                # OpenFOAM criterion with relTol / minIter: same stop and history as the oracle
                ost2, ox2, oit2, ores2, ohist2 = ofn(g, g.b, tol=1e-6, maxIter=5000,
                                                     norm=oracle.NORM_OPENFOAM, relTol=0.01,
                                                     minIter=3, history=True)
                of = [o[solver + "_of"] for o in gathered]
                x_of = np.concatenate([o[3] for o in of])
                rel_of = float(np.linalg.norm(x_of - ox2) / np.linalg.norm(ox2))
                hist = of[0][4]
                hist_ok = len(hist) == of[0][1] + 1 and np.allclose(hist[:len(ohist2)], ohist2[:len(hist)], rtol=1e-6)
                r[solver + "_openfoam"] = dict(iters=sorted({o[1] for o in of}), oracle_iters=oit2,
                                               rel=rel_of, history_ok=bool(hist_ok))
                ok &= {o[0] for o in of} == {0} and {o[1] for o in of} == {oit2}
                ok &= rel_of <= 1e-8 and hist_ok
            if "pipecg_rr" in gathered[0]:
                ost3, ox3, oit3, ores3, ohist3 = oracle.pipecg(g, g.b, tol=1e-10, maxIter=5000,
                                                               history=True, replace_every=25)
                rr = [o["pipecg_rr"] for o in gathered]
                x_rr = np.concatenate([o[3] for o in rr])
                rel_rr = float(np.linalg.norm(x_rr - ox3) / np.linalg.norm(ox3))
                h3 = rr[0][4]
                m3 = min(len(h3), len(ohist3), 60)
                hist_rr = bool(np.allclose(h3[:m3], ohist3[:m3], rtol=1e-7))
                r["pipecg_replace25"] = dict(iters=sorted({o[1] for o in rr}), oracle_iters=oit3,
                                             rel=rel_rr, history_ok=hist_rr)
                ok &= {o[0] for o in rr} == {0} and len({o[1] for o in rr}) == 1
                ok &= abs(rr[0][1] - oit3) <= max(1, round(0.02 * oit3))
                ok &= rel_rr <= 1e-8 and hist_rr
            results[name] = r
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(("DIST_OK " if ok else "DIST_FAIL ") + json.dumps(results), flush=True)
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
