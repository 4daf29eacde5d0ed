"""Multi-rank worker for the distributed AMG parity test (block-Jacobi AMG, reading Z33).

Every rank takes its contiguous slab of the same global system, builds the AMG hierarchy of its
LOCAL matrix on the device (ldu_amg_setup), and runs AMG-PCG / AMG-PipeCG through the C ABI with
the halo exchange in the Krylov SpMV.  Rank 0 compares with the oracle's serial emulation
(oracle.amg.block_hierarchies + amg_block_solve on the global system): per-rank hierarchy sizes
and level-0 aggregates bit-exact, iteration counts within +-2 % (+-1), solution rel-L2 <= 1e-8 at
tol 1e-10, fixed-iteration residual histories.  Prints "DIST_AMG_OK <json>" on success.
With argument "dic" the same checks run for block-Jacobi DIC (ldu_dic_setup, dic_*_solve; readings
Z35-Z36) against oracle.dic_pcg(bounds=...).
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


def main():
    from dist_boot import boot
    rank, world, comm = boot()
    import paper_1505_07630_b200 as ldu
    dic = len(sys.argv) > 1 and sys.argv[1] == "dic"
    cases = {
        "hex": lambda: meshgen.hex_laplacian(24, 20, 32, dirichlet=dict(x0=1.0)),
        "hex_sigma": lambda: meshgen.hex_laplacian(21, 17, 19, conductance_sigma=0.6, seed=3,
                                                   dirichlet=dict(x0=1.0)),
        "irregular": lambda: meshgen.irregular_mesh(14, seed=7),
    }
    ok = True
    results = {}
    for name, mk in cases.items():
        g = mk()
        parts = meshgen.slab_partition(g, world)
        bounds = meshgen.slab_bounds(g.nCells, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        A = ldu.LduMatrix.from_system(parts[rank], comm)
        if dic:
            A.dic_setup()
            out = {}
        else:
            info = A.amg_setup()
            out = {"sizes": info["n"], "agg0": A.amg_aggregates(0) if info["nLevels"] else None}
        b = torch.from_numpy(g.b[lo:hi].copy()).cuda()
        for solver in ("pcg", "pipecg"):
            if dic:
                fn = A.dic_pcg_solve if solver == "pcg" else A.dic_pipecg_solve
            else:
                fn = A.amg_pcg_solve if solver == "pcg" else A.amg_pipecg_solve
            x = torch.zeros_like(b)
            st, it, res = fn(b, x, tol=1e-10, maxIter=500)
            reds = A.stats()["allreduces"]
            x2 = torch.zeros_like(b)
            st2, it2, _ = fn(b, x2, tol=1e-10, maxIter=500)
            assert st2 == st and it2 == it and torch.equal(x2, x), "repeat solve differs"
            xf = torch.zeros_like(b)
            stf, itf, _ = fn(b, xf, tol=0.0, maxIter=6, record_history=True, batch=4)
            out[solver] = (st, it, res, x.cpu().numpy(), reds, stf, itf, A.history())
        A.close()
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            import oracle
            from oracle import amg
            if dic:
                r = {}
            else:
                Hs = amg.block_hierarchies(parts)
                r = {"sizes_ok": all(gathered[k]["sizes"] == Hs[k].sizes for k in range(world))}
                ok &= r["sizes_ok"]
                ok &= all(gathered[k]["agg0"] is None or np.array_equal(gathered[k]["agg0"], Hs[k].levels[0].agg)
                          for k in range(world))
            for solver in ("pcg", "pipecg"):
                pip = solver == "pipecg"
                if dic:
                    ost, ox, oit, ores = oracle.dic_pcg(g, g.b, tol=1e-10, maxIter=500,
                                                        pipelined=pip, bounds=bounds)
                    _, _, _, _, ohist = oracle.dic_pcg(g, g.b, tol=0.0, maxIter=6, pipelined=pip,
                                                       bounds=bounds, history=True)
                else:
                    ost, ox, oit, ores = amg.amg_block_solve(g, g.b, bounds, Hs, tol=1e-10,
                                                             maxIter=500, pipelined=pip)
                    _, _, _, _, ohist = amg.amg_block_solve(g, g.b, bounds, Hs, tol=0.0,
                                                            maxIter=6, pipelined=pip, history=True)
                sts = {o[solver][0] for o in gathered}
                its = {o[solver][1] for o in gathered}
                it = gathered[0][solver][1]
                x_all = np.concatenate([o[solver][3] for o in gathered])
                rel = float(np.linalg.norm(x_all - ox) / np.linalg.norm(ox))
                hist = gathered[0][solver][7]
                hist_ok = len(hist) == 7 and bool(np.allclose(hist, ohist, rtol=1e-8))
                r[solver] = dict(status=sorted(sts), iters=sorted(its), oracle_iters=oit, rel=rel,
                                 allreduces=gathered[0][solver][4], history_ok=hist_ok,
                                 fixed=(gathered[0][solver][5], gathered[0][solver][6]))
                ok &= sts == {0} and len(its) == 1 and abs(it - oit) <= max(1, round(0.02 * oit))
                ok &= rel <= 1e-8 and hist_ok and gathered[0][solver][6] == 6
                ok &= gathered[0][solver][4] >= (1 if pip else 3) * it  # reductions per iteration
            results[name] = r
    comm.close()
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(("DIST_AMG_OK " if ok else "DIST_AMG_FAIL ") + json.dumps(results), flush=True)
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
