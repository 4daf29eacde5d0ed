"""Time to solution of AMG-PCG / AMG-PipeCG (block-Jacobi across ranks, reading Z33) vs
Jacobi-PCG / PipeCG on an n^3 Poisson split into z-slabs, one rank per GPU (torchrun).
Rank 0 prints one JSON line per solver: iterations, device ms (max over ranks), setup ms."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mesh", type=int, default=256)
    ap.add_argument("--tol", type=float, default=1e-8)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        uid = [ldu.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ldu.Comm(rank, world, uid[0], local)
    n = a.mesh
    if world == 1:
        sys_ = meshgen.hex_laplacian(n, n, n, dirichlet=dict(x0=1.0))
    else:
        sys_ = meshgen.hex_laplacian_slab(n, n, n, world, rank, dirichlet=dict(x0=1.0))
    A = ldu.LduMatrix.from_system(sys_, comm)
    info = A.amg_setup()
    b = torch.from_numpy(sys_.b).cuda()

    def gmax(v):
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    setup = gmax(info["setupMs"])
    for name, fn in (("amg_pcg", A.amg_pcg_solve), ("amg_pipecg", A.amg_pipecg_solve),
                     ("jacobi_pcg", A.pcg_solve), ("jacobi_pipecg", A.pipecg_solve)):
        ms = []
        for r in range(a.reps + 1):
            x = torch.zeros_like(b)
            st, it, res = fn(b, x, tol=a.tol, maxIter=20000)
            if r:
                ms.append(gmax(A.stats()["solveMs"]))
        ms.sort()
        if rank == 0:
            print(json.dumps({"n": n, "gpus": world, "solver": name, "tol": a.tol, "status": st,
                              "iters": it, "solve_ms": ms[len(ms) // 2],
                              "ms_per_iter": ms[len(ms) // 2] / max(1, it),
                              "amg_setup_ms_max_rank": setup if name.startswith("amg") else None,
                              "local_levels_rank0": info["n"] if name.startswith("amg") else None}),
                  flush=True)
    A.close()
    if comm is not None:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
