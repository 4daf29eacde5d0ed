"""Repro of the 512^3 / 4-rank pipelined-CG failure: fresh handle pipecg (tol), then pcg -> pipecg,
then fixed-iteration pipecg; prints per-step status on rank 0."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import meshgen  # noqa: E402
import paper_1505_07630_b200 as ldu  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
uid = [ldu.Comm.unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
comm = ldu.Comm(rank, world, uid[0], local)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = sys.argv[2].split(",") if len(sys.argv) > 2 else ["pipe", "pipe", "pcg", "pipe", "pipe0"]
sys_ = meshgen.hex_laplacian_slab(n, n, n, world, rank, dirichlet=dict(x0=1.0))
A = ldu.LduMatrix.from_system(sys_, comm)
b = torch.from_numpy(sys_.b).cuda()
for k, stp in enumerate(steps):
    x = torch.zeros_like(b)
    try:
        if stp == "pipe":
            r = A.pipecg_solve(b, x, tol=1e-8, maxIter=20000)
        elif stp == "pipe0":
            r = A.pipecg_solve(b, x, tol=0.0, maxIter=300)
        elif stp == "pcg":
            r = A.pcg_solve(b, x, tol=1e-8, maxIter=20000)
        torch.cuda.synchronize()
        if rank == 0:
            print(f"step {k} {stp}: {r} {A.stats()['solveMs']:.1f} ms", flush=True)
    except Exception as e:
        print(f"rank {rank} step {k} {stp}: FAILED {e}", flush=True)
        sys.exit(1)
dist.barrier()
if rank == 0:
    print("REPRO_DONE", flush=True)
