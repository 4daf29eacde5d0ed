"""Process-group + library-communicator bootstrap shared by the multi-rank test workers.

LDU_DIST_BOOT=nccl (default when every rank has its own GPU): torch.distributed over NCCL and
ldu_comm_init (NCCL unique id broadcast over it).
LDU_DIST_BOOT=host: torch.distributed over gloo and ldu_comm_init_host -- no NCCL anywhere; every
in-solve exchange runs over the library's peer-memory mailboxes (CUDA IPC), so several ranks may
share one GPU (rank r uses device r % torch.cuda.device_count()).  This is how the multi-rank
CUDA path is parity-tested on a single-GPU box.
"""
import os

import torch
import torch.distributed as dist


def boot():
    """Returns (rank, world, comm) after torch.cuda.set_device and init_process_group."""
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    mode = os.environ.get("LDU_DIST_BOOT", "nccl")
    import paper_1505_07630_b200 as ldu
    if mode == "host":
        dev = local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")
        comm = ldu.Comm.host(rank, world, dev)
    else:
        dev = local
        torch.cuda.set_device(dev)
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        uid = [ldu.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = ldu.Comm(rank, world, uid[0], dev)
    return rank, world, comm
