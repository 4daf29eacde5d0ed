#!/bin/bash
# Device %globaltimer breakdown of the multi-rank pipelined loop (LDU_TRACE=2) at N ranks.
cd $GRAFT_REPO_ROOT
N=$1; shift
env "$@" LDU_TRACE=2 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
    --master-addr=127.0.0.1 --master-port=2971$N bench.py --gpus $N --steps 3 --warmup 3 \
    --no-amg --no-e2e --no-secondary --no-profile 2>&1 >/dev/null | grep gtimer | sort | uniq | head -8
