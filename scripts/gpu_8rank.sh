#!/bin/bash
# 8-rank path on a box with fewer GPUs (host bootstrap, ranks share GPUs): parity worker and a
# short bench run -- correctness / no-hang evidence for the driver's 8-GPU step (timings here are
# NOT a scaling measurement: two ranks time-share each GPU).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2_8rank
LDU_DIST_BOOT=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
  --master-addr=127.0.0.1 --master-port=29621 tests/dist_worker.py > gpurun_out/r2_8rank/worker.log 2>&1
echo "worker rc=$? $(grep -o 'DIST_[A-Z]*' gpurun_out/r2_8rank/worker.log | head -1)"
LDU_DIST_BOOT=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
  --master-addr=127.0.0.1 --master-port=29622 tests/dist_amg_worker.py > gpurun_out/r2_8rank/amg.log 2>&1
echo "amg worker rc=$? $(grep -o 'DIST_AMG_[A-Z]*' gpurun_out/r2_8rank/amg.log | head -1)"
LDU_DIST_BOOT=host timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 \
  --master-addr=127.0.0.1 --master-port=29623 bench.py --gpus 8 --steps 3 --warmup 3 --no-amg \
  > gpurun_out/r2_8rank/bench8.json 2> gpurun_out/r2_8rank/bench8.err
echo "bench8 rc=$?"; tail -c 600 gpurun_out/r2_8rank/bench8.json
