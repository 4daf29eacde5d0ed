#!/bin/bash
# c5 recipe at 256^3 base (16.8M cells, RCM, SELL-32) on 1 / 2 / 4 identical GPUs: pipelined CG,
# equal-cell / equal-nnz / Eq 5-8 / FPM slabs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2_c5dist
for N in 4 2 1; do
  C5_N=${C5_N:-256} timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
    --master-addr=127.0.0.1 --master-port=2984$N scripts/bench_configs.py c5dist \
    > gpurun_out/r2_c5dist/c5d_$N.jsonl 2> gpurun_out/r2_c5dist/c5d_$N.err
  echo "N=$N rc=$?"; cut -c1-260 gpurun_out/r2_c5dist/c5d_$N.jsonl | head -2
done
