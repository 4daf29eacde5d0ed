#!/bin/bash
# NEXT-3 measurement: c5-like irregular mesh with one emulated slow rank (40 SMs), N = 4 and 2.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2_c5het
for N in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=2981$N scripts/bench_configs.py c5het 40 > gpurun_out/r2_c5het/c5h_$N.jsonl 2> gpurun_out/r2_c5het/c5h_$N.err
  cut -c1-400 gpurun_out/r2_c5het/c5h_$N.jsonl
done
