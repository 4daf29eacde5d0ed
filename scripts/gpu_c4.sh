#!/bin/bash
# c4: 512^3 Poisson (134M cells), pipelined CG, 1 / 2 / 4 GPUs (z-slabs), fixed iterations.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2_c4
ARGS="--cube 512 --iters 100 --steps 3 --warmup 3 --no-secondary --no-amg --no-e2e --no-cpu-baseline"
timeout 900 python bench.py $ARGS > gpurun_out/r2_c4/bench_1.json 2> gpurun_out/r2_c4/bench_1.err
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=2983$N bench.py --gpus $N $ARGS > gpurun_out/r2_c4/bench_$N.json 2> gpurun_out/r2_c4/bench_$N.err
done
for N in 1 2 4; do python - "$N" <<'PY'
import json, sys
N = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/r2_c4/bench_{N}.json").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"512^3 N={N}: {d['value']:.1f} it/s ({1e6/d['value']:.1f} us/it), pass {r['launch_us']:.1f} us frac {r['frac']:.3f}")
except Exception as e:
    print(f"512^3 N={N}: FAILED {e}")
PY
done
