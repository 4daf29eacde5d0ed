#!/bin/bash
# Multi-GPU measurements on one box: bench.py at N ranks (torchrun) for a list of env variants.
# Usage: bash scripts/gpu_multi.sh <tag> "<N list>" "<variant env list, ';'-separated>" [bench args]
cd $GRAFT_REPO_ROOT
TAG=$1; NS=$2; VARS=$3; shift 3
mkdir -p gpurun_out/$TAG
IFS=';' read -ra VA <<< "$VARS"
for N in $NS; do
  i=0
  for V in "${VA[@]}"; do
    i=$((i+1))
    env $V timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N \
      --master-addr=127.0.0.1 --master-port=296$N$i bench.py --gpus $N --steps 10 --warmup 3 \
      --no-amg --no-e2e "$@" > gpurun_out/$TAG/bench_${N}_v$i.json 2> gpurun_out/$TAG/bench_${N}_v$i.err
    python - "$N" "$V" "gpurun_out/$TAG/bench_${N}_v$i.json" <<'PY'
import json, sys
N, V, path = sys.argv[1:4]
try:
    d = json.loads(open(path).read().strip().splitlines()[-1])
    r = d["roofline"]; s = d.get("secondary") or {"value": float("nan")}
    print("N=%s [%s] pipe %.0f it/s (%.1f us/it, pass %.1f us, share %.3f, frac %.3f) | pcg %.0f it/s" % (
        N, V, d["value"], 1e6 / d["value"], r["launch_us"], r["share_of_step"], r["frac"], s["value"]))
except Exception as e:
    print("N=%s [%s] FAILED %s" % (N, V, e))
PY
  done
done
