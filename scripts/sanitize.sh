#!/bin/bash
# compute-sanitizer sweep, ONE tool per gpurun call (B200_PROFILING.md): smoke(), small SpMV /
# solver / AMG / DIC parity cases, and (memcheck only) a 2-rank shared-GPU multi-rank run.
#   bash scripts/sanitize.sh memcheck|racecheck|synccheck|initcheck
cd $GRAFT_REPO_ROOT
T=$1
OUT=gpurun_out/r2_sanitize_$T
mkdir -p $OUT
CS="compute-sanitizer --tool $T --print-limit 30 --error-exitcode 99"
run() {  # name, command...
  local name=$1; shift
  timeout 1200 $CS "$@" > $OUT/$name.log 2>&1
  echo "$T $name rc=$? $(grep -h 'ERROR SUMMARY' $OUT/$name.log | tail -1)"
}
run smoke python __graft_entry__.py smoke
run parity python -m pytest -q -x tests/test_gpu_parity.py -k "amul_parity or (solve_parity and c1_hot) or edge_cases or fixed_iterations"
run amg python -m pytest -q -x tests/test_gpu_amg.py -k "hex16 or vcycle_parity"
run dic python -m pytest -q -x tests/test_gpu_dic.py -k "not 128 and not 256"
if [ "$T" == "memcheck" ]; then
  LDU_DIST_BOOT=host timeout 1500 $CS --target-processes all python -m torch.distributed.run --nnodes=1 \
    --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29599 tests/dist_worker.py > $OUT/dist2.log 2>&1
  echo "$T dist2 rc=$? $(grep -h 'ERROR SUMMARY' $OUT/dist2.log | sort | uniq -c | head -3) $(grep -c DIST_OK $OUT/dist2.log)"
fi
