mkdir -p gpurun_out
for cfg in "16 1.25" "16 1.5" "16 1.8" "32 1.25"; do set -- $cfg
  LDU_AMG_LANE_ENTRIES=$1 LDU_AMG_SELL_PAD=$2 timeout 600 python scripts/amg_bench.py --n 256 --reps 3 --jacobi 0 --setups 1 > gpurun_out/tune_$1_$2.jsonl 2>gpurun_out/tune_$1_$2.err; echo "rc=$?"; tail -2 gpurun_out/tune_$1_$2.err
  python -c "
import json
for l in open('gpurun_out/tune_$1_$2.jsonl'):
    d=json.loads(l); print('lane $1 pad $2', d['solver'], d['iters'], round(d['solve_ms'],2), round(d['ms_per_iter'],4), [round(x,4) for x in d['pass_ms_per_iter']], d['hierarchy_bytes'])"
done
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
LDU_AMG_SELL_PAD=1.8 timeout 900 python -m pytest tests/test_gpu_amg.py -q -x -k "vcycle or solve_parity" > gpurun_out/amg_pytest2.log 2>&1; echo "amg pytest pad1.8 rc=$?"; tail -3 gpurun_out/amg_pytest2.log
