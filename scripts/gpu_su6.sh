mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/su6_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/su6_pytest.log
for g in 1 2 4; do
  if [ $g = 1 ]; then timeout 900 python bench.py > gpurun_out/su6_scale_$g.json 2> gpurun_out/su6_scale_$g.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus $g > gpurun_out/su6_scale_$g.json 2> gpurun_out/su6_scale_$g.err; fi
  echo "scale $g rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/su6_scale_$g.json').read().strip().splitlines()[-1]); r=d['roofline']; a=d.get('amg') or {}
print($g, round(d['value'],1), round(r['launch_us'],1), round(r['format_frac'],4), d['secondary']['value'], a.get('ms_per_solve'), (a.get('vcycle') or {}).get('frac'))"
done
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29551"
timeout 300 $R scripts/p2p_repro.py 512 pipe,pipe,pcg,pipe,pipe0 > gpurun_out/su6_repro.log 2>&1; echo "repro rc=$?"; grep "step\|REPRO" gpurun_out/su6_repro.log
timeout 900 python scripts/amg_bench.py --n 256 --tol 1e-8 --reps 3 > gpurun_out/su6_amg.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/su6_amg.jsonl'):
    d=json.loads(l); print(d['solver'], d['iters'], round(d['solve_ms'],2), round(d['ms_per_iter'],4), d['true_res'])"
