mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29551"
timeout 300 $R scripts/p2p_repro.py 512 pipe,pipe,pcg,pipe,pipe0 > gpurun_out/repro1.log 2>&1; echo "repro1 rc=$?"; grep "step\|REPRO" gpurun_out/repro1.log
timeout 900 $R scripts/amg_dist_bench.py --mesh 512 > gpurun_out/amgd_512_4.jsonl 2> gpurun_out/amgd_512_4.err; echo "amgd 512/4 rc=$?"; cat gpurun_out/amgd_512_4.jsonl
timeout 1200 python -m pytest tests/test_dist_gpu.py -q -x > gpurun_out/dist_all.log 2>&1; echo "dist all rc=$?"; tail -3 gpurun_out/dist_all.log
for g in 1 2 4; do
  if [ $g = 1 ]; then timeout 600 python bench.py --no-amg --no-cpu-baseline > gpurun_out/scale_$g.json 2> gpurun_out/scale_$g.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus $g > gpurun_out/scale_$g.json 2> gpurun_out/scale_$g.err; fi
  echo "scale $g rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/scale_$g.json').read().strip().splitlines()[-1]); print($g, round(d['value'],1), d['secondary']['value'])"
done
