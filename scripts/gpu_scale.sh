# Multi-GPU: distributed parity + bench at N = 1, 2, 4 (whatever the box has)
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29533 tests/dist_worker.py 2>&1 | grep DIST | cut -c1-200
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  if [ $n -eq 1 ]; then
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/scale_$n.json 2> gpurun_out/scale_$n.err
  fi
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/scale_$n.json') if l.startswith('{')][0]; r=d['roofline']; s2=d['secondary']
print('N=$n', d['config']['solver'], round(d['value'],1), 'e2e', round(d['e2e']['value'],1), r['kernel'], round(r['launch_us'],1), 'us fmt', round(r['format_frac'],3), '| pcg', round(s2['value'],1), '| clk', d['clocks'])" || tail -5 gpurun_out/scale_$n.err
done
