mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for r in 0 4 16; do
  for s in pipecg pcg; do
    LDU_RESERVE_SMS=$r timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 5 --warmup 3 --solver $s --no-secondary --no-e2e > gpurun_out/res_${r}_${s}.json 2> gpurun_out/res_${r}_${s}.err
    python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/res_${r}_${s}.json') if l.startswith('{')][0]; r=d['roofline']
print('N=$NG reserve=$r $s', round(d['value'],1), 'ms/step', round(d['ms_per_step'],2), r['kernel'], round(r['launch_us'],1), 'share', round(r['share_of_step'],2))" || tail -3 gpurun_out/res_${r}_${s}.err
  done
done
