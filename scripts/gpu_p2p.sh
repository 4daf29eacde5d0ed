mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29533 tests/dist_worker.py 2>&1 | grep -E "DIST|Error|error" | cut -c1-400 | head -5
LDU_PIPE_FUSE=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29533 tests/dist_worker.py 2>&1 | grep -E "DIST|Error|error" | cut -c1-100 | head -5
for cfg in "1 1 pipecg" "1 0 pipecg" "1 1 pcg"; do
  set -- $cfg; p=$1; f=$2; s=$3
  LDU_P2P=$p LDU_PIPE_FUSE=$f timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 5 --warmup 3 --solver $s --no-secondary --no-e2e > gpurun_out/p2p_${p}_${f}_${s}.json 2> gpurun_out/p2p_${p}_${f}_${s}.err
  python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/p2p_${p}_${f}_${s}.json') if l.startswith('{')][0]; r=d['roofline']
print('N=$NG p2p=$p fuse=$f $s', round(d['value'],1), 'ms/step', round(d['ms_per_step'],2), r['kernel'], round(r['launch_us'],1), 'share', round(r['share_of_step'],2))" || grep -v "^\*\|OMP" gpurun_out/p2p_${p}_${f}_${s}.err | tail -5
done
