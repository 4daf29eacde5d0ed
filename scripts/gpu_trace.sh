mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
LDU_TRACE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 2 --warmup 3 --solver pipecg --no-secondary --no-e2e --no-profile > gpurun_out/trace.json 2> gpurun_out/trace.err
grep "ldu trace" gpurun_out/trace.err | tail -8
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 5 --warmup 3 --solver pipecg --no-secondary --no-e2e --no-profile > gpurun_out/noprof.json 2> gpurun_out/noprof.err
grep "^{" gpurun_out/noprof.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('no-profile', d['value'])"
