mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
LDU_TRACE=2 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 2 --warmup 3 --solver pipecg --no-secondary --no-e2e --no-profile > gpurun_out/gt.json 2> gpurun_out/gt.err
grep "ldu gtimer" gpurun_out/gt.err | tail -4
