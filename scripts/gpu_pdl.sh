mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29533 tests/dist_worker.py > gpurun_out/dw.log 2>&1; echo "dist rc=$?"; grep -E "DIST" gpurun_out/dw.log | cut -c1-40; grep -iE "error|assert" gpurun_out/dw.log | head -3
bash scripts/gpu_gtimer.sh
for pdl in 1 0; do
LDU_PDL=$pdl timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $NG --steps 5 --warmup 3 --no-e2e > gpurun_out/b4.json 2>gpurun_out/b4.err; grep "^{" gpurun_out/b4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"N=$NG pdl=$pdl\", round(d[\"value\"],1), \"pcg\", round(d[\"secondary\"][\"value\"],1))"
done
