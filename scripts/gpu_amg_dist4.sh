mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x -k amg > gpurun_out/amg_dist4.log 2>&1; echo "dist amg rc=$?"; tail -3 gpurun_out/amg_dist4.log
for g in 1 2 4; do for n in 256 512; do
  if [ $g = 1 ]; then LDU_AMG_TRACE=1 timeout 900 python scripts/amg_dist_bench.py --mesh $n > gpurun_out/amgd_${n}_$g.jsonl 2> gpurun_out/amgd_${n}_$g.err;
  else timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr=127.0.0.1 --master-port=29541 scripts/amg_dist_bench.py --mesh $n > gpurun_out/amgd_${n}_$g.jsonl 2> gpurun_out/amgd_${n}_$g.err; fi
  echo "n=$n gpus=$g rc=$?"; cat gpurun_out/amgd_${n}_$g.jsonl; tail -2 gpurun_out/amgd_${n}_$g.err
done; done
