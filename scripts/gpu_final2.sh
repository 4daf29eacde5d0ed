# Round-end evidence (4-GPU box): full GPU tests, smoke, bench at 1/2/4 GPUs, reference arm,
# headline launch list and full captures (CSV), AMG launch list.
mkdir -p gpurun_out/final2
O=gpurun_out/final2
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
for g in 1 2 4; do
  if [ $g = 1 ]; then timeout 900 python bench.py > $O/bench_1.json 2> $O/bench_1.err;
  else timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$g --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus $g > $O/bench_$g.json 2> $O/bench_$g.err; fi
  echo "bench $g rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile --no-amg"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_headline_iters20.csv $CMD > $O/ncu_l.log 2>&1; echo "ncu list rc=$?"
for k in k_pipe_SU k_cg_passA2 k_cg_passA1; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 5 -c 1 -o /tmp/$k $CMD > $O/ncu_$k.log 2>&1; echo "ncu $k rc=$?"
ncu -i /tmp/$k.ncu-rep --page details --csv > $O/ncu_full_$k.details.csv 2>&1
ncu -i /tmp/$k.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > $O/ncu_full_$k.raw_subset.csv 2>&1
done
CMD2="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_vc|k_csr_vec|k_sell_rows|k_dense_mv|k_amg" --log-file $O/launches_amg_pcg_256.csv $CMD2 > $O/amg_ncu.log 2>&1; echo "ncu amg rc=$?"
