mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile --solver pcg --no-secondary"
$CMD > gpurun_out/a12_small.json 2> gpurun_out/a12_small.err && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passA1 -s 5 -c 1 -o gpurun_out/passA1 $CMD > gpurun_out/ncu_a1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passA2 -s 5 -c 1 -o gpurun_out/passA2s $CMD > gpurun_out/ncu_a2.log 2>&1
echo ncu rc=$?
