mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile"
LDU_VARIANT=4 $CMD > gpurun_out/t_small.json 2> gpurun_out/t_small.err && \
LDU_VARIANT=4 ncu --set full --clock-control none --import-source on -k regex:k_tma_march -s 5 -c 1 -o gpurun_out/tmaA $CMD > gpurun_out/ncu_t.log 2>&1
echo ncu rc=$?
