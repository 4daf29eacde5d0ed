mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile"
LDU_VARIANT=3 $CMD > gpurun_out/m_small.json 2> gpurun_out/m_small.err && \
LDU_VARIANT=3 ncu --set full --clock-control none --import-source on -k regex:k_march -s 5 -c 1 -o gpurun_out/marchA $CMD > gpurun_out/ncu_m.log 2>&1
echo rc=$?; tail -2 gpurun_out/ncu_m.log
