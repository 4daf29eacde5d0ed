mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/h_small.json 2> gpurun_out/h_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv $CMD > gpurun_out/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pipe_SU -s 5 -c 1 -o gpurun_out/pipeSU $CMD > gpurun_out/ncu_su.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passA -s 5 -c 1 -o gpurun_out/passA2 $CMD > gpurun_out/ncu_a.log 2>&1
echo ncu rc=$?
