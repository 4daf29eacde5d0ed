set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/b_pcg.json 2> gpurun_out/b_pcg.err; tail -3 gpurun_out/b_pcg.err
python bench.py --steps 5 --warmup 3 --solver pipecg --no-cpu-baseline > gpurun_out/b_pipe.json 2> gpurun_out/b_pipe.err; tail -3 gpurun_out/b_pipe.err
LDU_LAYOUT=sell python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_sell.json 2> gpurun_out/b_sell.err; tail -3 gpurun_out/b_sell.err
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile"
$CMD > gpurun_out/small.json 2> gpurun_out/small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passA -s 3 -c 1 -o gpurun_out/passA $CMD > gpurun_out/ncu2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passB -s 3 -c 1 -o gpurun_out/passB $CMD > gpurun_out/ncu3.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu2.log
