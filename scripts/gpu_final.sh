# Round-end evidence: full GPU tests, smoke, default bench line (incl. AMG leg), reference arm,
# ncu launch list of the headline bench command, ncu --set full of the dominant kernels (CSV).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?"; cat gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc=$?"; cat gpurun_out/final_ref.json
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile --no-amg"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches.csv $CMD > gpurun_out/final_ncu_l.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pipe_SU -s 5 -c 1 -o /tmp/pipeSU $CMD > gpurun_out/final_ncu_su.log 2>&1; echo "ncu SU rc=$?"
ncu -i /tmp/pipeSU.ncu-rep --page details --csv > gpurun_out/final_pipeSU.details.csv 2>&1
ncu -i /tmp/pipeSU.ncu-rep --page raw --csv > gpurun_out/final_pipeSU.raw.csv 2>&1
CMD2="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sell_rows -s 10 -c 1 -o /tmp/sell $CMD2 > gpurun_out/final_ncu_sell.log 2>&1; echo "ncu sell rc=$?"
ncu -i /tmp/sell.ncu-rep --page details --csv > gpurun_out/final_sell_rows.details.csv 2>&1
