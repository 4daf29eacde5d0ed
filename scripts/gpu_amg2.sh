# AMG parity tests, time to solution, and the ncu launch list of one 256^3 AMG-PCG solve
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_amg.py -q > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -15 gpurun_out/amg_pytest.log
timeout 900 python scripts/amg_bench.py --n 128 256 --tol 1e-8 --jacobi 0 > gpurun_out/amg_bench.jsonl 2> gpurun_out/amg_bench.err; echo "amg bench rc=$?"; cat gpurun_out/amg_bench.jsonl; tail -5 gpurun_out/amg_bench.err
CMD="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_vc|k_csr_vec|k_dense_mv|k_amg" --log-file gpurun_out/amg_launches.csv $CMD > gpurun_out/amg_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/amg_ncu.log
