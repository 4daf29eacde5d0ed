# AMG parity tests + ncu launch list of one 256^3 AMG-PCG / AMG-PipeCG solve (solve kernels only)
mkdir -p gpurun_out
#timeout 1500 python -m pytest tests/test_gpu_amg.py -q > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -15 gpurun_out/amg_pytest.log
CMD="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_vc|k_csr_vec|k_dense_mv|k_amg" --log-file gpurun_out/amg_launches.csv $CMD > gpurun_out/amg_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/amg_ncu.log
