mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dist_gpu.py -q -x -k amg > gpurun_out/amg_dist.log 2>&1; echo "dist amg rc=$?"; tail -30 gpurun_out/amg_dist.log
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
