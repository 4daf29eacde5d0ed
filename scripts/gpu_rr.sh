mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/rr_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/rr_all.log; grep -B5 "Error" gpurun_out/rr_all.log | head -30
