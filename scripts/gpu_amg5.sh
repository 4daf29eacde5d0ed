mkdir -p gpurun_out
LDU_AMG_TRACE=1 timeout 600 python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg --setups 5 > gpurun_out/amg_trace.jsonl 2> gpurun_out/amg_trace.err; echo "trace rc=$?"; grep "amg setup" gpurun_out/amg_trace.err | grep -v "  0\.\| 1\.\| 2\." ; cat gpurun_out/amg_trace.jsonl
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
