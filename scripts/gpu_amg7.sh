mkdir -p gpurun_out
LDU_AMG_TRACE=1 timeout 600 python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --setups 3 --only amg_pcg > gpurun_out/amg_trace.jsonl 2> gpurun_out/amg_trace.err; echo "trace rc=$?"; grep "amg setup" gpurun_out/amg_trace.err | tail -24 | head -13; cut -c1-200 gpurun_out/amg_trace.jsonl
LDU_AMG_RADIX=1 LDU_AMG_TRACE=1 timeout 600 python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --setups 3 --only amg_pcg > gpurun_out/amg_trace2.jsonl 2> gpurun_out/amg_trace2.err; echo "trace2 rc=$?"; grep "amg setup" gpurun_out/amg_trace2.err | tail -24 | head -13
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
