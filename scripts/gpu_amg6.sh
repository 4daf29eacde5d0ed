mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
LDU_AMG_TRACE=1 timeout 600 python scripts/amg_bench.py --n 256 --reps 2 --jacobi 0 --setups 4 > gpurun_out/amg_trace.jsonl 2> gpurun_out/amg_trace.err; echo "trace rc=$?"; grep "amg setup" gpurun_out/amg_trace.err | tail -24; cat gpurun_out/amg_trace.jsonl | cut -c1-300
timeout 600 python scripts/amg_bench.py --n 512 --reps 1 --jacobi 0 --setups 2 > gpurun_out/amg_512.jsonl 2> gpurun_out/amg_512.err; echo "512 rc=$?"; cat gpurun_out/amg_512.jsonl | cut -c1-400; tail -2 gpurun_out/amg_512.err
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -4 gpurun_out/smoke.log
