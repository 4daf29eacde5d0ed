# AMG (NEXT-2) first GPU pass: parity tests, then time-to-solution at 64^3 / 128^3 / 256^3.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_amg.py -x -q > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -30 gpurun_out/amg_pytest.log
timeout 900 python scripts/amg_bench.py --n 64 128 256 --tol 1e-8 > gpurun_out/amg_bench.jsonl 2> gpurun_out/amg_bench.err; echo "amg bench rc=$?"; cat gpurun_out/amg_bench.jsonl; tail -5 gpurun_out/amg_bench.err
