mkdir -p gpurun_out
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ref.json 2> gpurun_out/ref.err; cat gpurun_out/ref.json; tail -2 gpurun_out/ref.err
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 7 python __graft_entry__.py smoke > gpurun_out/memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"; tail -4 gpurun_out/memcheck_smoke.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests/test_gpu_variants.py -q -x -k "bitwise or (pcg and 64x64)" > gpurun_out/memcheck_var.log 2>&1; echo "memcheck variants rc=$?"; tail -4 gpurun_out/memcheck_var.log
