mkdir -p gpurun_out
timeout 900 python scripts/amg_bench.py --n 256 --tol 1e-8 --reps 3 --jacobi 0 > gpurun_out/cv_amg.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/cv_amg.jsonl'):
    d=json.loads(l); print(d['solver'], d['iters'], round(d['solve_ms'],2), round(d['ms_per_iter'],4), [round(x,4) for x in d['pass_ms_per_iter']])"
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/cv_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/cv_pytest.log
