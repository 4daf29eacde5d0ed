mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/gr_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gr_pytest.log
timeout 900 python bench.py > gpurun_out/gr_bench.json 2> gpurun_out/gr_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/gr_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; a=d.get('amg') or {}; sc=d['secondary']
print(round(d['value'],1), round(r['launch_us'],1), round(r['format_frac'],4), 'pcg', round(sc['value'],1), round(sc['roofline']['launch_us'],1), round(sc['roofline']['format_frac'],4), 'amg', a.get('ms_per_solve'), a.get('ms_per_iter'), (a.get('vcycle') or {}).get('frac'))"
timeout 900 python scripts/amg_bench.py --n 256 --tol 1e-8 --reps 3 --jacobi 0 > gpurun_out/gr_amg.jsonl 2>/dev/null; python -c "
import json
for l in open('gpurun_out/gr_amg.jsonl'):
    d=json.loads(l); print(d['solver'], d['iters'], round(d['solve_ms'],2), round(d['ms_per_iter'],4), [round(x,4) for x in d['pass_ms_per_iter']])"
