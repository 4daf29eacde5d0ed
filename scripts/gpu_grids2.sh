mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/gr2_bench.json 2> gpurun_out/gr2_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/gr2_bench.json').read().strip().splitlines()[-1]); r=d['roofline']; a=d.get('amg') or {}; sc=d['secondary']
print(round(d['value'],1), round(r['launch_us'],1), round(r['format_frac'],4), 'pcg', round(sc['value'],1), round(sc['roofline']['launch_us'],1), round(sc['roofline']['format_frac'],4), 'amg', a.get('ms_per_solve'), a.get('ms_per_iter'), (a.get('vcycle') or {}).get('frac'))"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amg.py -q -x > gpurun_out/gr2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/gr2_pytest.log
