mkdir -p gpurun_out
for mb in 0 6 8; do
  LDU_SU_MINB=$mb timeout 600 python bench.py --no-amg --no-secondary --no-cpu-baseline --no-e2e > gpurun_out/su_$mb.json 2> gpurun_out/su_$mb.err; echo "minb $mb rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/su_$mb.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$mb', round(d['value'],1), round(r['launch_us'],1), round(r['format_frac'],4))"
done
LDU_SU_MINB=8 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k pipecg > gpurun_out/su_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/su_pytest.log
