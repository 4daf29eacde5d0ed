mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for pv in 0 1; do
  LDU_PERSIST=$pv timeout 300 python scripts/bench_configs.py c1 > gpurun_out/p_c1_$pv.jsonl 2>&1; echo "persist=$pv"; cut -c1-200 gpurun_out/p_c1_$pv.jsonl
  LDU_PERSIST=$pv timeout 600 python scripts/bench_configs.py c2 > gpurun_out/p_c2_$pv.jsonl 2>&1; grep icoFoam gpurun_out/p_c2_$pv.jsonl | cut -c1-250
  LDU_PERSIST=$pv timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p_c3_$pv.json 2>&1; python -c "import json;d=[json.loads(l) for l in open('gpurun_out/p_c3_$pv.json') if l.startswith('{')][0];print('c3', round(d['value'],1), 'pcg', round(d['secondary']['value'],1))"
done
