mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in 0 6; do
  LDU_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --solver pcg --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/v6_$v.json 2> gpurun_out/v6_$v.err
  python -c "import json;d=json.load(open('gpurun_out/v6_$v.json'));r=d['roofline'];print('v$v pcg', round(d['value'],1), r['kernel'], round(r['launch_us'],1),'us fmt', round(r['format_frac'],3))" || tail -3 gpurun_out/v6_$v.err
done
timeout 600 python scripts/bench_configs.py c2 > gpurun_out/cfg_c2b.jsonl 2> gpurun_out/cfg_c2b.err; cat gpurun_out/cfg_c2b.jsonl | cut -c1-250
