mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -2
for v in 0 7; do
  LDU_VARIANT=$v timeout 300 python bench.py --steps 5 --warmup 3 --solver pcg --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/v7_$v.json 2> gpurun_out/v7_$v.err
  python -c "import json;d=json.load(open('gpurun_out/v7_$v.json'));r=d['roofline'];print('v$v pcg', round(d['value'],1), r['kernel'], round(r['launch_us'],1),'us')" || tail -3 gpurun_out/v7_$v.err
done
