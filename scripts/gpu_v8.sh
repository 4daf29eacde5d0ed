mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x 2>&1 | tail -2
for cfg in "7 8" "8 8" "8 4"; do set -- $cfg
  LDU_VARIANT=$1 LDU_YR=$2 timeout 300 python bench.py --steps 5 --warmup 3 --solver pcg --no-cpu-baseline --no-e2e --no-secondary > gpurun_out/v8_$1_$2.json 2> gpurun_out/v8_$1_$2.err
  python -c "import json;d=json.load(open('gpurun_out/v8_$1_$2.json'));r=d['roofline'];print('v$1 R$2 pcg', round(d['value'],1), r['kernel'], round(r['launch_us'],1),'us')" || tail -3 gpurun_out/v8_$1_$2.err
done
