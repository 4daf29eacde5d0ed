mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -2
for cfg in "0 2048" "5 1024" "5 2048" "5 4096" "5 8192"; do
  set -- $cfg; v=$1; K=$2
  for s in pcg pipecg; do
    LDU_VARIANT=$v LDU_CHUNK=$K timeout 300 python bench.py --steps 3 --warmup 3 --iters 100 --solver $s --no-cpu-baseline --no-e2e \
      > gpurun_out/var_${v}_K${K}_${s}.json 2> gpurun_out/var_${v}_K${K}_${s}.err
    python -c "import json;d=json.load(open('gpurun_out/var_${v}_K${K}_${s}.json'));r=d['roofline'];print('v$v K$K $s', round(d['value'],1), 'iter/s eff', round(d['effective_frac_of_hbm'],3), r['kernel'], round(r['launch_us'],1),'us fmt_frac', round(r['format_frac'],3), 'share', round(r['share_of_step'],3))" || tail -3 gpurun_out/var_${v}_K${K}_${s}.err
  done
done
