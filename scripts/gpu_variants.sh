# Compare SpMV-pass kernel variants (LDU_VARIANT) on config 3; then the GPU test-suite.
mkdir -p gpurun_out
for v in 0 1 2; do
  for s in pcg pipecg; do
    LDU_VARIANT=$v python bench.py --steps 3 --warmup 3 --iters 100 --solver $s --no-cpu-baseline --no-e2e \
      > gpurun_out/var_${v}_${s}.json 2> gpurun_out/var_${v}_${s}.err
    python -c "import json;d=json.load(open('gpurun_out/var_${v}_${s}.json'));r=d['roofline'];print('v$v $s', round(d['value'],1), 'iter/s eff', round(d['effective_frac_of_hbm'],3), r['kernel'], round(r['launch_us'],1),'us fmt_frac', round(r['format_frac'],3))" || tail -3 gpurun_out/var_${v}_${s}.err
  done
done
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
