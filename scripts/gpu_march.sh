# march variant: parity first (stop on failure), then variants 0 vs 3 on config 3
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -5 || exit 1
for v in 0 3; do
  for s in pcg pipecg; do
    LDU_VARIANT=$v python bench.py --steps 3 --warmup 3 --iters 100 --solver $s --no-cpu-baseline --no-e2e \
      > gpurun_out/var_${v}_${s}.json 2> gpurun_out/var_${v}_${s}.err
    python -c "import json;d=json.load(open('gpurun_out/var_${v}_${s}.json'));r=d['roofline'];print('v$v $s', round(d['value'],1), 'iter/s eff', round(d['effective_frac_of_hbm'],3), r['kernel'], round(r['launch_us'],1),'us fmt_frac', round(r['format_frac'],3), 'share', round(r['share_of_step'],3))" || tail -3 gpurun_out/var_${v}_${s}.err
  done
done
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile"
LDU_VARIANT=3 $CMD > gpurun_out/m_small.json 2> gpurun_out/m_small.err && \
LDU_VARIANT=3 ncu --set full --clock-control none --import-source on -k regex:k_march -s 5 -c 1 -o gpurun_out/marchA $CMD > gpurun_out/ncu_m.log 2>&1
echo ncu rc=$?
