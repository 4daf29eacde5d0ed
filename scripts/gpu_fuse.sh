mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for f in 1 0; do
  LDU_PIPE_FUSE=$f timeout 300 python bench.py --steps 3 --warmup 3 --iters 100 --solver pipecg --no-cpu-baseline --no-e2e > gpurun_out/fuse_$f.json 2> gpurun_out/fuse_$f.err
  python -c "import json;d=json.load(open('gpurun_out/fuse_$f.json'));r=d['roofline'];print('fuse $f', round(d['value'],1), 'iter/s eff', round(d['effective_frac_of_hbm'],3), r['kernel'], round(r['launch_us'],1),'us fmt_frac', round(r['format_frac'],3), 'share', round(r['share_of_step'],3))" || tail -3 gpurun_out/fuse_$f.err
done
