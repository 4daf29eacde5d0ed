# Multi-GPU: distributed parity + bench at N = 1, 2, 4 (whatever the box has)
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29533 tests/dist_worker.py 2>&1 | grep DIST
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  for s in pcg pipecg; do
    if [ $n -eq 1 ]; then
      python bench.py --steps 5 --warmup 3 --solver $s --no-cpu-baseline > gpurun_out/scale_${s}_$n.json 2> gpurun_out/scale_${s}_$n.err
    else
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=29534 bench.py --gpus $n --steps 5 --warmup 3 --solver $s > gpurun_out/scale_${s}_$n.json 2> gpurun_out/scale_${s}_$n.err
    fi
    python -c "import json;d=json.load(open('gpurun_out/scale_${s}_$n.json'));r=d['roofline'];print('N=$n $s', round(d['value'],1), 'iter/s eff', round(d['effective_frac_of_hbm'],3), r['kernel'], round(r['launch_us'],1),'us', 'e2e', d['e2e'] and round(d['e2e']['value'],1), 'clk', d['clocks'])" || tail -5 gpurun_out/scale_${s}_$n.err
  done
done
