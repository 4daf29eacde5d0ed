mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
free -g | head -2; nproc
timeout 300 python scripts/bench_configs.py c1 > gpurun_out/cfg_c1.jsonl 2> gpurun_out/cfg_c1.err; cat gpurun_out/cfg_c1.jsonl; tail -2 gpurun_out/cfg_c1.err
timeout 600 python scripts/bench_configs.py c2 > gpurun_out/cfg_c2.jsonl 2> gpurun_out/cfg_c2.err; cat gpurun_out/cfg_c2.jsonl; tail -2 gpurun_out/cfg_c2.err
timeout 900 python scripts/bench_configs.py c5 > gpurun_out/cfg_c5.jsonl 2> gpurun_out/cfg_c5.err; cat gpurun_out/cfg_c5.jsonl; tail -2 gpurun_out/cfg_c5.err
for n in 1 2 4; do
  [ $n -gt $NG ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=29535 scripts/bench_configs.py c4 > gpurun_out/cfg_c4_$n.jsonl 2> gpurun_out/cfg_c4_$n.err; grep "^{" gpurun_out/cfg_c4_$n.jsonl; grep -i error gpurun_out/cfg_c4_$n.err | head -3
done
