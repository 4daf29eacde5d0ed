mkdir -p gpurun_out
timeout 900 python scripts/bench_configs.py c2amg > gpurun_out/cfg_c2amg.jsonl 2> gpurun_out/cfg_c2amg.err; echo "c2amg rc=$?"; cat gpurun_out/cfg_c2amg.jsonl; tail -2 gpurun_out/cfg_c2amg.err
timeout 1500 python scripts/bench_configs.py c5amg > gpurun_out/cfg_c5amg.jsonl 2> gpurun_out/cfg_c5amg.err; echo "c5amg rc=$?"; cat gpurun_out/cfg_c5amg.jsonl; tail -2 gpurun_out/cfg_c5amg.err
