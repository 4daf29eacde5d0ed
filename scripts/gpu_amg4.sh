# AMG kernel tuning + DRAM stagger experiment
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_amg.py -q -x > gpurun_out/amg_pytest.log 2>&1; echo "amg pytest rc=$?"; tail -3 gpurun_out/amg_pytest.log
for st in 0 4096 1536 65792; do
  LDU_STAGGER=$st timeout 600 python scripts/amg_bench.py --n 256 --tol 1e-8 --reps 3 > gpurun_out/amg_bench_st$st.jsonl 2> gpurun_out/amg_bench_st$st.err; echo "stagger $st rc=$?"
  python -c "
import json
for l in open('gpurun_out/amg_bench_st$st.jsonl'):
    d=json.loads(l); print('$st', d['solver'], d['iters'], round(d['solve_ms'],2), round(d['ms_per_iter'],4), [round(x,4) for x in d['pass_ms_per_iter']])"
  LDU_STAGGER=$st timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_st$st.json 2> gpurun_out/bench_st$st.err
  python -c "
import json; d=json.loads(open('gpurun_out/bench_st$st.json').read().strip().splitlines()[-1]); print('$st bench', round(d['value'],1), d['roofline']['format_frac'], d['secondary']['value'])"
done
CMD="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_vc|k_csr_vec|k_sell_rows|k_dense_mv|k_amg" --log-file gpurun_out/amg_launches.csv $CMD > gpurun_out/amg_ncu.log 2>&1; echo "ncu rc=$?"
