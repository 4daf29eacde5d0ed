# AMG launch list + full capture of K4 (RHO / no RHO), exported to CSV on the box
mkdir -p gpurun_out
CMD="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0 --only amg_pcg"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_vc|k_csr_vec|k_sell_rows|k_dense_mv|k_amg" --log-file gpurun_out/amg_launches.csv $CMD > gpurun_out/amg_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/amg_ncu.log
CMD2="python scripts/amg_bench.py --n 256 --reps 1 --jacobi 0"
for spec in "rho 30" "norho 80"; do set -- $spec
timeout 600 ncu --set full --clock-control none -k regex:k_vc_post -s $2 -c 1 -o /tmp/vc_$1 $CMD2 > gpurun_out/ncu_full_$1.log 2>&1; echo "ncu full $1 rc=$?"
ncu -i /tmp/vc_$1.ncu-rep --page details --csv > gpurun_out/vc_post_$1.details.csv 2>&1
ncu -i /tmp/vc_$1.ncu-rep --page raw --csv > gpurun_out/vc_post_$1.raw.csv 2>&1
done
ls -la gpurun_out
