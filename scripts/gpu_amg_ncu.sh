#!/bin/bash
# Per-kernel time and DRAM bytes of one AMG-PCG solve at 256^3 (launch list with DRAM metrics).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2_amg_ncu
python scripts/amg_solve_once.py 256 > gpurun_out/r2_amg_ncu/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_vc|k_amg|k_sell|k_csr|k_dense|k_ell" --csv --log-file gpurun_out/r2_amg_ncu/launches.csv \
    python scripts/amg_solve_once.py 256 > gpurun_out/r2_amg_ncu/ncu.log 2>&1
echo rc=$?; cat gpurun_out/r2_amg_ncu/plain.log
