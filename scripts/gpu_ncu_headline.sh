#!/bin/bash
# Headline evidence at 256^3 (one GPU): launch list of the timed command and one `ncu --set full`
# capture each of the fused pipelined pass and the classical pass A kernels.  Usage: <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
mkdir -p gpurun_out/$TAG
CMD="python bench.py --steps 1 --warmup 3 --iters 20 --no-cpu-baseline --no-e2e --no-profile --no-amg"
$CMD > gpurun_out/$TAG/h_small.json 2> gpurun_out/$TAG/h_small.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_headline_iters20.csv $CMD > gpurun_out/$TAG/ncu_l.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pipe_SU -s 5 -c 1 -o gpurun_out/$TAG/pipeSU $CMD > gpurun_out/$TAG/ncu_su.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_cg_passA -s 10 -c 2 -o gpurun_out/$TAG/passA $CMD > gpurun_out/$TAG/ncu_a.log 2>&1
echo ncu rc=$?
# keep what is judged (raw metrics + details pages), drop the large reports before copy-back
for r in pipeSU passA; do
  if [ -f gpurun_out/$TAG/$r.ncu-rep ]; then
    ncu -i gpurun_out/$TAG/$r.ncu-rep --page raw --csv > gpurun_out/$TAG/ncu_full_$r.raw.csv 2>/dev/null
    ncu -i gpurun_out/$TAG/$r.ncu-rep --page details --csv > gpurun_out/$TAG/ncu_full_$r.details.csv 2>/dev/null
    rm -f gpurun_out/$TAG/$r.ncu-rep
  fi
done
ls -la gpurun_out/$TAG
