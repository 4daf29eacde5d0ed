cd $GRAFT_REPO_ROOT
for m in 1 0; do
echo "=== LDU_PIPE_FUSE=$m"
LDU_DIST_BOOT=host LDU_PIPE_FUSE=$m timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=2955$m tests/dist_worker.py > gpurun_out/r2_diag_f$m.log 2>&1
grep -v "Warning\|warn" gpurun_out/r2_diag_f$m.log | grep "DIST\|differs\|rank\|Error" | cut -c1-600 | head -20
done
