mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29551"
timeout 300 $R scripts/p2p_repro.py 512 pipe,pipe,pcg,pipe,pipe0 > gpurun_out/repro1.log 2>&1; echo "repro1 rc=$?"; grep "step\|REPRO" gpurun_out/repro1.log
timeout 300 $R scripts/p2p_repro.py 512 pipe0,pipe0 > gpurun_out/repro2.log 2>&1; echo "repro2 rc=$?"; grep "step\|REPRO" gpurun_out/repro2.log
LDU_P2P=0 timeout 300 $R scripts/p2p_repro.py 512 pipe,pcg > gpurun_out/repro3.log 2>&1; echo "repro3 (nccl) rc=$?"; grep "step\|REPRO" gpurun_out/repro3.log
LDU_PDL=0 timeout 300 $R scripts/p2p_repro.py 512 pipe,pipe > gpurun_out/repro4.log 2>&1; echo "repro4 (no pdl) rc=$?"; grep "step\|REPRO" gpurun_out/repro4.log
