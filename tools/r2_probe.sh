mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2p_smi.txt
timeout 900 python tools/profile_classes.py probminhash1,probminhash2,probminhash3,probminhash4 > gpurun_out/r2p_classes.log 2>&1
