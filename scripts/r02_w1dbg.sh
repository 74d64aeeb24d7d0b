for d in 64 128 256; do CUDA_LAUNCH_BLOCKING=1 CP_W1_DBG=$d timeout 60 python scripts/w1_debug.py > gpurun_out/r02m_dbg$d.log 2>&1; echo "dbg $d rc=$?"; done
