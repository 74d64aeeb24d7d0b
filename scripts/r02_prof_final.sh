# ncu --set full of one whole N=1 training step on the final build (all kernels in the NVTX "step" range)
timeout 300 python scripts/prof_step.py > gpurun_out/r02z_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -o gpurun_out/r02z_step python scripts/prof_step.py > gpurun_out/r02z_ncu.log 2>&1; echo "ncu rc=$?"
