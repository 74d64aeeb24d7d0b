# e2e gap probe, then ncu --set full of one whole training step (all kernels in the NVTX "step" range)
timeout 300 python scripts/e2e_probe.py > gpurun_out/r02d_e2e.txt 2>&1; echo "e2e rc=$?"
timeout 300 python scripts/prof_step.py > gpurun_out/r02d_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -o gpurun_out/r02d_step python scripts/prof_step.py > gpurun_out/r02d_ncu.log 2>&1; echo "ncu rc=$?"
