P=8 timeout 200 python scripts/prof_step.py > gpurun_out/r02q_plain.log 2>&1 && \
P=8 timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -k regex:conv1 -o gpurun_out/r02q_c1p8 python scripts/prof_step.py > gpurun_out/r02q_ncu.log 2>&1; echo "ncu rc=$?"
