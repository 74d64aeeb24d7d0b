timeout 120 python scripts/conv1_bench.py > gpurun_out/r02g_conv1.jsonl 2>&1; echo "c1 rc=$?"
timeout 300 python -m pytest tests/test_gpu_full_size.py -x -q > gpurun_out/r02g_full.log 2>&1; echo "full rc=$?"
timeout 200 python scripts/prof_step.py > gpurun_out/r02g_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -k regex:conv1 -o gpurun_out/r02g_c1 python scripts/prof_step.py > gpurun_out/r02g_ncu.log 2>&1; echo "ncu rc=$?"
