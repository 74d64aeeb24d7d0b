timeout 120 python scripts/conv1_bench.py > gpurun_out/r02p2_conv1.jsonl 2>&1; echo "c1 rc=$?"
timeout 300 python -m pytest tests/test_gpu_layers.py tests/test_gpu_full_size.py tests/test_gpu_trajectory.py -x -q -k "forward_parity or backward_parity or full_step or image_dgrad or full_size or head or trajectory" > gpurun_out/r02p2_t.log 2>&1; echo "t rc=$?"
timeout 300 python bench.py > gpurun_out/r02p2_n1.json 2> gpurun_out/r02p2_n1.err; echo "n1 rc=$?"
timeout 200 python scripts/prof_step.py > gpurun_out/r02p2_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "step/" -k regex:conv1 -o gpurun_out/r02p2_c1 python scripts/prof_step.py > gpurun_out/r02p2_ncu.log 2>&1; echo "ncu rc=$?"
