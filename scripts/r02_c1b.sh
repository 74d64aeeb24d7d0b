timeout 120 python scripts/conv1_bench.py > gpurun_out/r02f_conv1.jsonl 2>&1; echo "c1 rc=$?"
timeout 300 python -m pytest tests/test_gpu_layers.py -x -q -k "test_backward_parity or full_step_p1 or image_dgrad" > gpurun_out/r02f_bwd.log 2>&1; echo "bwd rc=$?"
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02f_all.log 2>&1; echo "all rc=$?"
timeout 300 python bench.py > gpurun_out/r02f_n1.json 2> gpurun_out/r02f_n1.err; echo "n1 rc=$?"
