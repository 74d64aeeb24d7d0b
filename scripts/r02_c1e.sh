timeout 120 python scripts/conv1_bench.py > gpurun_out/r02r_conv1.jsonl 2>&1; echo "c1 rc=$?"
timeout 300 python -m pytest tests/test_gpu_layers.py -x -q -k "forward_parity or backward_parity" > gpurun_out/r02r_t.log 2>&1; echo "t rc=$?"
