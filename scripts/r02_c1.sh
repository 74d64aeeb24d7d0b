# new conv1 forward kernel: targeted parity first (short timeout), then the GPU suite, then bench N=1
timeout 180 python -m pytest tests/test_gpu_layers.py -x -q -k "test_forward_parity" > gpurun_out/r02e_fwd.log 2>&1; echo "fwd rc=$?"
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02e_all.log 2>&1; echo "all rc=$?"
timeout 300 python bench.py > gpurun_out/r02e_n1.json 2> gpurun_out/r02e_n1.err; echo "n1 rc=$?"
