timeout 300 python -m pytest tests/test_gpu_layers.py tests/test_gpu_loopback.py tests/test_gpu_full_size.py -x -q -k "backward_parity or loopback or full_size or planner" > gpurun_out/r02x_t.log 2>&1; echo "t rc=$?"
for v in 0 1; do CP_TC_DGRAD_PAIRS=$v timeout 300 python bench.py > gpurun_out/r02x_n1_pairs$v.json 2> gpurun_out/r02x_n1_pairs$v.err; echo "n1 pairs=$v rc=$?"; done
for v in 0 1; do CP_TC_DGRAD_PAIRS=$v timeout 300 python bench.py > gpurun_out/r02x_n1b_pairs$v.json 2> gpurun_out/r02x_n1b_pairs$v.err; echo "n1b pairs=$v rc=$?"; done
