timeout 600 python -m pytest tests/test_gpu_layers.py -x -q -k "variants" > gpurun_out/c1_tests.log 2>&1; echo "tests rc=$?"
CP_TC_FWD_T_IMAGES=1 timeout 300 python -m pytest tests/test_gpu_full_size.py -x -q > gpurun_out/c1_fs.log 2>&1; echo "fullsize rc=$?"
for P in 1 4; do for t in 0 1 0 1; do P=$P CP_TC_FWD_T_IMAGES=$t timeout 60 python scripts/conv1_fwd_time.py; done; done
