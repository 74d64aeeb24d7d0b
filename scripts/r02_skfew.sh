# split-K reduce for S <= 8 (one thread per float4, all splits in flight) vs the 8-lane kernel; P=8 slice step
for v in 0 1; do
  CP_TC_SPLITK_FEW=$v P=8 STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:splitk --csv --log-file gpurun_out/r02k_P8_few$v.csv python scripts/slice_step.py > gpurun_out/r02k_ncu_$v.log 2>&1; echo "ncu few=$v rc=$?"
  CP_TC_SPLITK_FEW=$v P=8 timeout 300 python scripts/slice_step.py > gpurun_out/r02k_P8_few$v.json 2>&1; echo "few=$v rc=$?"; tail -1 gpurun_out/r02k_P8_few$v.json
done
timeout 1200 python -m pytest tests/test_gpu_layers.py tests/test_gpu_full_size.py tests/test_gpu_trajectory.py tests/test_gpu_loopback.py -x -q -m gpu > gpurun_out/r02k_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02k_tests.log
