# conv1 wgrad reduce: 8-deep batches (skfew lib) vs 16-deep (c1red) vs all-in-flight (c1red2)
for v in skfew c1red c1red2; do for P in 1 4; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:conv1_wgrad_reduce --csv --log-file gpurun_out/r02r_${v}_P$P.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py -x -q -m gpu > gpurun_out/r02r_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02r_tests.log
