# conv2 wgrad stream-tail reduce: 8-deep vs 32-deep piece batches (same order)
for v in wt8 wt32; do for P in 1 4 8; do
  CP_LIB=exp/libconvpart_$v.so P=$P STEPS=3 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:wgrad_tail --csv --log-file gpurun_out/r02w_${v}_P$P.csv python scripts/slice_step.py > /dev/null 2>&1; echo "$v P=$P rc=$?"
done; done
timeout 900 python -m pytest tests/test_gpu_layers.py tests/test_gpu_trajectory.py tests/test_gpu_full_size.py -x -q -m gpu > gpurun_out/r02w_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02w_tests.log
